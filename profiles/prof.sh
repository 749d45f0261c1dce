#!/bin/bash
# Full GPU round-trip under gpurun: launch list + ncu --set full of the c3 job's top kernels,
# per-line source summaries and the summaries that get committed under profiles/<round>/.
# Usage: profiles/prof.sh <tag>
set -u
TAG=${1:-r2}
bash profiles/run_ncu.sh $TAG
for k in decode_kernel encode_kernel sst_meta_kernel merge_kernel; do
  ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source=cuda,sass -k regex:$k > gpurun_out/src_${TAG}_$k.csv 2>/dev/null
  python profiles/ncu_lines.py gpurun_out/src_${TAG}_$k.csv "" 40 > gpurun_out/lines_${TAG}_$k.txt
done
python profiles/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep > gpurun_out/ncu_full_${TAG}_summary.txt 2>&1
python profiles/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_${TAG}_summary.txt 2>&1
python profiles/traffic_from_ncu.py gpurun_out/prof_$TAG.ncu-rep $TAG > gpurun_out/traffic_$TAG.txt 2>&1; cp profiles/traffic.json gpurun_out/traffic_$TAG.json
gzip -f gpurun_out/src_${TAG}_*.csv
ls -la gpurun_out
