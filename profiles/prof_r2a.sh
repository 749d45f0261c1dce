set -u
bash profiles/run_ncu.sh r2a
for k in decode_kernel encode_kernel sst_meta_kernel merge_kernel; do
  ncu -i gpurun_out/prof_r2a.ncu-rep --page source --csv --print-source=cuda,sass -k regex:$k > gpurun_out/src_r2a_$k.csv 2>/dev/null
  python profiles/ncu_lines.py gpurun_out/src_r2a_$k.csv "" 40 > gpurun_out/lines_r2a_$k.txt
done
python profiles/ncu_summary.py gpurun_out/prof_r2a.ncu-rep > gpurun_out/ncu_full_r2a_summary.txt 2>&1
python profiles/launch_summary.py gpurun_out/launches_r2a.csv > gpurun_out/launches_r2a_summary.txt 2>&1
gzip -f gpurun_out/src_r2a_*.csv
ls -la gpurun_out
