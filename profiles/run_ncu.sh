#!/bin/bash
# Profiling recipe (run under gpurun on ONE B200; numbers printed under ncu are never bench values).
#   1. launch list of one compaction step (cold-cache, serialised: compare shares, not absolutes)
#   2. ncu --set full of the top kernels of the c3 job
# Usage: profiles/run_ncu.sh <tag> [kernel-regex]
set -u
TAG=${1:-r1}
RE=${2:-"decode_kernel|encode_kernel|merge_kernel|sst_meta_kernel|block_scan_kernel|block_jump_kernel"}
mkdir -p gpurun_out
BENCH="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu --extras ''"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_${TAG}.csv $BENCH > gpurun_out/launches_${TAG}.log 2>&1
# the synthesis step builds the inputs with encode/sst_meta too: skip those launches (-s counts filtered launches)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${RE}" -s 6 -c 6 \
  -o gpurun_out/prof_${TAG} -f $BENCH > gpurun_out/prof_${TAG}.log 2>&1
ls -la gpurun_out
