#!/bin/bash
# ncu --set full of ONE kernel of the c3 bench job (first compaction step).
# Usage: profiles/run_ncu_one.sh <tag> <kernel-regex> [skip]
TAG=$1; RE=$2; SKIP=${3:-0}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${RE}" -s ${SKIP} -c 1 \
  -o gpurun_out/prof_${TAG} -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu > gpurun_out/prof_${TAG}.log 2>&1
tail -3 gpurun_out/prof_${TAG}.log
