#!/bin/bash
# Run the c3 bench (device-resident leg only) once per library variant in exp_libs/.
# Usage (under gpurun): profiles/sweep.sh tag lib_a lib_b ...
TAG=$1; shift
for v in "$@"; do
  echo "== $v"
  LUDA_LIB=exp_libs/$v.so timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu --extras '' 2>&1 \
    | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()}, d['phases_ms'])"
done 2>&1 | tee gpurun_out/sweep_$TAG.txt
