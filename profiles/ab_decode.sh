#!/bin/bash
# A/B the c3 job across library builds in exp_libs/ (experiment): prints
# "<lib> ms_per_step decode_ms" per run, libraries interleaved.
# Usage: profiles/ab_decode.sh reps lib1 lib2 ...
reps=$1; shift
for r in $(seq 1 $reps); do
  for v in "$@"; do
    LUDA_LIB=exp_libs/lib_$v.so python bench.py --steps 5 --warmup 3 --extras "" --no-cpu --e2e-steps 0 > gpurun_out/ab_$v.log 2>&1
    python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}.log").read().strip().splitlines()[-1])
    print(v, d["ms_per_step"], d["kernels"]["decode"]["ms"], flush=True)
except Exception as e:
    print(v, "fail", e)
PY
  done
done
