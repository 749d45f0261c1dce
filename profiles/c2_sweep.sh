#!/bin/bash
# c2 latency (bench.py --extras c2) once per library variant in exp_libs/.
for v in "$@"; do
  echo "== $v"
  LUDA_LIB=exp_libs/$v.so timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu --extras c2 2>&1 \
    | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['workloads']['c2']; print(d['ms_per_step'], c['device_ms_p50'], c['host_ms_p50'], c['e2e_ms_p50'])"
done
