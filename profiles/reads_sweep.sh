#!/bin/bash
# The read-path workload (bench.py --extras reads) once per library variant in exp_libs/.
for v in "$@"; do
  echo "== $v"
  LUDA_LIB=exp_libs/$v.so timeout 300 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu --extras reads 2>&1 \
    | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['workloads']['reads']; print(r['ms'], r['value'], r['e2e']['value'])"
done
