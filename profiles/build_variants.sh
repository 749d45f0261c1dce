#!/bin/bash
# Build tuning variants of the library into exp_libs/ (git-ignored; shipped by gpurun).
# Usage: profiles/build_variants.sh name:"-DFOO=1 -DBAR=2" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p exp_libs
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    --extended-lambda -diag-suppress 177 $flags -o exp_libs/lib_$name.so paper_2004_03054_b200/csrc/luda_b200.cu &
done
wait
ls exp_libs
