#!/bin/bash
# Build scheduling variants of libpald_gpu.so into tools/ab/ for A/B timing.
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/ab
build() {  # name flags...
  local name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -I include "$@" -o tools/ab/lib_$name.so paper_2307_16652_b200/csrc/pald_gpu.cu paper_2307_16652_b200/csrc/pald_epilogue.cu paper_2307_16652_b200/csrc/pald_io.cu
  echo built $name
}
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  build $name $flags &
done
wait
