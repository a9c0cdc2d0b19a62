#!/bin/bash
# Build libprng_b200.so variants with extra -D flags into build/var_<tag>/ for
# A/B timing on the GPU (PRNG_B200_LIB=build/var_<tag>/libprng_b200.so).
# usage: tools/build_variants.sh tag1 "-DFOO=1" tag2 "-DFOO=2" ...
set -e
cd "$(dirname "$0")/../paper_2109_01329_b200/csrc"
NVCC=/usr/local/cuda/bin/nvcc
FL="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 -Xptxas -v --expt-relaxed-constexpr"
pids=()
while [ $# -gt 0 ]; do
  tag=$1; defs=$2; shift 2
  d=../../build/var_$tag; mkdir -p $d
  ( $NVCC $FL $defs -c -o $d/api.o api.cu 2> $d/api.ptxas.log && \
    $NVCC $FL $defs -c -o $d/calo.o calo.cu 2> $d/calo.ptxas.log && \
    $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $d/libprng_b200.so $d/api.o $d/calo.o && echo "built $tag" ) &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
