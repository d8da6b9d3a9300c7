#!/bin/bash
# Builds an A/B variant of the library into ab/<name>.so with extra nvcc defines:
#   scripts/build_variant.sh noopt -DEBL_PREFETCH=0 -DEBL_LAMBDA_ALL=0
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2512_06102_b200/csrc"
mkdir -p /tmp/ab_build_$name ../../ab
for f in ember_kernels ember_blocked ember_warp ember_det ember_rl_bits ember_synth ember_capi; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
       -Xcompiler -ffp-contract=off --expt-relaxed-constexpr "$@" -c $f.cu -o /tmp/ab_build_$name/$f.o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../../ab/$name.so /tmp/ab_build_$name/*.o build/ember_host.o \
     -Xcompiler -fopenmp -lgomp -lcudart
echo built ab/$name.so
