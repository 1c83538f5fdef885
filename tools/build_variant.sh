#!/bin/bash
# Build an experiment variant of the library next to the product one:
#   tools/build_variant.sh NAME [nvcc flags...]  ->  build/variants/libthiim_gpu_NAME.so
# then run anything with THIIM_LIB=build/variants/libthiim_gpu_NAME.so (A/B on one box).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
  -Xcompiler -fPIC,-fopenmp,-ffp-contract=off,-O2 -shared "$@" \
  -o build/variants/libthiim_gpu_$name.so paper_1510_05218_b200/csrc/thiim_gpu.cu -lgomp
echo build/variants/libthiim_gpu_$name.so
