#!/bin/bash
# Diagnosis build (timing only, results are WRONG): level 2's ring reads
# (LDS.128 of BOX_H2 / BOX_E2 coefficient boxes, 1,288 of the ~8,700
# shared-memory pipe cycles of a plane-iteration) replaced by constants; the
# producer stream, TMA writes, ring protocol, arithmetic and stores unchanged.
# If the capped sweep is co-limited by the shared-memory pipe (DESIGN.md "The
# second ceiling"), this build runs measurably faster than the product.
#   bash tools/smem_probe.sh           (in the dev container: builds)
#   THIIM_LIB=build/variants/libthiim_gpu_nol2lds.so python bench.py ...   (on the GPU box)
set -e
cd "$(dirname "$0")/.."
tmp=build/variants/nol2lds/csrc
rm -rf build/variants/nol2lds; mkdir -p $tmp build/variants/include; cp include/thiim_gpu.h build/variants/include/
cp paper_1510_05218_b200/csrc/* $tmp/
sed -i -E 's/RD\(([0-3]), BOX_(H2|E2)\)/make_double2(0.25 + \1, 0.125)/g' $tmp/thiim_tblock.cuh
grep -c "make_double2(0.25" $tmp/thiim_tblock.cuh
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
  -I include -Xcompiler -fPIC,-fopenmp,-ffp-contract=off,-O2 -shared \
  -o build/variants/libthiim_gpu_nol2lds.so $tmp/thiim_gpu.cu -lgomp
echo build/variants/libthiim_gpu_nol2lds.so
