#!/bin/bash
# Build variant libraries of the 64x64 SIMT GEMM tile (ring depth STAGES, k-tile BK)
# next to the product library, for tools/x2/gemm_variants.py. (WIDE=1: 4x8 interleaved-column tile, 128 threads). Usage: gemm_variants.sh "2:32:0 2:32:1"
set -e
cd "$(dirname "$0")/../../paper_2507_12805_b200/csrc"
make -s -j8
for v in $1; do
  IFS=: read S K W <<< "$v"
  d=../build/var_s${S}_k${K}_w${W}; mkdir -p $d
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -prec-div=true \
    -prec-sqrt=true -ftz=false -Xcompiler -fPIC,-ffp-contract=off,-O2 -DPMKLC_G44_STAGES=$S -DPMKLC_G44_BK=$K -DPMKLC_G44_WIDE=$W \
    -c kernels/dm_kernels.cu -o $d/dm_kernels.cu.o
  objs=$(ls ../build/kernels/*.o ../build/host/*.o ../build/capi.cpp.o | grep -v dm_kernels)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../lib/var_s${S}_k${K}_w${W}.so $d/dm_kernels.cu.o $objs -ldl
done
