#!/bin/bash
# Build variant libraries of the throughput-regime NT weight-gradient launch
# (8 rows per thread: ring depth S, k-tile BK) next to the product library, for
# tools/x2/gemm_variants.py. Usage: nt_variants.sh "3:32:2 4:32:2 3:64:4" (S:BK:warps per block)
set -e
cd "$(dirname "$0")/../../paper_2507_12805_b200/csrc"
make -s -j8
for v in $1; do
  IFS=: read S K NW <<< "$v"
  d=../build/var_nt_s${S}_k${K}_w${NW}; mkdir -p $d
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -prec-div=true \
    -prec-sqrt=true -ftz=false -Xcompiler -fPIC,-ffp-contract=off,-O2 -DPMKLC_NT8_S=$S -DPMKLC_NT8_BK=$K -DPMKLC_NW_WARPS=$NW \
    -c kernels/dm_kernels.cu -o $d/dm_kernels.cu.o &
done
wait
objs=$(ls ../build/kernels/*.o ../build/host/*.o ../build/capi.cpp.o | grep -v dm_kernels)
for v in $1; do
  IFS=: read S K NW <<< "$v"
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../lib/var_nt_s${S}_k${K}_w${NW}.so \
    ../build/var_nt_s${S}_k${K}_w${NW}/dm_kernels.cu.o $objs -ldl
done
