#!/bin/bash
# Build variant libraries of the fused SPuM layer-1 BiGRU kernel (warps per
# block; MACRO=PMKLC_REC_WARPS sweeps the layer-0 recurrence instead) next to
# the product library, for tools/x2/gemm_variants.py. Usage: bigru_variants.sh "4 8 16"
set -e
MACRO=${MACRO:-PMKLC_FUSE_WARPS}
cd "$(dirname "$0")/../../paper_2507_12805_b200/csrc"
make -s -j8
for nw in $1; do
  d=../build/var_fuse_w${nw}; mkdir -p $d
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -prec-div=true \
    -prec-sqrt=true -ftz=false -Xcompiler -fPIC,-ffp-contract=off,-O2 -D$MACRO=$nw \
    -c kernels/bigru_kernels.cu -o $d/bigru_kernels.cu.o &
done
wait
objs=$(ls ../build/kernels/*.o ../build/host/*.o ../build/capi.cpp.o | grep -v bigru_kernels)
for nw in $1; do
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../lib/var_fuse_w${nw}.so \
    ../build/var_fuse_w${nw}/bigru_kernels.cu.o $objs -ldl
done
