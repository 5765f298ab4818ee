#!/bin/bash
# Resource A/B of the fused attention backward (experiment builds only; results are numerically wrong
# by construction, only the timing is read): each variant drops one consumer (TT_EXP_BWD in
# attention_bwd_sm100.cu) and is timed on the c2 leaf batch with tools/attn_bench.py.
set -eu
cd paper_2602_00482_b200/csrc
make -j8 trace > /dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr"
mkdir -p ../../build/exp
OTHERS=$(ls ../../build/csrc_trace/*.o ../../build/csrc_trace/kernels/*.o | grep -v attention_bwd_sm100)
for v in ${AB_VARIANTS:-1 2 3 4 5}; do
  nvcc $FL -DTT_EXP_BWD=$v -c kernels/attention_bwd_sm100.cu -o ../../build/exp/bwd_$v.o
  nvcc $ARCH -shared -o ../../build/exp/libbwd_$v.so ../../build/exp/bwd_$v.o $OTHERS -ldl
done
cd ../..
echo "== product"; python tools/attn_bench.py 16 32768 1024 14 64 | grep bwd
for v in ${AB_VARIANTS:-1 2 3 4 5}; do echo "== TT_EXP_BWD=$v"; ATTN_LIB=build/exp/libbwd_$v.so python tools/attn_bench.py 16 32768 1024 14 64 | grep bwd; done
