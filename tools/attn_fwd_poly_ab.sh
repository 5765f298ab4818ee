#!/bin/bash
# A/B of the forward's exponential split (POLY = element pairs in 4 on the FMA pipe) on the c2 leaf
# batch: experiment builds of attention_sm100.cu with -DTT_EXP_FWD_POLY=p linked into the trace build.
set -eu
cd paper_2602_00482_b200/csrc
make -j8 trace > /dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr"
mkdir -p ../../build/exp
OTHERS=$(ls ../../build/csrc_trace/*.o ../../build/csrc_trace/kernels/*.o | grep -v attention_sm100)
for v in 0 2; do
  nvcc $FL -DTT_EXP_FWD_POLY=$v -c kernels/attention_sm100.cu -o ../../build/exp/fwd_$v.o
  nvcc $ARCH -shared -o ../../build/exp/libfwd_$v.so ../../build/exp/fwd_$v.o $OTHERS -ldl
done
cd ../..
echo "== product (POLY 1)"; python tools/attn_bench.py 16 32768 1024 14 64 | grep fwd
for v in 0 2; do echo "== POLY $v"; ATTN_LIB=build/exp/libfwd_$v.so python tools/attn_bench.py 16 32768 1024 14 64 | grep fwd; done
