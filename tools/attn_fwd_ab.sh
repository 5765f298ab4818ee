#!/bin/bash
# Resource A/B of the attention forward (experiment builds only; timings, not results): TT_EXP_FWD
# in attention_sm100.cu drops one step (1 exponentials, 2 P store, 3 PV MMAs, 4 row max; 5 = the
# test_wait-first S wait). POLY: -DTT_EXP_FWD_POLY. AB_VARIANTS selects variants, AB_SHAPE the attn_bench args.
set -eu
cd paper_2602_00482_b200/csrc
make -j8 trace > /dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr"
mkdir -p ../../build/exp
OTHERS=$(ls ../../build/csrc_trace/*.o ../../build/csrc_trace/kernels/*.o | grep -v attention_sm100)
for v in ${AB_VARIANTS:-1 2 3 4}; do
  nvcc $FL -DTT_EXP_FWD=$v -c kernels/attention_sm100.cu -o ../../build/exp/fwd_$v.o
  nvcc $ARCH -shared -o ../../build/exp/libfwd_$v.so ../../build/exp/fwd_$v.o $OTHERS -ldl
done
cd ../..
SH=${AB_SHAPE:-16 32768 1024 14 64}
echo "== product"; python tools/attn_bench.py $SH | grep fwd
for v in ${AB_VARIANTS:-1 2 3 4}; do echo "== TT_EXP_FWD=$v"; ATTN_LIB=build/exp/libfwd_$v.so python tools/attn_bench.py $SH | grep fwd; done
