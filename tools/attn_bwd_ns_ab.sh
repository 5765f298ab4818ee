set -eu
cd paper_2602_00482_b200/csrc
make -j8 trace > /dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr"
mkdir -p ../../build/exp
OTHERS=$(ls ../../build/csrc_trace/*.o ../../build/csrc_trace/kernels/*.o | grep -v attention_bwd_sm100)
nvcc $FL -DTT_EXP_BWD_NS=2 -c kernels/attention_bwd_sm100.cu -o ../../build/exp/bwdns2.o
nvcc $ARCH -shared -o ../../build/exp/libbwdns2.so ../../build/exp/bwdns2.o $OTHERS -ldl
cd ../..
python tools/attn_bench.py 16 32768 1024 14 64 | grep bwd
ATTN_LIB=build/exp/libbwdns2.so python tools/attn_bench.py 16 32768 1024 14 64 | grep bwd
