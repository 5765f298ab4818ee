#!/bin/bash
# A/B of the attention backward kernels on the c2 leaf-batch shape (16 siblings x 2048 over a 1024 prefix)
export TT_ATTN_NSEG=16
B="python tools/attn_bench.py 1 1 32768 1024 14 64"
echo "== head"; TT_LIB_PATH=build_ab/lib_head.so $B 2>&1 | grep bwd
echo "== persistent kv2 ns4"; $B 2>&1 | grep bwd; TT_ATTN_BWD_PART=2 $B 2>&1 | grep bwd
echo "== persistent kv1 ns5"; TT_ATTN_DKV_KV1=1 $B 2>&1 | grep bwd; TT_ATTN_DKV_KV1=1 TT_ATTN_BWD_PART=2 $B 2>&1 | grep bwd
echo "== head again"; TT_LIB_PATH=build_ab/lib_head.so $B 2>&1 | grep bwd
