#!/bin/bash
# Attention kernel parity tests + timing sweep (run on the GPU box): tools/attn_sweep.sh <tag>
T=${1:-attn}
O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k attention -x > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
for P in ${POLYS:-0 1}; do for s in "2048 1024 14 64" "8192 1024 14 64" "2048 2048 12 128"; do
  TT_ATTN_POLY=$P timeout 120 python tools/attn_bench.py 1 1 $s | sed "s/^/poly=$P /"; done; done > $O/${T}_bench.log 2>&1
