#!/bin/bash
# Profiling pass of one round (run on the GPU box under gpurun, one GPU):
#   1. launch list (device time of every launch, cold-cache + serialised) of the bench command;
#   2. one `ncu --set full` capture each of the dominant GEMM (LM head, c2 shape) and the two
#      attention kernels (c2-like segment: 8192 queries over a 1024-row prefix, 14 heads x 64).
# Summaries are then produced here with profiles/summarize_launches.py and profiles/ncu_summary.py.
# Usage: tools/profile_round.sh <tag>     (outputs gpurun_out/<tag>_*)
set -u
T=${1:-r1}
O=gpurun_out
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 4000 --csv \
  --log-file $O/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-flat --no-cpu --no-e2e \
  > $O/${T}_launches_bench.log 2>&1
GEMM_ONLY="fwd head" timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 \
  -o $O/${T}_gemm_head python tools/gemm_shapes.py > $O/${T}_ncu_gemm.log 2>&1
GEMM_ONLY="fwd mlp_in" timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 \
  -o $O/${T}_gemm_mlp_in python tools/gemm_shapes.py >> $O/${T}_ncu_gemm.log 2>&1
GEMM_ONLY="dW mlp_out" timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 \
  -o $O/${T}_gemm_dw_mlp_out python tools/gemm_shapes.py >> $O/${T}_ncu_gemm.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -s 2 -c 1 \
  -o $O/${T}_attn_fwd python tools/attn_bench.py 1 1 8192 1024 14 64 > $O/${T}_ncu_attn.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fa_bwd -s 4 -c 2 \
  -o $O/${T}_attn_bwd python tools/attn_bench.py 1 1 8192 1024 14 64 >> $O/${T}_ncu_attn.log 2>&1
ls -la $O | grep ${T}_
