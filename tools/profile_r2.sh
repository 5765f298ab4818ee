#!/bin/bash
# Profiling pass of round 2 (run on the GPU box under gpurun, one GPU):
#   1. launch list (device time of every launch, cold-cache + serialised) of the bench command;
#   2. ncu --set full of the attention kernels on the c2 leaf-batch shape (16 sibling segments of
#      2048 queries over a 1024-row prefix, 14 heads x 64; tools/attn_bench.py);
#   3. ncu --set full of every HBM-bound kernel of the step (RMSNorm fwd/bwd, dK/dV pack (stack pop),
#      embedding-grad scatter, CE, attention-bwd D pre-pass) at the c2 shape inside bench.py (one
#      prompt = one 32K-token leaf batch), 2 launches each after the first step.
# Summaries: profiles/summarize_launches.py, profiles/ncu_summary.py.
# Usage: tools/profile_r2.sh <tag> [what]   what: all | attn | hbm | launches   (outputs gpurun_out/<tag>_*)
set -u
T=${1:-r2}
W=${2:-all}
O=gpurun_out
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
if [ "$W" = all ] || [ "$W" = launches ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 4000 --csv \
  --log-file $O/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-flat --no-cpu --no-e2e \
  > $O/${T}_launches_bench.log 2>&1
fi
if [ "$W" = all ] || [ "$W" = attn ]; then
timeout 300 $NCU -k regex:fa_fwd -s 2 -c 1 -o $O/${T}_attn_fwd python tools/attn_bench.py 16 32768 1024 14 64 \
  > $O/${T}_ncu_attn.log 2>&1
timeout 300 $NCU -k regex:fa_bwd -s 2 -c 1 -o $O/${T}_attn_bwd python tools/attn_bench.py 16 32768 1024 14 64 \
  >> $O/${T}_ncu_attn.log 2>&1
# dh 128 (c3-like: 4 sibling segments of 2048 queries over a 2048-row prefix, 12 heads)
timeout 300 $NCU -k regex:fa_bwd -s 2 -c 1 -o $O/${T}_attn_bwd128 python tools/attn_bench.py 4 8192 2048 12 128 \
  >> $O/${T}_ncu_attn.log 2>&1
fi
if [ "$W" = all ] || [ "$W" = hbm ]; then
for k in rmsnorm_bwd rmsnorm_fwd pack_dqkv embed_grad ce_bf16_kernel attn_bwd_pre; do
  timeout 400 $NCU -k regex:$k -s 40 -c 1 -o $O/${T}_hbm_$k python bench.py --prompts 1 --steps 1 --warmup 1 \
    --no-flat --no-cpu --no-e2e >> $O/${T}_ncu_hbm.log 2>&1
done
fi
ls -la $O | grep ${T}_
