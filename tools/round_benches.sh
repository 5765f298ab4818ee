#!/bin/bash
# The secondary bench lines of a round (1 GPU): c1, c3, c4 (32 trees per GPU = the per-GPU share of
# 256 trees on 8 GPUs), the c5 prefix-share sweep and the partition ablation. Outputs gpurun_out/<tag>_*.
set -u
T=${1:-r2}
O=gpurun_out
mkdir -p $O
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 > $O/${T}_bench_c1.log 2>&1
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 > $O/${T}_bench_c3.log 2>&1
timeout 1800 python bench.py --config c4 --steps 2 --warmup 3 --no-flat --no-cpu > $O/${T}_bench_c4.log 2>&1
timeout 1800 python tools/sweep_c5.py --out $O/${T}_c5_sweep.json > $O/${T}_c5_sweep.log 2>&1
timeout 1200 python tools/partition_ablation.py --out $O/${T}_partition_ablation.json > $O/${T}_partition_ablation.log 2>&1
ls -la $O | grep ${T}_
