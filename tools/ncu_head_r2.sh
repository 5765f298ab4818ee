#!/bin/bash
# ncu --set full of the c2 LM-head logits GEMM with the engine's bf16-logits + statistics epilogue
# (6656 x 151936 x 896, EPI_STORE_BF16_STATS): DRAM bytes per launch for bench.py's roofline.traffic.
mkdir -p gpurun_out
GEMM_ONLY="fwd head bf16 c2" timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 \
  -o gpurun_out/${TAG:-r2}_gemm_head_bf16 python tools/gemm_shapes.py > gpurun_out/${TAG:-r2}_ncu_head.log 2>&1
GEMM_ONLY="fwd head bf16 c2" python tools/gemm_shapes.py
