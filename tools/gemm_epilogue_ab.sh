#!/bin/bash
# A/B of the SiLU epilogue's cost components (experiment builds, never the product library): the
# MLP-in GEMM shape with the product epilogue, (ONESTORE) the silu(h) store dropped, (NOSTORE) both
# stores dropped (compute and staging kept), against the plain bf16-store GEMM of the same shape.
# Builds gemm_sm100.cu variants into build/exp/ and links them with the trace build's other objects.
# Usage (GPU box): bash tools/gemm_epilogue_ab.sh   (env: EPI_VARIANTS, AB_SHAPES, AB_PLAIN, GEMM_ITERS)
set -eu
cd paper_2602_00482_b200/csrc
make -j8 trace > /dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr"
mkdir -p ../../build/exp
OTHERS=$(ls ../../build/csrc_trace/*.o ../../build/csrc_trace/kernels/*.o | grep -v gemm_sm100)
for v in ${EPI_VARIANTS:-ONESTORE NOSTORE}; do
  if [ "$v" = HEAD ]; then  # tools/_ab/gemm_head.cu: an older gemm_sm100.cu (untracked) for a same-box A/B
    nvcc $FL -Ikernels -c ../../tools/_ab/gemm_head.cu -o ../../build/exp/gemm_$v.o
  elif [ "${v#EPI}" != "$v" ]; then  # EPI8 / EPI16: epilogue warps per CTA
    nvcc $FL -DTT_GEMM_EPI_WARPS=${v#EPI} -c kernels/gemm_sm100.cu -o ../../build/exp/gemm_$v.o
  else
    nvcc $FL -DTT_EXP_SILU_$v -c kernels/gemm_sm100.cu -o ../../build/exp/gemm_$v.o
  fi
  nvcc $ARCH -shared -o ../../build/exp/lib_$v.so ../../build/exp/gemm_$v.o $OTHERS -ldl
done
cd ../..
for lib in paper_2602_00482_b200/libtreetrain_b200.so $(for v in ${EPI_VARIANTS:-ONESTORE NOSTORE}; do echo build/exp/lib_$v.so; done); do
  echo "== $lib"
  GEMM_LIB=$lib GEMM_ONLY="${AB_SHAPES:-fwd mlp_in}" python tools/gemm_shapes.py
done
GEMM_ONLY="${AB_PLAIN:-fwd mlp_in plain}" python tools/gemm_shapes.py
