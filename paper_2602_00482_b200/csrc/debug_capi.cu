// Kernel-level debug entry points (device pointers in, device pointers out). Used only by the
// kernel unit tests in tests/test_kernels_gpu.py; the product entry points are in capi.cpp.
#include <cuda_runtime.h>

#include "capi_internal.h"
#include "kernels/gemm.h"

extern "C" {

// C = A * B^T with the operand majorness flags of ttb::GemmOperand; see gemm.h for modes.
int tt_debug_gemm(const void* a, long lda, int a_mn, const void* b, long ldb, int b_mn, int M, int N, int K, int mode,
                  void* out0, void* out1, void* out2, long ldo, int split_w, void* out_act, const void* aux,
                  int splits) {
  return ttb::guarded([&] {
    ttb::GemmOperand A{static_cast<const __nv_bfloat16*>(a), lda, a_mn != 0};
    ttb::GemmOperand B{static_cast<const __nv_bfloat16*>(b), ldb, b_mn != 0};
    ttb::EpiParams e;
    e.mode = mode;
    e.split_w = split_w;
    e.out[0] = out0;
    e.out[1] = out1;
    e.out[2] = out2;
    e.ldo[0] = e.ldo[1] = e.ldo[2] = ldo;
    e.out2 = out_act;
    e.ldo2 = ldo;
    e.aux = static_cast<const __nv_bfloat16*>(aux);
    e.ld_aux = ldo;
    ttb::gemm_bf16(A, B, M, N, K, e, splits, nullptr);
    ttb::check_cuda(cudaGetLastError(), "tt_debug_gemm launch");
    ttb::check_cuda(cudaDeviceSynchronize(), "tt_debug_gemm sync");
  });
}

}  // extern "C"
