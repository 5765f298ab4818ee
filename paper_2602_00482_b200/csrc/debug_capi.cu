// Kernel-level debug entry points (device pointers in, device pointers out). Used only by the
// kernel unit tests in tests/test_kernels_gpu.py; the product entry points are in capi.cpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "capi_internal.h"
#include "kernels/attention.h"
#include "kernels/elementwise.h"
#include "kernels/gemm.h"

extern "C" {

namespace {
int debug_gemm(bool sync, const void* a, long lda, int a_mn, const void* b, long ldb, int b_mn, int M, int N, int K,
               int mode, void* out0, void* out1, void* out2, long ldo, int split_w, void* out_act, const void* aux,
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
    e.ldo2 = (mode == ttb::EPI_STORE_F32_STATS || mode == ttb::EPI_STORE_BF16_STATS) ? (N + 31) / 32
                                                                                   : ldo;  // stats: float2 per 32-column group
    e.aux = static_cast<const __nv_bfloat16*>(aux);
    e.ld_aux = ldo;
    e.resid = static_cast<const float*>(aux);  // EPI_RESID_F32: aux is the fp32 residual input
    e.ld_resid = ldo;
    ttb::gemm_bf16(A, B, M, N, K, e, splits, nullptr);
    ttb::check_cuda(cudaGetLastError(), "tt_debug_gemm launch");
    if (sync) ttb::check_cuda(cudaDeviceSynchronize(), "tt_debug_gemm sync");
  });
}
}  // namespace

// C = A * B^T with the operand majorness flags of ttb::GemmOperand; see gemm.h for modes.
int tt_debug_gemm(const void* a, long lda, int a_mn, const void* b, long ldb, int b_mn, int M, int N, int K, int mode,
                  void* out0, void* out1, void* out2, long ldo, int split_w, void* out_act, const void* aux,
                  int splits) {
  return debug_gemm(true, a, lda, a_mn, b, ldb, b_mn, M, N, K, mode, out0, out1, out2, ldo, split_w, out_act, aux,
                    splits);
}
// Same without the device synchronisation (for timing loops).
int tt_debug_gemm_async(const void* a, long lda, int a_mn, const void* b, long ldb, int b_mn, int M, int N, int K,
                        int mode, void* out0, void* out1, void* out2, long ldo, int split_w, void* out_act,
                        const void* aux, int splits) {
  return debug_gemm(false, a, lda, a_mn, b, ldb, b_mn, M, N, K, mode, out0, out1, out2, ldo, split_w, out_act, aux,
                    splits);
}
int tt_debug_gemm_splits(int M, int N, int K) { return ttb::gemm_choose_splits(M, N, K); }

// rmsnorm_backward kernel (model.hpp:258-271) on device buffers; synchronises.
int tt_debug_rmsnorm_bwd(const float* gy, const float* x, const float* inv, const float* gain, const float* gres,
                         float* gx, void* gxb, float* ggain, int n, int d) {
  return ttb::guarded([&] {
    ttb::k_rmsnorm_bwd(gy, x, inv, gain, gres, gx, static_cast<__nv_bfloat16*>(gxb), ggain, n, d, nullptr);
    ttb::check_cuda(cudaGetLastError(), "tt_debug_rmsnorm_bwd launch");
    ttb::check_cuda(cudaDeviceSynchronize(), "tt_debug_rmsnorm_bwd sync");
  });
}
// The same with a bf16 gy (the engine's grad_normed path; d_model % 8 == 0, <= 4096).
int tt_debug_rmsnorm_bwd16(const void* gy, const float* x, const float* inv, const float* gain, const float* gres,
                           float* gx, void* gxb, float* ggain, int n, int d) {
  return ttb::guarded([&] {
    ttb::k_rmsnorm_bwd(static_cast<const __nv_bfloat16*>(gy), x, inv, gain, gres, gx, static_cast<__nv_bfloat16*>(gxb),
                       ggain, n, d, nullptr);
    ttb::check_cuda(cudaGetLastError(), "tt_debug_rmsnorm_bwd16 launch");
    ttb::check_cuda(cudaDeviceSynchronize(), "tt_debug_rmsnorm_bwd16 sync");
  });
}
void tt_debug_gemm_set_2cta(int on) { ttb::gemm_set_2cta(on); }
void tt_debug_gemm_set_transpose(int mode) { ttb::gemm_set_transpose(mode); }
void tt_debug_gemm_force_bn2(int bn) { ttb::gemm_force_bn2(bn); }
void tt_debug_gemm_force_bn1(int bn) { ttb::gemm_force_bn1(bn); }

static int g_attn_nseg = 1;
// Timing tools: the n queries of tt_debug_attn form nseg equal sibling segments over the shared prefix
// (the c2 leaf-batch shape), with the engine's work-item chunking.
void tt_debug_attn_set_segments(int nseg) { g_attn_nseg = nseg < 1 ? 1 : nseg; }

// Segment attention on one segment of n queries over stack rows [0, S) + own rows [S, S+n)
// (k/v: [rows_cap x H*dh] bf16), tcgen05 kernels (impl must be 1). dir 0: forward -> o, lse.
// dir 1: backward from o, lse, dO -> dq (fp32, overwritten), dk/dv (added).
// iters > 0: additionally time `iters` back-to-back launches with CUDA events -> *ms_out (per launch).
int tt_debug_attn(int impl, int dir, const void* q, const void* k, const void* v, void* o, float* lse, const void* dO,
                  float* D, float* dq, float* dk, float* dv, int n, int S, int H, int dh, long rows_cap, int iters,
                  float* ms_out) {
  return ttb::guarded([&] {
    cudaEvent_t e0, e1;
    ttb::check_cuda(cudaEventCreate(&e0), "event");
    ttb::check_cuda(cudaEventCreate(&e1), "event");
    auto timed = [&](auto&& launch) {
      launch();
      if (iters > 0 && ms_out) {
        ttb::check_cuda(cudaDeviceSynchronize(), "sync");
        cudaEventRecord(e0, nullptr);
        for (int i = 0; i < iters; ++i) launch();
        cudaEventRecord(e1, nullptr);
        ttb::check_cuda(cudaEventSynchronize(e1), "sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        *ms_out = ms / iters;
      }
    };
    const int d = H * dh;
    if (impl != 1) throw std::invalid_argument("tt_debug_attn: only the tcgen05 kernels (impl 1) exist");
    const int nseg = g_attn_nseg;
    const int seg = (n + nseg - 1) / nseg;
    std::vector<int> q128;
    for (int so = 0; so < n; so += seg)
      for (int qs = so; qs < std::min(n, so + seg); qs += 128)
        q128.insert(q128.end(), {qs, std::min({qs + 128, so + seg, n}), so, 0});
    auto up = [](const std::vector<int>& h) {
      void* p = nullptr;
      ttb::check_cuda(cudaMalloc(&p, std::max<size_t>(16, h.size() * 4)), "cudaMalloc");
      if (!h.empty()) ttb::check_cuda(cudaMemcpy(p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "memcpy");
      return p;
    };
    void* d128 = up(q128);
    const float scale = 1.0f / std::sqrt(static_cast<float>(dh));
    if (dir == 0) {
      ttb::AttnFwdArgs a;
      a.q = static_cast<const __nv_bfloat16*>(q);
      a.ldq = d;
      a.k = static_cast<const __nv_bfloat16*>(k);
      a.v = static_cast<const __nv_bfloat16*>(v);
      a.ldkv = d;
      a.o = static_cast<__nv_bfloat16*>(o);
      a.ldo = d;
      a.lse = lse;
      a.n = n;
      a.H = H;
      a.dh = dh;
      a.S = S;
      a.scale = scale;
      a.qblocks = static_cast<const int4*>(d128);
      a.nqb = static_cast<int>(q128.size() / 4);
      timed([&] { ttb::attn_fwd_sm100(a, rows_cap, nullptr); });
    } else {
      ttb::AttnBwdArgs a;
      a.q = static_cast<const __nv_bfloat16*>(q);
      a.dO = static_cast<const __nv_bfloat16*>(dO);
      a.o = static_cast<const __nv_bfloat16*>(o);
      a.ldq = d;
      a.k = static_cast<const __nv_bfloat16*>(k);
      a.v = static_cast<const __nv_bfloat16*>(v);
      a.ldkv = d;
      a.lse = lse;
      a.D = D;
      a.dq = dq;
      a.lddq = d;
      a.dk = dk;
      a.dv = dv;
      a.lddkv = d;
      a.n = n;
      a.H = H;
      a.dh = dh;
      a.S = S;
      a.scale = scale;
      {
        std::vector<int> k128, k128b;
        const int chunk_pre = nseg > 1 ? 4096 : n, chunk_own = nseg > 1 ? 2048 : n;  // engine.cpp kQChunk*
        for (int kv = 0; kv < S; kv += 128)
          for (int q0 = 0; q0 < n; q0 += chunk_pre) {
            k128.insert(k128.end(), {kv, std::min(128, S - kv), q0, std::min(n, q0 + chunk_pre)});
            k128b.insert(k128b.end(), {0, 0});
          }
        for (int so = 0; so < n; so += seg) {
          const int end = std::min(n, so + seg);
          for (int kt = 0; kt < end - so; kt += 128)
            for (int q0 = so + kt; q0 < end; q0 += chunk_own) {
              k128.insert(k128.end(), {S + so + kt, std::min(128, end - so - kt), q0, std::min(end, q0 + chunk_own)});
              k128b.insert(k128b.end(), {so, 1});
            }
        }
        {  // longest first, as build_meta orders them
          const size_t ni = k128.size() / 4;
          std::vector<int> order(ni), a4(ni * 4), a2(ni * 2);
          for (size_t i = 0; i < ni; ++i) order[i] = static_cast<int>(i);
          std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
            return k128[4 * x + 3] - k128[4 * x + 2] > k128[4 * y + 3] - k128[4 * y + 2];
          });
          for (size_t i = 0; i < ni; ++i) {
            for (int j = 0; j < 4; ++j) a4[4 * i + j] = k128[4 * order[i] + j];
            for (int j = 0; j < 2; ++j) a2[2 * i + j] = k128b[2 * order[i] + j];
          }
          k128.swap(a4);
          k128b.swap(a2);
        }
        void *dk128 = up(k128), *dk128b = up(k128b);
        timed([&] {
          ttb::attn_bwd_sm100(a, rows_cap, static_cast<const int4*>(dk128), static_cast<const int2*>(dk128b),
                              static_cast<int>(k128.size() / 4), nullptr);
        });
        ttb::check_cuda(cudaDeviceSynchronize(), "tt_debug_attn sync");
        cudaFree(dk128);
        cudaFree(dk128b);
      }
    }
    ttb::check_cuda(cudaGetLastError(), "tt_debug_attn launch");
    ttb::check_cuda(cudaDeviceSynchronize(), "tt_debug_attn sync");
    cudaFree(d128);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

}  // extern "C"
