// HBM-bound kernels of the push/pop path (elementwise.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

namespace ttb {

void k_embed_pe(const int32_t* tok, const int32_t* pos, const __nv_bfloat16* emb, const float* pe, float* x, int n,
                int d, cudaStream_t s);
void k_rmsnorm_fwd(const float* x, const float* gain, float* inv, __nv_bfloat16* y, int n, int d, cudaStream_t s);
// gx = gres + d(rmsnorm)/dx (gres may be null; gx may alias gres), bf16 copy into gxb, gain grad into ggain.
void k_rmsnorm_bwd(const float* gy, const float* x, const float* inv, const float* gain, const float* gres, float* gx,
                   __nv_bfloat16* gxb, float* ggain, int n, int d, cudaStream_t s);
// The same with a bf16 gy (the grad_normed GEMM outputs; 16 instead of 18 bytes per element), TMA-fed
// kernel only: d_model a multiple of 8 and <= 4096 (rmsnorm_bwd_bf16_gy_ok).
bool rmsnorm_bwd_bf16_gy_ok(int d);
void k_rmsnorm_bwd(const __nv_bfloat16* gy, const float* x, const float* inv, const float* gain, const float* gres,
                   float* gx, __nv_bfloat16* gxb, float* ggain, int n, int d, cudaStream_t s);
// stats: optional per-row (max, sum exp) of 32-column groups from the LM-head GEMM epilogue
// (EPI_STORE_F32_STATS, n_groups = ceil(V/32) per row); NULL = two passes over the logits row.
void k_ce(const float* logits, int m, long V, const int32_t* pair_off, const int32_t* tgt, const double* w,
          __nv_bfloat16* dl, double* loss, cudaStream_t s, const float2* stats = nullptr, int n_groups = 0);
// standalone weighted_nll: fp32 grad_logits, two passes over each logits row
// weighted_nll from bf16 logits relative to their 32-column group max + the per-group (max, sum) stats
// (the LM-head GEMM's EPI_STORE_BF16_STATS output); dlogits bf16.
void k_ce_bf16(const __nv_bfloat16* y, int m, long V, const int32_t* pair_off, const int32_t* tgt, const double* w,
               __nv_bfloat16* dl, double* loss, cudaStream_t s, const float2* stats, int n_groups);
void k_ce_f32(const float* logits, int m, long V, const int32_t* pair_off, const int32_t* tgt, const double* w,
              float* dl, double* loss, cudaStream_t s);
// dst[i] += src[i], n a multiple of 4
void k_add_f32(float* dst, const float* src, long n, cudaStream_t s);
void k_gather_rows_bf16(const __nv_bfloat16* src, const int32_t* idx, __nv_bfloat16* dst, int m, int d,
                        cudaStream_t s);
void k_scatter_rows_f32(const float* src, const int32_t* idx, float* dst, int m, int d, cudaStream_t s);
void k_pack_dqkv(const float* dq, float* dk, float* dv, __nv_bfloat16* out, int n, int d, cudaStream_t s);
// the k/v blocks only (dq already written as bf16 by the attention backward): out row pitch 3d
void k_pack_dkv(float* dk, float* dv, __nv_bfloat16* out, int n, int d, cudaStream_t s);
void k_embed_grad(const float* gx, const int32_t* tok, float* gemb, int n, int d, cudaStream_t s);
void k_f32_to_bf16_2d(const float* src, long lds, __nv_bfloat16* dst, long ldd, int rows, int cols, cudaStream_t s);
// transposed: dst[c * ldd + r] = bf16(src[r * lds + c])
void k_f32_to_bf16_2d_t(const float* src, long lds, __nv_bfloat16* dst, long ldd, int rows, int cols, cudaStream_t s);
void k_init_normal(float* out, long n, uint64_t seed, float stdv, cudaStream_t s);
void k_fill(float* out, long n, float v, cudaStream_t s);

}  // namespace ttb
