// Host interface of the sm_100a tcgen05 GEMM (gemm_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace ttb {

// A(m,k) / B(n,k) operand view. K-major: ptr[row*ld + k]; MN-major: ptr[k*ld + row].
struct GemmOperand {
  const __nv_bfloat16* ptr = nullptr;
  long ld = 0;
  bool mn_major = false;
};

enum EpiMode : int {
  EPI_STORE_BF16 = 0,  // out[blk] (bf16) = alpha*acc
  EPI_STORE_F32 = 1,   // out[blk] (fp32) = alpha*acc
  EPI_ADD_F32 = 2,     // out[blk] (fp32) += alpha*acc   (residual add / dW accumulate)
  EPI_SILU = 3,        // out[0] (bf16) = acc, out2 (bf16) = silu(acc)
  EPI_DSILU = 4,       // out[0] (bf16) = acc * silu'(aux)
  EPI_RESID_F32 = 5,   // out[0] (fp32) = resid + alpha*acc   (residual stream, model.hpp:427-428,447-448)
  EPI_STORE_F32_STATS = 6,  // out[0] (fp32) = alpha*acc, and out2 (float2, pitch ldo2) gets the per-row
                            // (max, sum exp(v - max)) of every 32-column group: the softmax statistics
                            // of LM-head logits, so the CE pass reads each logit row once
  EPI_ADD_F32_T = 7,   // out[0] (fp32) [n * ldo + m] += alpha*acc: the transposed accumulate that
                       // gemm_bf16 launches for EPI_ADD_F32 when C^T = B A^T tiles the SMs better
  EPI_STORE_BF16_STATS = 8,  // as EPI_STORE_F32_STATS, but out[0] (bf16) = alpha*acc - (its 32-column
                             // group's max): LM-head logits at 2 B each, exact to bf16 rounding of the
                             // offset from the group max (the entries near the max keep the most bits)
};

// Column blocks of width split_w go to out[n / split_w] (row pitch ldo[...]) so one GEMM can
// write e.g. q/k/v (or dWq/dWk/dWv) into three separate tensors. split_w = 0: single output.
struct EpiParams {
  int mode = EPI_STORE_BF16;
  int split_w = 0;
  void* out[3] = {nullptr, nullptr, nullptr};
  long ldo[3] = {0, 0, 0};
  void* out2 = nullptr;
  long ldo2 = 0;
  const __nv_bfloat16* aux = nullptr;
  long ld_aux = 0;
  const float* resid = nullptr;
  long ld_resid = 0;
  float alpha = 1.0f;
  int atomic = 0;
};

void gemm_bf16(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const EpiParams& epi, int splits,
               cudaStream_t stream);
int gemm_choose_splits(int M, int N, int K);
// EPI_ADD_F32 GEMMs (dW accumulates) run as C^T = B A^T when the wave model prefers that shape
bool gemm_prefer_transposed(int M, int N, int K);
void gemm_set_transpose(int mode);  // 0 never, 1 modelled (default), 2 always
int gemm_pick_bn(int N, bool b_mn_major);
int gemm_pick_bn2(int M, int N);
// 2-CTA (cta_group::2) tiles for M >= 256 (default 1: where the padding model allows); 0 forces the
// single-CTA kernel, 2 forces pair tiles (measurement only).
void gemm_set_2cta(int on);
// Programmatic dependent launch for every kernel (kernels/launch.cuh): 1 (default) launches with the
// PDL attribute, 0 in plain stream order (A/B measurement; engine option "pdl").
extern int g_pdl;
void set_pdl(int on);
// Debug / measurement only: force the 2-CTA tile width (128 or 256; 0 = the wave model's choice).
void gemm_force_bn2(int bn);
void gemm_force_bn1(int bn);  // single-CTA tile width (128 / 192 / 256; 0 = modelled)
// Per-device launch helpers (a process may drive engines on several GPUs; the current device is
// whatever the calling engine selected): one-time MaxDynamicSharedMemorySize per (kernel, device),
// the SM count of the current device, and a launch-status check that throws.
void ensure_smem_attr(const void* fn, int bytes);
int device_sm_count();
void check_launch(cudaError_t e, const char* what);

void make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer);
// fp32 [rows x width] (row pitch ld elements) in 32 x 32 boxes, SWIZZLE_128B: the staging layout of a
// warp that holds one 32-float row per lane (reduce-add / store epilogues)
void make_tmap_f32_sw128(CUtensorMap* map, const void* ptr, uint64_t width, uint64_t rows, uint64_t ld);
void make_tmap_f32_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                      uint32_t box_inner, uint32_t box_outer);

}  // namespace ttb
