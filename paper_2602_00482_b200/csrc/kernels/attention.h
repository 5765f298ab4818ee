// Segment attention over the device KV stack (attention.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace ttb {

// One forward work item per query block: {q_start, q_end, seg_off, 0}, batch-local rows.
struct AttnFwdArgs {
  const __nv_bfloat16* q = nullptr;  // [n x ldq] batch rows, heads packed
  long ldq = 0;
  const __nv_bfloat16* k = nullptr;  // stack rows (absolute), this layer
  const __nv_bfloat16* v = nullptr;
  long ldkv = 0;
  __nv_bfloat16* o = nullptr;  // [n x ldo]
  long ldo = 0;
  float* lse = nullptr;  // [H x n], natural log
  int n = 0, H = 0, dh = 0, S = 0;
  // stack rows: the prefix is rows [pbase, pbase + S), the batch's own rows start at r0 (< 0: r0 = S)
  int pbase = 0, r0 = -1;
  const int4* qblocks = nullptr;
  int nqb = 0;
  float scale = 1.0f;
};

// Backward arguments (the work lists are passed to attn_bwd_sm100 separately).
struct AttnBwdArgs {
  const __nv_bfloat16* q = nullptr;
  const __nv_bfloat16* dO = nullptr;  // same pitch as q
  const __nv_bfloat16* o = nullptr;   // forward output, same pitch as q
  long ldq = 0;
  const __nv_bfloat16* k = nullptr;
  const __nv_bfloat16* v = nullptr;
  long ldkv = 0;
  const float* lse = nullptr;  // [H x n]
  float* D = nullptr;          // [H x n] scratch: rowsum(dO * O)
  float* dq = nullptr;         // [n x lddq] fp32, overwritten (zeroed by the D pre-pass, then reduced into)
  long lddq = 0;
  float* dk = nullptr;  // fp32 dK/dV stack rows (absolute), accumulated
  float* dv = nullptr;
  long lddkv = 0;
  // prefix-row (grad_prefix) destination, absolute rows with pitch lddkv; nullptr = dk / dv
  float* dk_pre = nullptr;
  float* dv_pre = nullptr;
  // items flagged 2 (own rows with a single writer): scaled dK as bf16 into dkv16 [batch row x
  // lddkv16] at column h * dh, dV at column H * dh + h * dh (the dk / dv blocks of the packed operand)
  __nv_bfloat16* dkv16 = nullptr;
  long lddkv16 = 0;
  int n = 0, H = 0, dh = 0, S = 0;
  int pbase = 0, r0 = -1;  // as in AttnFwdArgs (the dK/dV items carry absolute rows already)
  float scale = 1.0f;
};


// tcgen05/TMEM/TMA forward (attention_sm100.cu): qblocks hold 128-row query blocks; k/v are the
// layer's stack base pointers with rows_cap rows.
constexpr int kFwdBlockQ = 128;
void attn_fwd_sm100(const AttnFwdArgs& a, long rows_cap, cudaStream_t stream);



// D = rowsum(dO * O) per (head, row) (the softmax-backward correction term).
void attn_bwd_pre(const AttnBwdArgs& a, cudaStream_t stream);
// tcgen05 backward (attention_bwd_sm100.cu, one fused kernel per head size): kv_items/kv_items2 are
// 128-row stack blocks {kv_row0, kv_rows, q_lo, q_hi} / {seg_off, 0 prefix | 1 own | 2 own, single
// writer}. dk/dv are accumulated (red.add) into the fp32 stack rows (prefix rows into dk_pre/dv_pre
// when set; flag-2 rows as bf16 into dkv16). dQ (scaled) is ADDED into the fp32 accumulator dq.
constexpr int kBwdBlockKV = 128;
void attn_bwd_sm100(const AttnBwdArgs& a, long rows_cap, const int4* kv_items, const int2* kv_items2, int n_kv,
                    cudaStream_t stream);

}  // namespace ttb
