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
  const int4* qblocks = nullptr;
  int nqb = 0;
  float scale = 1.0f;
};

// One backward work item per (stack KV block, query range):
//   items[i]  = {kv_row0 (absolute stack row), kv_rows (<=64), q_lo, q_hi}
//   items2[i] = {seg_off, is_own}
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
  float* dq = nullptr;         // [n x lddq] fp32, accumulated
  long lddq = 0;
  float* dk = nullptr;  // fp32 dK/dV stack rows (absolute), accumulated
  float* dv = nullptr;
  long lddkv = 0;
  int n = 0, H = 0, dh = 0, S = 0;
  const int4* items = nullptr;
  const int2* items2 = nullptr;
  int nitems = 0;
  float scale = 1.0f;
};

void attn_fwd(const AttnFwdArgs& a, cudaStream_t stream);
void attn_bwd(const AttnBwdArgs& a, cudaStream_t stream);

}  // namespace ttb
