// tcgen05 / TMEM / TMA segment attention backward over the device KV stack (sm_100a).
//
// Replaces the attention backward of backward_segment (model.hpp:546-604):
//   P = softmax(scale Q K^T) (recomputed from the forward LSE), dP = dO V^T,
//   dS = P * (dP - D) with D = rowsum(dO * O),  dQ = scale dS K,  dK = scale dS^T Q,  dV = P^T dO.
// Two kernels, both tensor-core only (no atomics on the hot product):
//   dq kernel   : CTA = (128-query block, head); loops over the block's KV blocks (BKV = 64).
//                 S, dP double-buffered in TMEM; dS -> swizzled smem; dQ accumulated in TMEM and
//                 written once (fp32) — the CTA owns its query rows.
//   dkdv kernel : CTA = (128-key stack block, head, query range); loops over 64-query blocks.
//                 S^T, dP^T double-buffered in TMEM; P^T, dS^T -> swizzled smem; dK, dV accumulated
//                 in TMEM, added once into the fp32 dK/dV stack rows (red.add.v4: several query-range
//                 items and several sibling segments contribute to the same prefix rows).
// Roles (192 threads): warp 0 TMA producer, warp 1 TMEM alloc + MMA issuer, warps 2..5 one
// TMEM lane (= query row / key row) per thread.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <stdexcept>

#include "attention.h"
#include "gemm.h"
#include "sm100.cuh"

namespace ttb {

namespace {

constexpr int kThreads = 320;   // warp 0 TMA, warp 1 MMA, warps 2..9: 2 per TMEM lane quadrant
constexpr int kSmxWarps = 8;   // softmax-gradient warps; the pair on a quadrant splits the columns
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// Writes 32 bf16 values (w[16] packed pairs) = chunks [4*half, 4*half+4) of a thread's 128B row.
__device__ __forceinline__ void st_halfrow_sw128(uint8_t* panel, int row, int half, const uint32_t (&w)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int ch = half * 4 + c;
    uint4* dst = reinterpret_cast<uint4*>(panel + row * 128 + ((ch ^ (row & 7)) * 16));
    *dst = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
  }
}

// ================================================================================= dQ kernel
template <int DH, int NS>
struct DqCfg {
  static constexpr int BQ = 128, BKV = 64;
  static constexpr int NB = 3;  // S/dP TMEM buffers: the MMA warp runs NB-1 blocks ahead of softmax
  static constexpr int kQBytes = BQ * DH * 2;
  static constexpr int kKVBytes = BKV * DH * 2;
  static constexpr int kDSBytes = BQ * BKV * 2;
  static constexpr int kOffDO = kQBytes;
  static constexpr int kOffK = 2 * kQBytes;
  static constexpr int kOffV = kOffK + NS * kKVBytes;
  static constexpr int kOffBar = kOffV + NS * kKVBytes;  // (dS lives in TMEM)
  static constexpr int kTmemCols = (2 * NB * BKV + DH) <= 256 ? 256 : 512;
  static_assert(2 * NB * BKV + DH <= 512 && NS >= NB, "dq kernel: TMEM / K-V ring too small");
  // a second co-resident CTA could not get TMEM (it would block in tcgen05.alloc while holding the
  // SM's warp slots): size smem so that exactly one CTA fits when all 512 columns are needed
  static constexpr int kSmemUsed = kOffBar + 256 + 1024;
  static constexpr int kSmem = (kTmemCols == 512 && kSmemUsed < 118 * 1024) ? 118 * 1024 : kSmemUsed;
  static constexpr uint32_t kIdescS = make_idesc_bf16(128, BKV, false, false);
  static constexpr uint32_t kIdescQ = make_idesc_bf16(128, DH, false, true);
};

struct BwdParams {
  const float* lse;  // [H x n]
  const float* D;    // [H x n]
  float* dq;         // [n x lddq]
  long lddq;
  __nv_bfloat16* dq16;  // if set: bf16 dQ [n x lddq16] instead of dq
  long lddq16;
  float* dk;  // stack rows (this layer), fp32
  float* dv;
  long lddkv;
  int n, S, H;
  int pbase, r0;        // prefix rows [pbase, pbase + S); own rows from r0
  const int4* blocks;   // dq: {q_start, q_end, seg_off, 0}; dkdv: {kv_row0, kv_rows, q_lo, q_hi}
  const int2* blocks2;  // dkdv: {seg_off, is_own}
  float scale, scale_log2;
};

// DBG (timing experiments only, TT_ATTN_DBG): 1 = softmax warps skip TMEM loads + math (MMA/TMA
// pipeline alone), 2 = softmax warps do not wait for S (softmax alone), 4 = + clock64 trace of one
// mid-grid CTA into g_attn_trace (tt_debug_attn_trace). TT_ATTN_DBG=3 -> trace, 5 -> skip + trace.
__device__ long long g_attn_trace[6][256];
// Two MMA-issuing warps: warp 1 issues S_j / dP_j, warp 10 issues dQ += dS_j K_j. An mbarrier wait in
// an issuing thread costs ~180 clk while MMAs are in flight (tools/umma_probe.cu, mode 8), longer than
// the tensor pipe takes for the 4-8 N=64 MMAs queued behind it; with one issuer per dependency chain
// a wait on one chain never starves the pipe of the other chain's MMAs.
constexpr int kThreadsDq = kThreads + 32;
template <int DH, int NS, int POLY, int DBG = 0>
__global__ void __launch_bounds__(kThreadsDq, 1)
    fa_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                     const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                     BwdParams p) {
  using C = DqCfg<DH, NS>;
  constexpr int BKV = C::BKV;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + NS;
  uint64_t* s_full = kv_empty + NS;    // [NB] S_j and dP_j in TMEM
  uint64_t* ds_full = s_full + C::NB;  // [NB] softmax done with block j: S/dP_j read, dS_j in smem
  // kv_empty[j % NS] completes when dQ_j (the last reader of K_j and of dS_j) is done: it frees the
  // K/V stage for the producer AND the dS buffer for the softmax warps (one commit, two waiters)
  uint64_t* dq_done = ds_full + C::NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 1);

  const int warp = warp_id_sync();
  const int lane = threadIdx.x & 31;
  const int4 blk = p.blocks[blockIdx.x];
  const int q_start = blk.x, q_end = blk.y, seg_off = blk.z;
  const int h = blockIdx.y;
  const int S = p.S;
  const int n_pre = (S + BKV - 1) / BKV;
  const int own_rows = q_end - seg_off;
  const int nblk = n_pre + (own_rows + BKV - 1) / BKV;
  auto kv_row0 = [&](int j) { return j < n_pre ? p.pbase + j * BKV : p.r0 + seg_off + (j - n_pre) * BKV; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < C::NB; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&ds_full[s], kSmxWarps);
    }
    mbar_init(dq_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: S[NB] at [0, NB*BKV), dP[NB] at [NB*BKV, 2*NB*BKV), dQ at [2*NB*BKV, +DH)
  constexpr int NB = C::NB;
  const uint32_t t_S = tmem, t_dP = tmem + NB * BKV, t_dQ = tmem + 2 * NB * BKV;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * C::kQBytes);
#pragma unroll
      for (int pn = 0; pn < DH / 64; ++pn) {
        tma_load_2d(&tm_q, q_full, smem + pn * (128 * 128), h * DH + pn * 64, q_start);
        tma_load_2d(&tm_do, q_full, smem + C::kOffDO + pn * (128 * 128), h * DH + pn * 64, q_start);
      }
      for (int j = 0; j < nblk; ++j) {
        const int st = j % NS;
        mbar_wait(&kv_empty[st], ((j / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * C::kKVBytes);
        const int r0 = kv_row0(j);
#pragma unroll
        for (int pn = 0; pn < DH / 64; ++pn) {
          tma_load_2d(&tm_k, &kv_full[st], smem + C::kOffK + st * C::kKVBytes + pn * (BKV * 128), h * DH + pn * 64, r0);
          tma_load_2d(&tm_v, &kv_full[st], smem + C::kOffV + st * C::kKVBytes + pn * (BKV * 128), h * DH + pn * 64, r0);
        }
      }
    }
  } else if (warp == 1) {
    // S_j = Q K_j^T ; dP_j = dO V_j^T into TMEM buffer j % NB, once the softmax is done with j - NB
    const uint64_t d16 = make_sdesc_sw128(smem_u32(smem), 16, 1024);  // K-major tiles
    const bool trace = (DBG & 4) && lane == 0 && blockIdx.x == gridDim.x / 2 && blockIdx.y == 0;
    mbar_wait(q_full, 0);
    for (int j = 0; j < nblk; ++j) {
      const int st = j % NS;
      // buffer j % NB holds dS_{j-NB} (the A operand of dQ_{j-NB}) until that MMA completes
      if (j >= NB) mbar_wait(&kv_empty[(j - NB) % NS], ((j - NB) / NS) & 1);
      if (trace && j < 256) g_attn_trace[4][j] = clock64();
      mbar_wait(&kv_full[st], (j / NS) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t k_off = C::kOffK + st * C::kKVBytes, v_off = C::kOffV + st * C::kKVBytes;
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint32_t ao = (k / 4) * (128 * 128) + (k % 4) * 32, bo = (k / 4) * (BKV * 128) + (k % 4) * 32;
          umma_bf16_ss(t_S + (j % NB) * BKV, sdesc_add(d16, ao), sdesc_add(sdesc_add(d16, k_off), bo), C::kIdescS,
                       k > 0);
          umma_bf16_ss(t_dP + (j % NB) * BKV, sdesc_add(d16, C::kOffDO + ao), sdesc_add(sdesc_add(d16, v_off), bo),
                       C::kIdescS, k > 0);
        }
        umma_commit(&s_full[j % NB]);
      }
      __syncwarp();
      if (trace && j < 256) g_attn_trace[5][j] = clock64();
    }
  } else if (warp == 10) {
    // dQ += dS_j K_j (B = K_j read MN-major: N = dh, K = keys), in block order
    const uint64_t dKmn = make_sdesc_sw128(smem_u32(smem), BKV * 128, 1024);
    const bool trace = (DBG & 4) && lane == 0 && blockIdx.x == gridDim.x / 2 && blockIdx.y == 0;
    for (int j = 0; j < nblk; ++j) {
      mbar_wait(&ds_full[j % NB], (j / NB) & 1);
      if (trace && j < 256) g_attn_trace[0][j] = clock64();
      tc_fence_after();
      if (lane == 0) {
        const int st = j % NS;
        const uint32_t k_off = C::kOffK + st * C::kKVBytes;
        // A = dS_j straight from TMEM (bf16 pairs in the S_j buffer, per half of the keys)
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k)
          umma_bf16_ts(t_dQ, t_S + (j % NB) * BKV + packed_col<BKV / 2>(k), sdesc_add(sdesc_add(dKmn, k_off), k * 2048), C::kIdescQ,
                       (j > 0 || k > 0));
        umma_commit(&kv_empty[st]);
        if (j == nblk - 1) umma_commit(dq_done);
      }
      __syncwarp();
      if (trace && j < 256) g_attn_trace[1][j] = clock64();
    }
  } else {
    const int quad = warp & 3;
    const int half = (warp - 2) / 4;  // key columns [32*half, 32*half+32) of each 64-key block
    const int rloc = quad * 32 + lane;
    const int row = q_start + rloc;
    const int t = row - seg_off;
    const bool row_ok = row < q_end;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    // invalid rows: lse2 = +inf -> P = 0 (their dQ rows are never stored)
    const float lse2 = row_ok ? p.lse[static_cast<long>(h) * p.n + row] * kLog2e : INFINITY;
    const float Dr = row_ok ? p.D[static_cast<long>(h) * p.n + row] : 0.f;
    const float c2 = p.scale_log2;
    constexpr int HC = BKV / 2;
    const bool trace = (DBG & 4) && threadIdx.x == 64 && blockIdx.x == gridDim.x / 2 && blockIdx.y == 0;
    for (int j = 0; j < nblk; ++j) {
      if (DBG != 2) mbar_wait(&s_full[j % NB], (j / NB) & 1);
      if (trace && j < 256) g_attn_trace[2][j] = clock64();
      tc_fence_after();
      if ((DBG & 1)) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ds_full[j % NB]);
        continue;
      }
      float s[HC], dp[HC];
#pragma unroll
      for (int c = 0; c < HC; c += 16) {
        uint32_t r[16], r2[16];
        tmem_ld16(t_S + (j % NB) * BKV + half * HC + c + lane_off, r);
        tmem_ld16(t_dP + (j % NB) * BKV + half * HC + c + lane_off, r2);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          s[c + i] = __uint_as_float(r[i]);
          dp[c + i] = __uint_as_float(r2[i]);
        }
      }
      tmem_ld_wait();
      const bool pre = j < n_pre;
      const int base = (pre ? j * BKV : (j - n_pre) * BKV) + half * HC;
      const int lim = pre ? (S - base) : (t - base + 1);  // valid key columns [0, lim) of this half
      if (__any_sync(0xffffffff, lim < HC)) {
#pragma unroll
        for (int i = 0; i < HC; ++i) s[i] = i < lim ? s[i] : -INFINITY;
      }
      uint32_t w[HC / 2];
      const float2 c22 = make_float2(c2, c2), nl2 = make_float2(-lse2, -lse2), nD2 = make_float2(-Dr, -Dr);
#pragma unroll
      for (int i = 0; i < HC; i += 2) {
        const float2 x = __ffma2_rn(make_float2(s[i], s[i + 1]), c22, nl2);
        const float2 pe = ((i / 2) & 3) < POLY ? ex2_poly2(x) : make_float2(ex2_approx(x.x), ex2_approx(x.y));
        const float2 ds = __fmul2_rn(pe, __fadd2_rn(make_float2(dp[i], dp[i + 1]), nD2));
        w[i / 2] = pack_bf16x2(ds.x, ds.y);
      }
      // dS_j (bf16 pairs) into the first HC/2 columns of this half's OWN S_j columns (the other half
      // may still be reading its S columns): the A operand of dQ_j
      tmem_st16(t_S + (j % NB) * BKV + half * HC + lane_off, w);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ds_full[j % NB]);
      if (trace && j < 256) g_attn_trace[3][j] = clock64();
    }
    mbar_wait(dq_done, 0);
    tc_fence_after();
#pragma unroll
    for (int c = half * (DH / 2); c < (half + 1) * (DH / 2); c += 16) {
      uint32_t r[16];
      tmem_ld16(t_dQ + c + lane_off, r);
      tmem_ld_wait();
      if (row_ok && p.dq16) {
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          w[i] = pack_bf16x2(__uint_as_float(r[2 * i]) * p.scale, __uint_as_float(r[2 * i + 1]) * p.scale);
        uint4* dst = reinterpret_cast<uint4*>(p.dq16 + static_cast<long>(row) * p.lddq16 + h * DH + c);
        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
        dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
      } else if (row_ok) {
        float4* dst = reinterpret_cast<float4*>(p.dq + static_cast<long>(row) * p.lddq + h * DH + c);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_float4(__uint_as_float(r[4 * i]) * p.scale, __uint_as_float(r[4 * i + 1]) * p.scale,
                               __uint_as_float(r[4 * i + 2]) * p.scale, __uint_as_float(r[4 * i + 3]) * p.scale);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::kTmemCols);
}

// ================================================================================= dK/dV kernel
template <int DH, int NS>
struct DkvCfg {
  static constexpr int BKV = 128, BQ = 64;
  static constexpr int NB = DH == 64 ? 3 : 2;  // S^T/dP^T TMEM buffers (TMEM: 2*NB*BQ + 2*DH <= 512)
  static constexpr int kKVBytes = BKV * DH * 2;   // K (or V) block, loaded once
  static constexpr int kQBytes = BQ * DH * 2;     // Q_i (or dO_i) tile
  static constexpr int kPBytes = BKV * BQ * 2;    // P^T (or dS^T) tile
  static constexpr int kOffV = kKVBytes;
  static constexpr int kOffQ = 2 * kKVBytes;
  static constexpr int kOffDO = kOffQ + NS * kQBytes;
  static constexpr int kOffStat = kOffDO + NS * kQBytes;  // [2][2][BQ] floats: lse2, D (P^T, dS^T in TMEM)
  static constexpr int kOffBar = kOffStat + 2 * 2 * BQ * 4;
  static constexpr int kSmem = kOffBar + 256 + 1024;
  static constexpr int kTmemCols = 512;
  static_assert(2 * NB * BQ + 2 * DH <= 512 && NS >= NB, "dkdv kernel: TMEM / Q ring too small");
  static constexpr uint32_t kIdescS = make_idesc_bf16(128, BQ, false, false);
  static constexpr uint32_t kIdescKV = make_idesc_bf16(128, DH, false, true);
};

// Like the dq kernel: two MMA-issuing warps (warp 1: S^T_i / dP^T_i; warp 10: dV / dK), and P^T_i /
// dS^T_i go back into TMEM (bf16 pairs over the S^T_i / dP^T_i buffers) as the A operands of dV / dK.
template <int DH, int NS, int POLY>
__global__ void __launch_bounds__(kThreadsDq, 1)
    fa_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                       BwdParams p) {
  using C = DkvCfg<DH, NS>;
  constexpr int BQ = C::BQ;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;
  uint64_t* q_empty = q_full + NS;
  uint64_t* s_full = q_empty + NS;    // [NB]
  uint64_t* p_full = s_full + C::NB;  // [NB] softmax done with block i (P^T / dS^T in TMEM)
  // q_empty[i % NS] completes when dV/dK_i are done: frees the Q/dO stage AND the TMEM buffers of i
  uint64_t* acc_done = p_full + C::NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);
  float* stat = reinterpret_cast<float*>(smem + C::kOffStat);

  const int warp = warp_id_sync();
  const int lane = threadIdx.x & 31;
  const int4 it = p.blocks[blockIdx.x];
  const int2 it2 = p.blocks2[blockIdx.x];
  const int kv0 = it.x, kv_rows = it.y, q_lo = it.z, q_hi = it.w;
  const int seg_off = it2.x;
  const bool own = it2.y != 0;
  const int kt_base = own ? kv0 - p.r0 - seg_off : 0;
  const int h = blockIdx.y;
  const int nq = (q_hi - q_lo + BQ - 1) / BQ;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_init(kv_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < C::NB; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], kSmxWarps);
    }
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: S^T[NB] at [0, NB*BQ), dP^T[NB] at [NB*BQ, 2*NB*BQ), then dK and dV (DH each)
  constexpr int NB = C::NB;
  const uint32_t t_S = tmem, t_dP = tmem + NB * BQ, t_dK = tmem + 2 * NB * BQ, t_dV = t_dK + DH;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * C::kKVBytes);
#pragma unroll
      for (int pn = 0; pn < DH / 64; ++pn) {
        tma_load_2d(&tm_k, kv_full, smem + pn * (128 * 128), h * DH + pn * 64, kv0);
        tma_load_2d(&tm_v, kv_full, smem + C::kOffV + pn * (128 * 128), h * DH + pn * 64, kv0);
      }
      for (int i = 0; i < nq; ++i) {
        const int st = i % NS;
        mbar_wait(&q_empty[st], ((i / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[st], 2 * C::kQBytes);
        const int q0 = q_lo + i * BQ;
#pragma unroll
        for (int pn = 0; pn < DH / 64; ++pn) {
          tma_load_2d(&tm_q, &q_full[st], smem + C::kOffQ + st * C::kQBytes + pn * (BQ * 128), h * DH + pn * 64, q0);
          tma_load_2d(&tm_do, &q_full[st], smem + C::kOffDO + st * C::kQBytes + pn * (BQ * 128), h * DH + pn * 64, q0);
        }
      }
    }
  } else if (warp == 1) {
    // S^T_i = K Q_i^T ; dP^T_i = V dO_i^T   (M = 128 keys, N = 64 queries) into TMEM buffer i % NB,
    // once dV/dK_{i-NB} (whose A operands P^T / dS^T live in that buffer) are done
    const uint64_t d16 = make_sdesc_sw128(smem_u32(smem), 16, 1024);  // K-major tiles
    mbar_wait(kv_full, 0);
    for (int i = 0; i < nq; ++i) {
      const int st = i % NS;
      if (i >= NB) mbar_wait(&q_empty[(i - NB) % NS], ((i - NB) / NS) & 1);
      mbar_wait(&q_full[st], (i / NS) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t q_off = C::kOffQ + st * C::kQBytes, do_off = C::kOffDO + st * C::kQBytes;
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint32_t ao = (k / 4) * (128 * 128) + (k % 4) * 32, bo = (k / 4) * (BQ * 128) + (k % 4) * 32;
          umma_bf16_ss(t_S + (i % NB) * BQ, sdesc_add(d16, ao), sdesc_add(sdesc_add(d16, q_off), bo), C::kIdescS,
                       k > 0);
          umma_bf16_ss(t_dP + (i % NB) * BQ, sdesc_add(d16, C::kOffV + ao), sdesc_add(sdesc_add(d16, do_off), bo),
                       C::kIdescS, k > 0);
        }
        umma_commit(&s_full[i % NB]);
      }
      __syncwarp();
    }
  } else if (warp == 10) {
    // dV += P^T dO_i ; dK += dS^T Q_i   (A from TMEM; B read MN-major: N = dh, K = queries)
    const uint64_t dmn = make_sdesc_sw128(smem_u32(smem), BQ * 128, 1024);  // Q_i / dO_i read MN-major
    for (int i = 0; i < nq; ++i) {
      mbar_wait(&p_full[i % NB], (i / NB) & 1);
      tc_fence_after();
      if (lane == 0) {
        const int st = i % NS;
        const uint32_t q_off = C::kOffQ + st * C::kQBytes, do_off = C::kOffDO + st * C::kQBytes;
#pragma unroll
        for (int k = 0; k < BQ / 16; ++k) {
          umma_bf16_ts(t_dV, t_S + (i % NB) * BQ + packed_col<BQ / 2>(k), sdesc_add(sdesc_add(dmn, do_off), k * 2048), C::kIdescKV,
                       (i > 0 || k > 0));
          umma_bf16_ts(t_dK, t_dP + (i % NB) * BQ + packed_col<BQ / 2>(k), sdesc_add(sdesc_add(dmn, q_off), k * 2048), C::kIdescKV,
                       (i > 0 || k > 0));
        }
        umma_commit(&q_empty[st]);  // frees the Q/dO stage and the TMEM buffers of block i
        if (i == nq - 1) umma_commit(acc_done);
      }
      __syncwarp();
    }
  } else {
    const int quad = warp & 3;
    const int half = (warp - 2) / 4;    // query columns [32*half, 32*half+32) of each 64-query block
    const int krow = quad * 32 + lane;  // key row within the block == TMEM lane
    const bool key_ok = krow < kv_rows;
    const int kt = kt_base + krow;      // own: local key index
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int tid = threadIdx.x - 64;   // 0..255
    constexpr int HC = BQ / 2;
    // LSE/D of query block i are loaded one block ahead into registers (tid < BQ) and published to
    // the stat buffer of that block at the start of its iteration (hides the global-load latency)
    float nl = INFINITY, nd = 0.f;
    auto fetch = [&](int i) {
      const int q = q_lo + i * BQ + tid;
      const bool ok = tid < BQ && i < nq && q < q_hi;
      // raw values only: the log2e scaling happens at the smem store one iteration later, so no
      // instruction consumes the global load until its latency is hidden
      nl = ok ? p.lse[static_cast<long>(h) * p.n + q] : INFINITY;
      nd = ok ? p.D[static_cast<long>(h) * p.n + q] : 0.f;
    };
    fetch(0);
    for (int i = 0; i < nq; ++i) {
      const int q0 = q_lo + i * BQ;
      float* st_lse = stat + (i & 1) * 2 * BQ;
      float* st_D = st_lse + BQ;
      if (tid < BQ) {
        st_lse[tid] = nl * kLog2e;
        st_D[tid] = nd;
      }
      named_bar_sync(1, 32 * kSmxWarps);
      fetch(i + 1);
      mbar_wait(&s_full[i % NB], (i / NB) & 1);
      tc_fence_after();
      float s[HC], dp[HC];
#pragma unroll
      for (int c = 0; c < HC; c += 16) {
        uint32_t r[16], r2[16];
        tmem_ld16(t_S + (i % NB) * BQ + half * HC + c + lane_off, r);
        tmem_ld16(t_dP + (i % NB) * BQ + half * HC + c + lane_off, r2);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          s[c + e] = __uint_as_float(r[e]);
          dp[c + e] = __uint_as_float(r2[e]);
        }
      }
      tmem_ld_wait();
      // own rows: key kt sees query t iff kt <= t, i.e. columns qi >= kt - (q0 - seg_off) (invalid
      // queries beyond q_hi already have lse2 = +inf -> P = 0; invalid keys are never stored)
      if (own) {
        const int lo = kt - (q0 - seg_off) - half * HC;
        if (__any_sync(0xffffffff, lo > 0)) {
#pragma unroll
          for (int c = 0; c < HC; ++c) s[c] = c >= lo ? s[c] : -INFINITY;
        }
      }
      const float c2 = p.scale_log2;
      const float* lz_base = st_lse + half * HC;
      const float* dz_base = st_D + half * HC;
      uint32_t wp[HC / 2], wd[HC / 2];
#pragma unroll
      for (int c = 0; c < HC; c += 4) {
        const float4 lz = *reinterpret_cast<const float4*>(lz_base + c);
        const float4 dz = *reinterpret_cast<const float4*>(dz_base + c);
        const float2 c22 = make_float2(c2, c2);
        const float2 xa = __ffma2_rn(make_float2(s[c], s[c + 1]), c22, make_float2(-lz.x, -lz.y));
        const float2 xb = __ffma2_rn(make_float2(s[c + 2], s[c + 3]), c22, make_float2(-lz.z, -lz.w));
        const float2 pa = ((c / 2) & 3) < POLY ? ex2_poly2(xa) : make_float2(ex2_approx(xa.x), ex2_approx(xa.y));
        const float2 pb = ((c / 2 + 1) & 3) < POLY ? ex2_poly2(xb) : make_float2(ex2_approx(xb.x), ex2_approx(xb.y));
        const float2 da = __fmul2_rn(pa, __fadd2_rn(make_float2(dp[c], dp[c + 1]), make_float2(-dz.x, -dz.y)));
        const float2 db = __fmul2_rn(pb, __fadd2_rn(make_float2(dp[c + 2], dp[c + 3]), make_float2(-dz.z, -dz.w)));
        wp[c / 2] = pack_bf16x2(pa.x, pa.y);
        wp[c / 2 + 1] = pack_bf16x2(pb.x, pb.y);
        wd[c / 2] = pack_bf16x2(da.x, da.y);
        wd[c / 2 + 1] = pack_bf16x2(db.x, db.y);
      }
      // P^T_i / dS^T_i (bf16 pairs) into this half's OWN columns of the S^T_i / dP^T_i buffers
      tmem_st16(t_S + (i % NB) * BQ + half * HC + lane_off, wp);
      tmem_st16(t_dP + (i % NB) * BQ + half * HC + lane_off, wd);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[i % NB]);
    }
    mbar_wait(acc_done, 0);
    tc_fence_after();
    float* dkr = p.dk + static_cast<long>(kv0 + krow) * p.lddkv + h * DH;
    float* dvr = p.dv + static_cast<long>(kv0 + krow) * p.lddkv + h * DH;
#pragma unroll
    for (int c = half * (DH / 2); c < (half + 1) * (DH / 2); c += 16) {
      uint32_t rk[16], rv[16];
      tmem_ld16(t_dK + c + lane_off, rk);
      tmem_ld16(t_dV + c + lane_off, rv);
      tmem_ld_wait();
      if (key_ok) {
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          red_add_v4_f32(dkr + c + e, __uint_as_float(rk[e]) * p.scale, __uint_as_float(rk[e + 1]) * p.scale,
                         __uint_as_float(rk[e + 2]) * p.scale, __uint_as_float(rk[e + 3]) * p.scale);
          red_add_v4_f32(dvr + c + e, __uint_as_float(rv[e]), __uint_as_float(rv[e + 1]), __uint_as_float(rv[e + 2]),
                         __uint_as_float(rv[e + 3]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::kTmemCols);
}

// ================================================================= dK/dV kernel, 128 x 128 blocks
// dh = 64 only. 128 keys x 128 queries per block: S^T / dP^T are N = 128 MMAs (full rate; the N = 64
// ones run at 2/3), and each issuer wait now covers twice the MMA work. TMEM: S^T[2] (128 each),
// ONE dP^T buffer (128), dK, dV (64 each) = 512 columns. P^T / dS^T (bf16 pairs) go over the S^T
// buffer: half h of the query columns packs P^T into [64h, 64h+32) and dS^T into [64h+32, 64h+64);
// the dP^T buffer is released as soon as the softmax has loaded it (dp_free), so dP^T_{i+1} is
// computed while the softmax of block i finishes.
template <int NS>
struct Dkv128Cfg {
  static constexpr int DH = 64, BKV = 128, BQ = 128;
  static constexpr int kKVBytes = BKV * DH * 2;  // K (or V) block
  static constexpr int kQBytes = BQ * DH * 2;    // Q_i (or dO_i) tile
  static constexpr int kOffV = kKVBytes;
  static constexpr int kOffQ = 2 * kKVBytes;
  static constexpr int kOffDO = kOffQ + NS * kQBytes;
  static constexpr int kOffStat = kOffDO + NS * kQBytes;  // [2][2][BQ] floats: lse2, D
  static constexpr int kOffBar = kOffStat + 2 * 2 * BQ * 4;
  static constexpr int kSmem = kOffBar + 256 + 1024;
  static constexpr int kTmemCols = 512;
  static_assert(kSmem <= 227 * 1024 && NS >= 2, "dkdv128: smem / ring");
  static constexpr uint32_t kIdescS = make_idesc_bf16(128, BQ, false, false);
  static constexpr uint32_t kIdescKV = make_idesc_bf16(128, DH, false, true);
};

template <int NS, int POLY>
__global__ void __launch_bounds__(kThreadsDq, 1)
    fa_bwd_dkdv128_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                          BwdParams p) {
  using C = Dkv128Cfg<NS>;
  constexpr int DH = C::DH, BQ = C::BQ;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;
  uint64_t* q_empty = q_full + NS;  // dV/dK_i done: frees the Q/dO stage and S^T buffer i % 2
  uint64_t* s_full = q_empty + NS;  // [2]
  uint64_t* p_full = s_full + 2;    // [2] softmax done with block i (P^T / dS^T in TMEM)
  uint64_t* dp_full = p_full + 2;   // dP^T_i computed (single buffer)
  uint64_t* dp_free = dp_full + 1;  // softmax has loaded dP^T_i
  uint64_t* acc_done = dp_free + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);
  float* stat = reinterpret_cast<float*>(smem + C::kOffStat);

  const int warp = warp_id_sync();
  const int lane = threadIdx.x & 31;
  const int4 it = p.blocks[blockIdx.x];
  const int2 it2 = p.blocks2[blockIdx.x];
  const int kv0 = it.x, kv_rows = it.y, q_lo = it.z, q_hi = it.w;
  const int seg_off = it2.x;
  const bool own = it2.y != 0;
  const int kt_base = own ? kv0 - p.r0 - seg_off : 0;
  const int h = blockIdx.y;
  const int nq = (q_hi - q_lo + BQ - 1) / BQ;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_init(kv_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], kSmxWarps);
    }
    mbar_init(dp_full, 1);
    mbar_init(dp_free, kSmxWarps);
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_S = tmem, t_dP = tmem + 256, t_dK = tmem + 384, t_dV = tmem + 448;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * C::kKVBytes);
      tma_load_2d(&tm_k, kv_full, smem, h * DH, kv0);
      tma_load_2d(&tm_v, kv_full, smem + C::kOffV, h * DH, kv0);
      for (int i = 0; i < nq; ++i) {
        const int st = i % NS;
        mbar_wait(&q_empty[st], ((i / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[st], 2 * C::kQBytes);
        const int q0 = q_lo + i * BQ;
        tma_load_2d(&tm_q, &q_full[st], smem + C::kOffQ + st * C::kQBytes, h * DH, q0);
        tma_load_2d(&tm_do, &q_full[st], smem + C::kOffDO + st * C::kQBytes, h * DH, q0);
      }
    }
  } else if (warp == 1) {
    // S^T_i = K Q_i^T into S buffer i % 2 (after dV/dK_{i-2}); dP^T_i = V dO_i^T into the single dP^T
    // buffer (after the softmax loaded dP^T_{i-1})
    const uint64_t d16 = make_sdesc_sw128(smem_u32(smem), 16, 1024);
    mbar_wait(kv_full, 0);
    for (int i = 0; i < nq; ++i) {
      const int st = i % NS;
      if (i >= 2) mbar_wait(&q_empty[(i - 2) % NS], ((i - 2) / NS) & 1);
      mbar_wait(&q_full[st], (i / NS) & 1);
      tc_fence_after();
      const uint32_t q_off = C::kOffQ + st * C::kQBytes, do_off = C::kOffDO + st * C::kQBytes;
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < DH / 16; ++k)
          umma_bf16_ss(t_S + (i & 1) * 128, sdesc_add(d16, k * 32), sdesc_add(sdesc_add(d16, q_off), k * 32), C::kIdescS,
                       k > 0);
        umma_commit(&s_full[i & 1]);
      }
      __syncwarp();
      if (i >= 1) mbar_wait(dp_free, (i - 1) & 1);
      tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < DH / 16; ++k)
          umma_bf16_ss(t_dP, sdesc_add(d16, C::kOffV + k * 32), sdesc_add(sdesc_add(d16, do_off), k * 32), C::kIdescS,
                       k > 0);
        umma_commit(dp_full);
      }
      __syncwarp();
    }
  } else if (warp == 10) {
    // dV += P^T dO_i ; dK += dS^T Q_i  (A from the S^T buffer: P^T at 64h + ..., dS^T at 64h + 32 + ...)
    const uint64_t dmn = make_sdesc_sw128(smem_u32(smem), BQ * 128, 1024);
    for (int i = 0; i < nq; ++i) {
      mbar_wait(&p_full[i & 1], (i >> 1) & 1);
      tc_fence_after();
      if (lane == 0) {
        const int st = i % NS;
        const uint32_t q_off = C::kOffQ + st * C::kQBytes, do_off = C::kOffDO + st * C::kQBytes;
#pragma unroll
        for (int k = 0; k < BQ / 16; ++k) {
          const uint32_t col = (k / 4) * 64 + (k % 4) * 8;
          umma_bf16_ts(t_dV, t_S + (i & 1) * 128 + col, sdesc_add(sdesc_add(dmn, do_off), k * 2048), C::kIdescKV,
                       (i > 0 || k > 0));
          umma_bf16_ts(t_dK, t_S + (i & 1) * 128 + col + 32, sdesc_add(sdesc_add(dmn, q_off), k * 2048), C::kIdescKV,
                       (i > 0 || k > 0));
        }
        umma_commit(&q_empty[st]);
        if (i == nq - 1) umma_commit(acc_done);
      }
      __syncwarp();
    }
  } else {
    const int quad = warp & 3;
    const int half = (warp - 2) / 4;    // query columns [64*half, 64*half+64) of each 128-query block
    const int krow = quad * 32 + lane;  // key row within the block == TMEM lane
    const bool key_ok = krow < kv_rows;
    const int kt = kt_base + krow;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int tid = threadIdx.x - 64;  // 0..255
    float nl = INFINITY, nd = 0.f;
    auto fetch = [&](int i) {
      const int q = q_lo + i * BQ + tid;
      const bool ok = tid < BQ && i < nq && q < q_hi;
      nl = ok ? p.lse[static_cast<long>(h) * p.n + q] : INFINITY;
      nd = ok ? p.D[static_cast<long>(h) * p.n + q] : 0.f;
    };
    fetch(0);
    const float c2 = p.scale_log2;
    // P^T / dS^T of one 32-query sub-chunk sc (columns 64*half + 32*sc ...)
    auto sub = [&](int i, int sc, const float (&s_in)[32], const float (&dp)[32], const float* st_lse,
                   const float* st_D, uint32_t (&wp)[16], uint32_t (&wd)[16]) {
      const int q0 = q_lo + i * BQ;
      const int cb = 64 * half + 32 * sc;  // block column of s_in[0]
      float s[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) s[c] = s_in[c];
      if (own) {
        const int lo = kt - (q0 - seg_off) - cb;  // key kt sees query column c iff c >= lo
        if (__any_sync(0xffffffff, lo > 0)) {
#pragma unroll
          for (int c = 0; c < 32; ++c) s[c] = c >= lo ? s[c] : -INFINITY;
        }
      }
      const float* lz_base = st_lse + cb;
      const float* dz_base = st_D + cb;
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        const float4 lz = *reinterpret_cast<const float4*>(lz_base + c);
        const float4 dz = *reinterpret_cast<const float4*>(dz_base + c);
        const float2 c22 = make_float2(c2, c2);
        const float2 xa = __ffma2_rn(make_float2(s[c], s[c + 1]), c22, make_float2(-lz.x, -lz.y));
        const float2 xb = __ffma2_rn(make_float2(s[c + 2], s[c + 3]), c22, make_float2(-lz.z, -lz.w));
        const float2 pa = ((c / 2) & 3) < POLY ? ex2_poly2(xa) : make_float2(ex2_approx(xa.x), ex2_approx(xa.y));
        const float2 pb = ((c / 2 + 1) & 3) < POLY ? ex2_poly2(xb) : make_float2(ex2_approx(xb.x), ex2_approx(xb.y));
        const float2 da = __fmul2_rn(pa, __fadd2_rn(make_float2(dp[c], dp[c + 1]), make_float2(-dz.x, -dz.y)));
        const float2 db = __fmul2_rn(pb, __fadd2_rn(make_float2(dp[c + 2], dp[c + 3]), make_float2(-dz.z, -dz.w)));
        wp[c / 2] = pack_bf16x2(pa.x, pa.y);
        wp[c / 2 + 1] = pack_bf16x2(pb.x, pb.y);
        wd[c / 2] = pack_bf16x2(da.x, da.y);
        wd[c / 2 + 1] = pack_bf16x2(db.x, db.y);
      }
    };
    auto ld32 = [&](uint32_t taddr, float (&v)[32]) {
      uint32_t r[16], r2[16];
      tmem_ld16(taddr + lane_off, r);
      tmem_ld16(taddr + 16 + lane_off, r2);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        v[e] = __uint_as_float(r[e]);
        v[16 + e] = __uint_as_float(r2[e]);
      }
    };
    for (int i = 0; i < nq; ++i) {
      float* st_lse = stat + (i & 1) * 2 * BQ;
      float* st_D = st_lse + BQ;
      if (tid < BQ) {
        st_lse[tid] = nl * kLog2e;
        st_D[tid] = nd;
      }
      named_bar_sync(1, 32 * kSmxWarps);
      fetch(i + 1);
      const uint32_t sb = t_S + (i & 1) * 128 + 64 * half;
      const uint32_t pb = t_dP + 64 * half;
      mbar_wait(&s_full[i & 1], (i >> 1) & 1);
      tc_fence_after();
      float s0[32], s1[32], dp[32];
      ld32(sb, s0);
      ld32(sb + 32, s1);  // loaded before dS^T of sub-chunk 0 overwrites these columns
      mbar_wait(dp_full, i & 1);
      tc_fence_after();
      ld32(pb, dp);
      uint32_t wp[16], wd[16];
      sub(i, 0, s0, dp, st_lse, st_D, wp, wd);
      ld32(pb + 32, dp);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dp_free);  // dP^T_i fully in registers: dP^T_{i+1} may overwrite it
      tmem_st16(sb + lane_off, wp);         // P^T sub-chunk 0 -> [64h, 64h+16)
      tmem_st16(sb + 32 + lane_off, wd);    // dS^T sub-chunk 0 -> [64h+32, 64h+48)
      sub(i, 1, s1, dp, st_lse, st_D, wp, wd);
      tmem_st16(sb + 16 + lane_off, wp);
      tmem_st16(sb + 48 + lane_off, wd);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[i & 1]);
    }
    mbar_wait(acc_done, 0);
    tc_fence_after();
    float* dkr = p.dk + static_cast<long>(kv0 + krow) * p.lddkv + h * DH;
    float* dvr = p.dv + static_cast<long>(kv0 + krow) * p.lddkv + h * DH;
#pragma unroll
    for (int c = half * (DH / 2); c < (half + 1) * (DH / 2); c += 16) {
      uint32_t rk[16], rv[16];
      tmem_ld16(t_dK + c + lane_off, rk);
      tmem_ld16(t_dV + c + lane_off, rv);
      tmem_ld_wait();
      if (key_ok) {
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          red_add_v4_f32(dkr + c + e, __uint_as_float(rk[e]) * p.scale, __uint_as_float(rk[e + 1]) * p.scale,
                         __uint_as_float(rk[e + 2]) * p.scale, __uint_as_float(rk[e + 3]) * p.scale);
          red_add_v4_f32(dvr + c + e, __uint_as_float(rv[e]), __uint_as_float(rv[e + 1]), __uint_as_float(rv[e + 2]),
                         __uint_as_float(rv[e + 3]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::kTmemCols);
}

template <int DH, int POLY>
void launch_bwd(const AttnBwdArgs& a, long rows_cap, const int4* dq_blocks, int n_dq, const int4* kv_items,
                const int2* kv_items2, int n_kv, cudaStream_t stream) {
  // ring depths: loads must run >= 2 blocks ahead of the MMA that frees their stage
  // Ring depths: a stage is held until the LAST MMA reading it completes (dQ_j reads K_j; dV/dK_i
  // read Q_i/dO_i), so the refill of the stage NS blocks ahead only starts then. The ring must cover
  // that plus the L2/HBM TMA latency (~1-2 us under load), i.e. several block periods.
  constexpr int NSQ = DH == 64 ? 8 : 4;  // dq kernel K/V stages (smem: 192 KB / 224 KB)
  constexpr int NSK = DH == 64 ? 8 : 4;  // dkdv kernel Q/dO stages
  using CQ = DqCfg<DH, NSQ>;
  using CK = DkvCfg<DH, NSK>;
  static const int part = [] {  // TT_ATTN_BWD_PART (timing experiments): 1 = dQ kernel only, 2 = dK/dV only
    const char* e = std::getenv("TT_ATTN_BWD_PART");
    return e ? std::atoi(e) : 0;
  }();
  if (part == 2) n_dq = 0;
  if (part == 1) n_kv = 0;
  const int d = a.H * DH;
  BwdParams p{a.lse, a.D, a.dq, a.lddq, a.dq16, a.lddq16, a.dk, a.dv, a.lddkv, a.n, a.S, a.H, a.pbase, a.r0 < 0 ? a.S : a.r0,
              dq_blocks, nullptr, a.scale,
              a.scale * kLog2e};
  if (n_dq > 0) {
    CUtensorMap tq, tdo, tk, tv;
    make_tmap_bf16(&tq, a.q, d, a.n, a.ldq, 64, 128);
    make_tmap_bf16(&tdo, a.dO, d, a.n, a.ldq, 64, 128);
    make_tmap_bf16(&tk, a.k, d, rows_cap, a.ldkv, 64, CQ::BKV);
    make_tmap_bf16(&tv, a.v, d, rows_cap, a.ldkv, 64, CQ::BKV);
    static bool once = (cudaFuncSetAttribute(fa_bwd_dq_kernel<DH, NSQ, POLY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             CQ::kSmem),
                        true);
    (void)once;
    static const int dbg = [] {
      const char* e = std::getenv("TT_ATTN_DBG");
      return e ? std::atoi(e) : 0;
    }();
    if (dbg == 1 || dbg == 2 || dbg == 3 || dbg == 5) {
      auto kfn = dbg == 1 ? fa_bwd_dq_kernel<DH, NSQ, POLY, 1>
                          : (dbg == 2 ? fa_bwd_dq_kernel<DH, NSQ, POLY, 2>
                                      : (dbg == 3 ? fa_bwd_dq_kernel<DH, NSQ, POLY, 4> : fa_bwd_dq_kernel<DH, NSQ, POLY, 5>));
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, CQ::kSmem);
      kfn<<<dim3(n_dq, a.H), kThreadsDq, CQ::kSmem, stream>>>(tq, tdo, tk, tv, p);
    } else {
      fa_bwd_dq_kernel<DH, NSQ, POLY><<<dim3(n_dq, a.H), kThreadsDq, CQ::kSmem, stream>>>(tq, tdo, tk, tv, p);
    }
  }
  if (n_kv > 0) {
    CUtensorMap tq, tdo, tk, tv;
    make_tmap_bf16(&tq, a.q, d, a.n, a.ldq, 64, CK::BQ);
    make_tmap_bf16(&tdo, a.dO, d, a.n, a.ldq, 64, CK::BQ);
    make_tmap_bf16(&tk, a.k, d, rows_cap, a.ldkv, 64, 128);
    make_tmap_bf16(&tv, a.v, d, rows_cap, a.ldkv, 64, 128);
    static bool once = (cudaFuncSetAttribute(fa_bwd_dkdv_kernel<DH, NSK, POLY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             CK::kSmem),
                        true);
    (void)once;
    p.blocks = kv_items;
    p.blocks2 = kv_items2;
    static const bool k128 = [] {  // TT_ATTN_DKDV128=0: the 64-query-block dK/dV kernel (A/B timing)
      const char* e = std::getenv("TT_ATTN_DKDV128");
      return !(e && std::atoi(e) == 0);
    }();
    if (DH == 64 && k128) {
      using C8 = Dkv128Cfg<5>;
      CUtensorMap tq8, tdo8;
      make_tmap_bf16(&tq8, a.q, d, a.n, a.ldq, 64, C8::BQ);
      make_tmap_bf16(&tdo8, a.dO, d, a.n, a.ldq, 64, C8::BQ);
      static bool once8 = (cudaFuncSetAttribute(fa_bwd_dkdv128_kernel<5, POLY>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, C8::kSmem),
                           true);
      (void)once8;
      fa_bwd_dkdv128_kernel<5, POLY><<<dim3(n_kv, a.H), kThreadsDq, C8::kSmem, stream>>>(tq8, tdo8, tk, tv, p);
    } else {
      fa_bwd_dkdv_kernel<DH, NSK, POLY><<<dim3(n_kv, a.H), kThreadsDq, CK::kSmem, stream>>>(tq, tdo, tk, tv, p);
    }
  }
}

}  // namespace

int attn_debug_trace(long long* host, int n) {
  const int m = n < 6 * 256 ? n : 6 * 256;
  return cudaMemcpyFromSymbol(host, g_attn_trace, m * sizeof(long long)) == cudaSuccess ? m : -1;
}

void attn_bwd_sm100(const AttnBwdArgs& a, long rows_cap, const int4* dq_blocks, int n_dq, const int4* kv_items,
                    const int2* kv_items2, int n_kv, cudaStream_t stream) {
  attn_bwd_pre(a, stream);
  // TT_ATTN_BWD_POLY: exponential pairs (of 4) on the FMA pipe (timing experiments)
  static const int bpoly = [] {
    const char* e = std::getenv("TT_ATTN_BWD_POLY");
    return e ? std::atoi(e) : 0;
  }();
#define TT_BWD(P)                                                                                          \
  if (a.dh == 64) return launch_bwd<64, P>(a, rows_cap, dq_blocks, n_dq, kv_items, kv_items2, n_kv, stream); \
  if (a.dh == 128) return launch_bwd<128, P>(a, rows_cap, dq_blocks, n_dq, kv_items, kv_items2, n_kv, stream);
  switch (bpoly) {
    case 1: TT_BWD(1) break;
    case 2: TT_BWD(2) break;
    default: TT_BWD(0) break;
  }
#undef TT_BWD
  throw std::invalid_argument("attention: head_dim must be 64 or 128");
}

}  // namespace ttb
