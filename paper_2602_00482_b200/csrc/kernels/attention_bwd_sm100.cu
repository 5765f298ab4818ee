// tcgen05 / TMEM / TMA segment attention backward over the device KV stack (sm_100a).
//
// Replaces the attention backward of backward_segment (model.hpp:546-604):
//   P = softmax(scale Q K^T) (recomputed from the forward LSE), dP = dO V^T,
//   dS = P * (dP - D) with D = rowsum(dO * O),  dQ = scale dS K,  dK = scale dS^T Q,  dV = P^T dO.
// ONE fused key-parallel kernel per head size (fa_bwd_fused_kernel: dh 64, 128-query blocks;
// fa_bwd_fused128_kernel: dh 128, 64-query blocks, dQ^T = K^T dS^T): P and dS once per (key block,
// query block) pair; dK/dV accumulate in TMEM and are added once into the fp32 dK/dV stack rows
// (red.add.v4: several query-range items and sibling segments contribute to the same prefix rows) or,
// for own rows with a single writer, stored as bf16 into the packed QKV-backward operand; dQ partials
// leave through cp.reduce.async.bulk into an fp32 accumulator. Two MMA-issuing warps, 8
// softmax-gradient warps (2 per TMEM lane quadrant, each owning half of the columns), 4 dQ-drain warps.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <stdexcept>

#include "attention.h"
#include "gemm.h"
#include "launch.cuh"
#include "sm100.cuh"

// Resource experiments (tools/attn_bwd_ab.sh builds; the product and trace builds define none of
// these): each drops one consumer of shared memory / the tensor pipe to find the binding resource.
#ifndef TT_EXP_BWD
#define TT_EXP_BWD 0  // 1 no dS^T smem stores, 2 no dQ drain stores/reduce, 3 no dK MMAs, 4 no dQ MMAs,
                      // 5 no stats LDS
#endif

// Pipeline trace (clock64 per event) of the fused dh=64 kernel: compiled only into the separate
// debug library (make trace -> libtreetrain_b200_trace.so, -DTT_TRACE=1); the product build has none.
#ifndef TT_TRACE
#define TT_TRACE 0
#endif
#if TT_TRACE
constexpr int kTrCtas = 96, kTrBlocks = 33, kTrEv = 10;  // block row kTrBlocks-1 holds CTA-level events
__device__ long long g_tt_trace[kTrCtas][kTrBlocks][kTrEv];
#define TT_TR(ev, i)                                                                            \
  do {                                                                                          \
    if (blockIdx.y == 0 && blockIdx.x < kTrCtas && (i) < kTrBlocks) g_tt_trace[blockIdx.x][(i)][(ev)] = clock64(); \
  } while (0)
constexpr int kTrBlocksLast = kTrBlocks - 1;
#else
constexpr int kTrBlocksLast = 0;
#define TT_TR(ev, i) \
  do {               \
  } while (0)
#endif

namespace ttb {

namespace {

constexpr int kSmxWarps = 8;   // softmax-gradient warps; the pair on a quadrant splits the columns
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}


struct BwdParams {
  const float* lse;  // [H x n]
  const float* D;    // [H x n]
  float* dq;         // [n x lddq]
  long lddq;
  float* dk;  // stack rows (this layer), fp32: the batch's own rows
  float* dv;
  long lddkv;
  float* dk_pre;  // where the prefix rows' dK/dV go (absolute rows, same pitch): the stack, or a
  float* dv_pre;  // separate buffer when the caller wants this pop's grad_prefix by itself
  int n, S, H;
  int pbase, r0;        // prefix rows [pbase, pbase + S); own rows from r0
  const int4* blocks;   // {kv_row0, kv_rows, q_lo, q_hi}
  const int2* blocks2;  // {seg_off, is_own}: 0 prefix rows, 1 own rows (red.add), 2 own rows with
                        // a single writer (fused kernel: bf16 store into kv16)
  float scale, scale_log2;
  __nv_bfloat16* kv16;  // packed-operand dk block (dv block at + H * 64), batch-local rows, pitch ldkv16
  long ldkv16;
};

// ============================================================ fused dQ / dK / dV kernel, dh = 64
// One kernel per (128-key stack block, head, query range) item; it loops over the range's 128-query
// blocks i and computes P and dS ONCE per (key block, query block) pair:
//   warp 1      S^T_i = K Q_i^T, dP^T_i = V dO_i^T                (SS, M = 128 keys, N = 128 queries)
//   warps 8-15  P^T = 2^(S^T c - lse2),  dS^T = P^T (dP^T scale - D scale)  (the softmax-gradient
//               stream): P^T back into TMEM as bf16 pairs over S^T_i columns [0, 64), dS^T into a
//               swizzled 32 KB smem tile (two of them: block i + 1's softmax never waits for block i's
//               dK / dQ MMAs)
//   warp 2      dV += P^T_i dO_i (TS), dK += dS^T_i Q_i (SS, the tile read K-major),
//               dQ_i = dS_i K (SS, the same tile read MN-major) into S^T_i columns [64, 128)
//   warps 4-7   dQ_i: TMEM -> registers -> swizzled smem -> cp.reduce.async.bulk .add into the fp32
//               dQ accumulator [n x d] (each query block receives one partial per key block)
//   warp 0      TMA: K, V once; Q_i / dO_i through an NS-stage ring
// The softmax scale is folded into dS, so dK and dQ need no epilogue scaling. The two separate
// kernels this replaces (query-parallel dQ, key-parallel dK/dV) each recomputed P and dS.
// TMEM (512 columns): S^T[2] (128 each; P^T / dQ_i reuse them), dP^T (128), dK (64), dV (64).
template <int NS>
struct FusedCfg {
  static constexpr int DH = 64, BKV = 128, BQ = 128;
  static constexpr int kKVBytes = BKV * DH * 2;                // K (or V) block, loaded once
  static constexpr int kQBytes = BQ * DH * 2;                  // Q_i (or dO_i) tile
  static constexpr int kOffV = kKVBytes;
  static constexpr int kOffQ = 2 * kKVBytes;
  static constexpr int kOffDO = kOffQ + NS * kQBytes;
  static constexpr int kDSBytes = 2 * BKV * 128;               // dS^T: 2 query panels x [128 keys][128 B]
  static constexpr int kOffDS = kOffDO + NS * kQBytes;         // two dS^T tiles (blocks i, i + 1)
  static constexpr int kOffDQ = kOffDS + 2 * kDSBytes;         // dQ staging: 4 warps x (32 x 32 fp32)
  static constexpr int kOffStat = kOffDQ + 4 * 4096;           // [2][2][BQ] floats: lse2, -scale D
  static constexpr int kOffBar = kOffStat + 2 * 2 * BQ * 4;
  static constexpr int kSmem = kOffBar + 256 + 1024;
  static_assert(kSmem <= 227 * 1024 && NS >= 2, "fused attention backward: smem / ring");
  static constexpr uint32_t kIdescS = make_idesc_bf16(128, BQ, false, false);  // S^T, dP^T
  static constexpr uint32_t kIdescKV = make_idesc_bf16(128, DH, false, true);  // dV (TS), dK (A K-major)
  static constexpr uint32_t kIdescQ = make_idesc_bf16(128, DH, true, true);    // dQ (A = dS MN-major)
};
constexpr int kThreadsFused = 512;  // warps 0-2 control (3 idle), 4-7 dQ drain, 8-15 softmax

__device__ __forceinline__ void tma_reduce_add_2d(const void* tmap, const void* smem_src, int32_t x, int32_t y) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(smem_src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int NS>
__global__ void __launch_bounds__(kThreadsFused, 1)
    fa_bwd_fused_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                        const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                        const __grid_constant__ CUtensorMap tm_dq, BwdParams p) {
  using C = FusedCfg<NS>;
  constexpr int DH = C::DH, BQ = C::BQ;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;
  uint64_t* q_empty = q_full + NS;  // dV/dK/dQ_i issued and done: the Q/dO stage is free
  uint64_t* s_full = q_empty + NS;  // [2] S^T_i in TMEM
  uint64_t* p_full = s_full + 2;    // [2] softmax done with block i: P^T_i in TMEM, dS^T_i in smem
  uint64_t* dp_full = p_full + 2;   // dP^T_i computed (single buffer)
  uint64_t* dp_free = dp_full + 1;  // softmax has loaded dP^T_i
  uint64_t* ds_free = dp_free + 1;  // [2] dK_i / dQ_i done: dS^T tile i % 2 may be rewritten
  uint64_t* dq_full = ds_free + 2;  // [2] dQ_i in TMEM
  uint64_t* dq_free = dq_full + 2;  // [2] dQ_i read out: S^T buffer i % 2 may take S^T_{i+2}
  uint64_t* acc_done = dq_free + 2;
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
    tma_prefetch_desc(&tm_dq);
    mbar_init(kv_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], kSmxWarps);
      mbar_init(&dq_full[s], 1);
      mbar_init(&dq_free[s], 4);
      mbar_init(&ds_free[s], 1);
    }
    mbar_init(dp_full, 1);
    mbar_init(dp_free, kSmxWarps);
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // predecessor grid complete (launch.cuh); TMEM held before the successor may start
  pdl_trigger_early();
  const uint32_t t_S = tmem, t_dP = tmem + 256, t_dK = tmem + 384, t_dV = tmem + 448;
  const int wg = warp >> 2;
  if (threadIdx.x == 0) TT_TR(0, kTrBlocksLast);

  if (wg == 0) {
    if (warp == 0 && lane == 0) {
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
    } else if (warp == 1) {
      // S^T_i into buffer i % 2 once dQ_{i-2} has been read out of it; dP^T_i once the softmax has
      // loaded dP^T_{i-1}
      const uint64_t d16 = make_sdesc_sw128(smem_u32(smem), 16, 1024);  // K-major tiles
      mbar_wait(kv_full, 0);
      if (lane == 0) TT_TR(1, kTrBlocksLast);
      for (int i = 0; i < nq; ++i) {
        const int st = i % NS;
        if (i >= 2) mbar_wait(&dq_free[i & 1], ((i - 2) >> 1) & 1);
        mbar_wait(&q_full[st], (i / NS) & 1);
        tc_fence_after();
        const uint32_t q_off = C::kOffQ + st * C::kQBytes, do_off = C::kOffDO + st * C::kQBytes;
        if (lane == 0) {
          TT_TR(0, i);
#pragma unroll
          for (int k = 0; k < DH / 16; ++k)
            umma_bf16_ss(t_S + (i & 1) * 128, sdesc_add(d16, k * 32), sdesc_add(d16, q_off + k * 32), C::kIdescS,
                         k > 0);
          umma_commit(&s_full[i & 1]);
        }
        __syncwarp();
        if (i >= 1) mbar_wait(dp_free, (i - 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          TT_TR(1, i);
#pragma unroll
          for (int k = 0; k < DH / 16; ++k)
            umma_bf16_ss(t_dP, sdesc_add(d16, C::kOffV + k * 32), sdesc_add(d16, do_off + k * 32), C::kIdescS, k > 0);
          umma_commit(dp_full);
        }
        __syncwarp();
      }
    } else if (warp == 2) {
      // dV += P^T_i dO_i ; dK += dS^T_i Q_i ; dQ_i = dS_i K
      const uint64_t dmn = make_sdesc_sw128(smem_u32(smem), BQ * 128, 1024);  // Q_i / dO_i / K as MN-major B
      const uint64_t dsk = make_sdesc_sw128(smem_u32(smem + C::kOffDS), 16, 1024);           // dS^T, K-major A
      const uint64_t dsm = make_sdesc_sw128(smem_u32(smem + C::kOffDS), C::BKV * 128, 1024);  // dS, MN-major A
      for (int i = 0; i < nq; ++i) {
        mbar_wait(&p_full[i & 1], (i >> 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          TT_TR(5, i);
          const int st = i % NS;
          const uint32_t q_off = C::kOffQ + st * C::kQBytes, do_off = C::kOffDO + st * C::kQBytes;
          const uint32_t ds_off = (i & 1) * C::kDSBytes;
          // dV_i (reads P^T_i from S^T buffer i % 2), then dQ_i (into the same buffer): the dq_full
          // commit covers both, so once dQ_i is drained the buffer is free for S^T_{i+2} — the
          // loop-carried dependency of the pipeline; dK_i runs behind it, during the drain
#pragma unroll
          for (int k = 0; k < BQ / 16; ++k)  // 16 queries per step
            umma_bf16_ts(t_dV, t_S + (i & 1) * 128 + 8 * k, sdesc_add(dmn, do_off + k * 2048), C::kIdescKV,
                         (i > 0 || k > 0));
#pragma unroll
          for (int k = 0; k < C::BKV / 16; ++k)  // 16 keys per step
            if (TT_EXP_BWD != 4)
              umma_bf16_ss(t_S + (i & 1) * 128 + 64, sdesc_add(dsm, ds_off + k * 2048), sdesc_add(dmn, k * 2048),
                           C::kIdescQ, k > 0);
          umma_commit(&dq_full[i & 1]);
#pragma unroll
          for (int k = 0; k < BQ / 16; ++k)
            if (TT_EXP_BWD != 3)
              umma_bf16_ss(t_dK, sdesc_add(dsk, ds_off + (k / 4) * 16384 + (k % 4) * 32),
                           sdesc_add(dmn, q_off + k * 2048), C::kIdescKV, (i > 0 || k > 0));
          umma_commit(&q_empty[st]);
          umma_commit(&ds_free[i & 1]);
          if (i == nq - 1) umma_commit(acc_done);
        }
        __syncwarp();
      }
    }
  } else if (wg == 1) {
    // dQ drain: warp w reads TMEM lanes (query rows) 32 (w % 4) .. +31 of dQ_i
    const int qd = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(qd * 32) << 16;
    uint8_t* stage = smem + C::kOffDQ + qd * 4096;
    for (int i = 0; i < nq; ++i) {
      const int q0 = q_lo + i * BQ;
      mbar_wait(&dq_full[i & 1], (i >> 1) & 1);
      tc_fence_after();
      if (warp == 4 && lane == 0) TT_TR(6, i);
      uint32_t r[64];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t t[16];
        tmem_ld16(t_S + (i & 1) * 128 + 64 + 16 * c + lane_off, t);
#pragma unroll
        for (int e = 0; e < 16; ++e) r[16 * c + e] = t[e];
      }
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dq_free[i & 1]);
#pragma unroll
      for (int cc = 0; cc < (TT_EXP_BWD == 2 ? 0 : 2); ++cc) {
        if (lane == 0) bulk_wait_read0();  // the previous reduce has read the staging buffer
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(stage + lane * 128 + ((c ^ (lane & 7)) * 16)) =
              make_uint4(r[32 * cc + 4 * c], r[32 * cc + 4 * c + 1], r[32 * cc + 4 * c + 2], r[32 * cc + 4 * c + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_reduce_add_2d(&tm_dq, stage, h * DH + 32 * cc, q0 + 32 * qd);
          bulk_commit();
        }
      }
      __syncwarp();
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  } else {
    const int qd = warp & 3;
    const int half = (warp - 8) >> 2;   // query columns [64 half, 64 half + 64) of each block
    const int krow = qd * 32 + lane;    // key row within the block == TMEM lane
    const bool key_ok = krow < kv_rows;
    const int kt = kt_base + krow;      // own: local key index
    const uint32_t lane_off = static_cast<uint32_t>(qd * 32) << 16;
    const int tid = threadIdx.x - 256;  // 0..255
    uint8_t* ds_rows = smem + C::kOffDS + half * (C::BKV * 128) + krow * 128;
    float nl = INFINITY, nd = 0.f;
    auto fetch = [&](int i) {
      const int q = q_lo + i * BQ + tid;
      const bool ok = tid < BQ && i < nq && q < q_hi;
      nl = ok ? p.lse[static_cast<long>(h) * p.n + q] : INFINITY;
      nd = ok ? p.D[static_cast<long>(h) * p.n + q] : 0.f;
    };
    fetch(0);
    const float c2 = p.scale_log2, sc = p.scale;
    for (int i = 0; i < nq; ++i) {
      const int q0 = q_lo + i * BQ;
      float* st_lse = stat + (i & 1) * 2 * BQ;
      float* st_nd = st_lse + BQ;
      if (tid < BQ) {
        st_lse[tid] = nl * kLog2e;
        st_nd[tid] = -nd * sc;
      }
      named_bar_sync(1, 32 * kSmxWarps);
      if (warp == 8 && lane == 0) TT_TR(8, i);
      fetch(i + 1);
      // visibility: invalid keys see nothing; own rows: key kt sees query t iff kt <= t, i.e. block
      // columns >= kt - (q0 - seg_off) (queries beyond q_hi have lse2 = +inf -> P = 0)
      const int lo0 = key_ok ? (own ? kt - (q0 - seg_off) - 64 * half : 0) : 64;
      const bool need_mask = __any_sync(0xffffffff, lo0 > 0);
      mbar_wait(&s_full[i & 1], (i >> 1) & 1);
      mbar_wait(dp_full, i & 1);
      tc_fence_after();
      if (warp == 8 && lane == 0) TT_TR(2, i);
      const uint32_t sbuf = t_S + (i & 1) * 128;
#pragma unroll
      for (int sub = 0; sub < 2; ++sub) {
        float sv[32], dp[32];
        {
          uint32_t r[16], r2[16], r3[16], r4[16];
          tmem_ld16(sbuf + 64 * half + 32 * sub + lane_off, r);
          tmem_ld16(sbuf + 64 * half + 32 * sub + 16 + lane_off, r2);
          tmem_ld16(t_dP + 64 * half + 32 * sub + lane_off, r3);
          tmem_ld16(t_dP + 64 * half + 32 * sub + 16 + lane_off, r4);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            sv[e] = __uint_as_float(r[e]);
            sv[16 + e] = __uint_as_float(r2[e]);
            dp[e] = __uint_as_float(r3[e]);
            dp[16 + e] = __uint_as_float(r4[e]);
          }
        }
        if (sub == 1) {
          if (warp == 8 && lane == 0) TT_TR(3, i);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dp_free);  // dP^T_i in registers: dP^T_{i+1} may overwrite it
          // half 0 has now loaded S^T columns [32, 64): half 1 may pack its P^T over them
          if (half == 0) named_bar_arrive(2 + qd, 64);
        }
        if (need_mask) {
          const int lo = lo0 - 32 * sub;
#pragma unroll
          for (int c = 0; c < 32; ++c) sv[c] = c >= lo ? sv[c] : -INFINITY;
        }
        const float* lz_base = st_lse + 64 * half + 32 * sub;
        const float* dz_base = st_nd + 64 * half + 32 * sub;
        uint32_t wp[16], wd[16];
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          const float4 lz = TT_EXP_BWD == 5 ? make_float4(nl, nl, nd, nd) : *reinterpret_cast<const float4*>(lz_base + c);
          const float4 dz = TT_EXP_BWD == 5 ? make_float4(nd, nl, nd, nl) : *reinterpret_cast<const float4*>(dz_base + c);
          const float2 c22 = make_float2(c2, c2), sc2 = make_float2(sc, sc);
          const float2 xa = __ffma2_rn(make_float2(sv[c], sv[c + 1]), c22, make_float2(-lz.x, -lz.y));
          const float2 xb = __ffma2_rn(make_float2(sv[c + 2], sv[c + 3]), c22, make_float2(-lz.z, -lz.w));
          const float2 pa = make_float2(ex2_approx(xa.x), ex2_approx(xa.y));
          const float2 pb = make_float2(ex2_approx(xb.x), ex2_approx(xb.y));
          const float2 da = __fmul2_rn(pa, __ffma2_rn(make_float2(dp[c], dp[c + 1]), sc2, make_float2(dz.x, dz.y)));
          const float2 db = __fmul2_rn(pb, __ffma2_rn(make_float2(dp[c + 2], dp[c + 3]), sc2, make_float2(dz.z, dz.w)));
          wp[c / 2] = pack_bf16x2(pa.x, pa.y);
          wp[c / 2 + 1] = pack_bf16x2(pb.x, pb.y);
          wd[c / 2] = pack_bf16x2(da.x, da.y);
          wd[c / 2 + 1] = pack_bf16x2(db.x, db.y);
        }
        // P^T (bf16 pairs): query q of the block -> column q / 2 of the S^T_i buffer. Half 0 packs over
        // its own, already loaded columns; half 1 over half 0's columns [32, 64), once half 0 has
        // loaded them (pair barrier; half 0 arrives right after its second S^T load)
        if (half == 1 && sub == 0) {
          named_bar_sync(2 + qd, 64);
          tc_fence_after();
        }
        tmem_st16(sbuf + 32 * half + 16 * sub + lane_off, wp);
        // dS^T (scaled) -> smem tile i % 2 (once dK_{i-2} / dQ_{i-2} have read it): row krow of query
        // panel `half`, 16-byte chunks 4 sub .. 4 sub + 3
        if (sub == 0 && i >= 2) mbar_wait(&ds_free[i & 1], ((i - 2) >> 1) & 1);
        uint8_t* ds_row = ds_rows + (i & 1) * C::kDSBytes;
#pragma unroll
        for (int c = 0; c < (TT_EXP_BWD == 1 ? 0 : 4); ++c)
          *reinterpret_cast<uint4*>(ds_row + (((4 * sub + c) ^ (krow & 7)) * 16)) =
              make_uint4(wd[4 * c], wd[4 * c + 1], wd[4 * c + 2], wd[4 * c + 3]);
      }
      tmem_st_wait();
      fence_proxy_async_smem();  // dS^T generic-proxy stores -> visible to the tensor core (async proxy)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[i & 1]);
      if (lane == 0 && warp == 8) TT_TR(4, i);
      if (lane == 0 && warp == 12) TT_TR(7, i);
    }
    mbar_wait(acc_done, 0);
    tc_fence_after();
    if (warp == 8 && lane == 0) TT_TR(2, kTrBlocksLast);
    float* dkr = (own ? p.dk : p.dk_pre) + static_cast<long>(kv0 + krow) * p.lddkv + h * DH;
    float* dvr = (own ? p.dv : p.dv_pre) + static_cast<long>(kv0 + krow) * p.lddkv + h * DH;
    const bool direct = it2.y == 2 && p.kv16 != nullptr;
    __nv_bfloat16* k16 = direct ? p.kv16 + static_cast<long>(kv0 + krow - p.r0) * p.ldkv16 + h * DH : nullptr;
#pragma unroll
    for (int c = half * (DH / 2); c < (half + 1) * (DH / 2); c += 16) {
      uint32_t rk[16], rv[16];
      tmem_ld16(t_dK + c + lane_off, rk);
      tmem_ld16(t_dV + c + lane_off, rv);
      tmem_ld_wait();
      if (key_ok && direct) {  // the row's only writer: bf16 straight into the packed operand
        uint32_t wk[8], wv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          wk[e] = pack_bf16x2(__uint_as_float(rk[2 * e]), __uint_as_float(rk[2 * e + 1]));  // scale is in dS
          wv[e] = pack_bf16x2(__uint_as_float(rv[2 * e]), __uint_as_float(rv[2 * e + 1]));
        }
        uint4* pk = reinterpret_cast<uint4*>(k16 + c);
        uint4* pv = reinterpret_cast<uint4*>(k16 + p.H * DH + c);
        pk[0] = make_uint4(wk[0], wk[1], wk[2], wk[3]);
        pk[1] = make_uint4(wk[4], wk[5], wk[6], wk[7]);
        pv[0] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        pv[1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
      } else if (key_ok) {
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          red_add_v4_f32(dkr + c + e, __uint_as_float(rk[e]), __uint_as_float(rk[e + 1]), __uint_as_float(rk[e + 2]),
                         __uint_as_float(rk[e + 3]));
          red_add_v4_f32(dvr + c + e, __uint_as_float(rv[e]), __uint_as_float(rv[e + 1]), __uint_as_float(rv[e + 2]),
                         __uint_as_float(rv[e + 3]));
        }
      }
    }
  }
  pdl_trigger_late();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    TT_TR(3, kTrBlocksLast);
#if TT_TRACE
    if (blockIdx.y == 0 && blockIdx.x < kTrCtas) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_tt_trace[blockIdx.x][kTrBlocksLast][4] = smid;
      g_tt_trace[blockIdx.x][kTrBlocksLast][5] = nq;
    }
#endif
  }
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ============================================================ fused dQ / dK / dV kernel, dh = 128
// Same schedule as the dh = 64 kernel with 64-query blocks: per (128-key block, query block i)
//   warp 1      S^T_i = K Q_i^T, dP^T_i = V dO_i^T          (SS, M = 128 keys, N = 64 queries)
//   warps 8-15  P^T / dS^T once: P^T back into TMEM (bf16 pairs, each softmax half into columns it
//               loaded itself: [0, 16) / [32, 48) of the S^T_i buffer), dS^T into a 16 KB smem tile
//   warp 2      dV += P^T_i dO_i (TS, N = 128), dQ^T_i = K^T dS^T_i (SS: A = K read MN-major, M = dh,
//               B = dS^T MN-major, N = 64 queries) into its own TMEM, dK += dS^T_i Q_i (SS, N = 128)
//   warps 4-7   dQ^T_i drain: lane = dh column, 64 query values -> swizzled smem rows -> two
//               cp.reduce.async.bulk .add per warp into the fp32 dQ accumulator
//   warp 0      TMA: K, V once (two 64-column panels each); Q_i / dO_i through an NS-stage ring
// TMEM (512): S^T[2] [0, 128), dP^T [128, 192), dQ^T [192, 256), dK [256, 384), dV [384, 512).
// dQ^T has its own columns, so S^T_{i+2} waits only for dV_i (the last reader of P^T_i).
template <int NS>
struct Fused128Cfg {
  static constexpr int DH = 128, BKV = 128, BQ = 64;
  static constexpr int kKVBytes = BKV * DH * 2;        // 32 KB: two 16 KB panels (dh 0-63, 64-127)
  static constexpr int kKVPanel = BKV * 128;
  static constexpr int kQBytes = BQ * DH * 2;          // 16 KB: two 8 KB panels
  static constexpr int kQPanel = BQ * 128;
  static constexpr int kOffV = kKVBytes;
  static constexpr int kOffQ = 2 * kKVBytes;
  static constexpr int kOffDO = kOffQ + NS * kQBytes;
  static constexpr int kDSBytes = BKV * BQ * 2;        // dS^T tile: [128 keys][64 queries] bf16 = 16 KB
  static constexpr int kOffDS = kOffDO + NS * kQBytes;
  static constexpr int kOffDQ = kOffDS + 2 * kDSBytes;  // dQ^T staging: 4 warps x (64 q x 32 dh fp32)
  static constexpr int kOffStat = kOffDQ + 4 * 8192;   // [2][2][BQ] floats: lse2, -scale D
  static constexpr int kOffBar = kOffStat + 2 * 2 * BQ * 4;
  static constexpr int kSmem = kOffBar + 256 + 1024;
  static_assert(kSmem <= 227 * 1024 && NS >= 2, "fused dh-128 attention backward: smem / ring");
  static constexpr uint32_t kIdescS = make_idesc_bf16(128, BQ, false, false);   // S^T, dP^T
  static constexpr uint32_t kIdescKV = make_idesc_bf16(128, DH, false, true);   // dV (TS), dK (A K-major)
  static constexpr uint32_t kIdescQ = make_idesc_bf16(128, BQ, true, true);     // dQ^T (A = K MN-major)
};

template <int NS>
__global__ void __launch_bounds__(kThreadsFused, 1)
    fa_bwd_fused128_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                           const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                           const __grid_constant__ CUtensorMap tm_dq, BwdParams p) {
  using C = Fused128Cfg<NS>;
  constexpr int DH = C::DH, BQ = C::BQ;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;
  uint64_t* q_empty = q_full + NS;  // dV/dK_i done: the Q/dO stage is free
  uint64_t* s_full = q_empty + NS;  // [2]
  uint64_t* p_full = s_full + 2;    // [2] softmax done with block i
  uint64_t* dp_full = p_full + 2;
  uint64_t* dp_free = dp_full + 1;
  uint64_t* ds_free = dp_free + 1;  // [2] dQ^T_i / dK_i done: dS^T tile i % 2 may be rewritten
  uint64_t* p_used = ds_free + 2;   // [2] dV_i done: S^T buffer i % 2 may take S^T_{i+2}
  uint64_t* dq_full = p_used + 2;   // dQ^T_i in TMEM (single buffer)
  uint64_t* dq_free = dq_full + 1;  // dQ^T_i read out
  uint64_t* acc_done = dq_free + 1;
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
    tma_prefetch_desc(&tm_dq);
    mbar_init(kv_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], kSmxWarps);
      mbar_init(&ds_free[s], 1);
      mbar_init(&p_used[s], 1);
    }
    mbar_init(dp_full, 1);
    mbar_init(dp_free, kSmxWarps);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 4);
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // predecessor grid complete (launch.cuh); TMEM held before the successor may start
  pdl_trigger_early();
  const uint32_t t_S = tmem, t_dP = tmem + 128, t_dQ = tmem + 192, t_dK = tmem + 256, t_dV = tmem + 384;
  const int wg = warp >> 2;

  if (wg == 0) {
    if (warp == 0 && lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * C::kKVBytes);
#pragma unroll
      for (int pn = 0; pn < 2; ++pn) {
        tma_load_2d(&tm_k, kv_full, smem + pn * C::kKVPanel, h * DH + pn * 64, kv0);
        tma_load_2d(&tm_v, kv_full, smem + C::kOffV + pn * C::kKVPanel, h * DH + pn * 64, kv0);
      }
      for (int i = 0; i < nq; ++i) {
        const int st = i % NS;
        mbar_wait(&q_empty[st], ((i / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[st], 2 * C::kQBytes);
        const int q0 = q_lo + i * BQ;
#pragma unroll
        for (int pn = 0; pn < 2; ++pn) {
          tma_load_2d(&tm_q, &q_full[st], smem + C::kOffQ + st * C::kQBytes + pn * C::kQPanel, h * DH + pn * 64, q0);
          tma_load_2d(&tm_do, &q_full[st], smem + C::kOffDO + st * C::kQBytes + pn * C::kQPanel, h * DH + pn * 64, q0);
        }
      }
    } else if (warp == 1) {
      const uint64_t d16 = make_sdesc_sw128(smem_u32(smem), 16, 1024);  // K-major tiles
      mbar_wait(kv_full, 0);
      for (int i = 0; i < nq; ++i) {
        const int st = i % NS;
        if (i >= 2) mbar_wait(&p_used[i & 1], ((i - 2) >> 1) & 1);
        mbar_wait(&q_full[st], (i / NS) & 1);
        tc_fence_after();
        const uint32_t q_off = C::kOffQ + st * C::kQBytes, do_off = C::kOffDO + st * C::kQBytes;
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < DH / 16; ++k) {
            const uint32_t ao = (k / 4) * C::kKVPanel + (k % 4) * 32, bo = (k / 4) * C::kQPanel + (k % 4) * 32;
            umma_bf16_ss(t_S + (i & 1) * BQ, sdesc_add(d16, ao), sdesc_add(d16, q_off + bo), C::kIdescS, k > 0);
          }
          umma_commit(&s_full[i & 1]);
        }
        __syncwarp();
        if (i >= 1) mbar_wait(dp_free, (i - 1) & 1);
        tc_fence_after();
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < DH / 16; ++k) {
            const uint32_t ao = (k / 4) * C::kKVPanel + (k % 4) * 32, bo = (k / 4) * C::kQPanel + (k % 4) * 32;
            umma_bf16_ss(t_dP, sdesc_add(d16, C::kOffV + ao), sdesc_add(d16, do_off + bo), C::kIdescS, k > 0);
          }
          umma_commit(dp_full);
        }
        __syncwarp();
      }
    } else if (warp == 2) {
      // dV += P^T_i dO_i ; dQ^T_i = K^T dS^T_i ; dK += dS^T_i Q_i
      const uint64_t dmn = make_sdesc_sw128(smem_u32(smem), C::kQPanel, 1024);        // Q_i / dO_i MN-major (N = dh)
      const uint64_t dkmn = make_sdesc_sw128(smem_u32(smem), C::kKVPanel, 1024);      // K read MN-major (M = dh)
      const uint64_t dsk = make_sdesc_sw128(smem_u32(smem + C::kOffDS), 16, 1024);     // dS^T, K-major A
      const uint64_t dsm = make_sdesc_sw128(smem_u32(smem + C::kOffDS), C::kDSBytes, 1024);  // dS^T, MN-major B
      for (int i = 0; i < nq; ++i) {
        mbar_wait(&p_full[i & 1], (i >> 1) & 1);
        if (i >= 1) mbar_wait(dq_free, (i - 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          const int st = i % NS;
          const uint32_t q_off = C::kOffQ + st * C::kQBytes, do_off = C::kOffDO + st * C::kQBytes;
          const uint32_t ds_off = (i & 1) * C::kDSBytes;
#pragma unroll
          for (int k = 0; k < BQ / 16; ++k)  // 16 queries per step; P^T of queries 32-63 sits at column 32
            umma_bf16_ts(t_dV, t_S + (i & 1) * BQ + (k < 2 ? 8 * k : 32 + 8 * (k - 2)),
                         sdesc_add(dmn, do_off + k * 2048), C::kIdescKV, (i > 0 || k > 0));
          umma_commit(&p_used[i & 1]);
#pragma unroll
          for (int k = 0; k < C::BKV / 16; ++k)  // 16 keys per step
            umma_bf16_ss(t_dQ, sdesc_add(dkmn, k * 2048), sdesc_add(dsm, ds_off + k * 2048), C::kIdescQ, k > 0);
          umma_commit(dq_full);
#pragma unroll
          for (int k = 0; k < BQ / 16; ++k)
            umma_bf16_ss(t_dK, sdesc_add(dsk, ds_off + k * 32), sdesc_add(dmn, q_off + k * 2048), C::kIdescKV,
                         (i > 0 || k > 0));
          umma_commit(&q_empty[st]);
          umma_commit(&ds_free[i & 1]);
          if (i == nq - 1) umma_commit(acc_done);
        }
        __syncwarp();
      }
    }
  } else if (wg == 1) {
    // dQ^T drain: warp w reads TMEM lanes (dh columns) 32 (w % 4) .. +31, 64 query values each
    const int qd = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(qd * 32) << 16;
    uint8_t* stage = smem + C::kOffDQ + qd * 8192;  // [64 query rows][32 dh] fp32, 128-byte swizzled rows
    for (int i = 0; i < nq; ++i) {
      const int q0 = q_lo + i * BQ;
      mbar_wait(dq_full, i & 1);
      tc_fence_after();
      uint32_t r[64];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t t[16];
        tmem_ld16(t_dQ + 16 * c + lane_off, t);
#pragma unroll
        for (int e = 0; e < 16; ++e) r[16 * c + e] = t[e];
      }
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_free);
      if (lane == 0) bulk_wait_read0();  // the previous block's reduces have read the staging rows
      __syncwarp();
#pragma unroll
      for (int q = 0; q < BQ; ++q)  // row q: this lane's dh column
        *reinterpret_cast<uint32_t*>(stage + q * 128 + (((lane >> 2) ^ (q & 7)) * 16) + (lane & 3) * 4) = r[q];
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_reduce_add_2d(&tm_dq, stage, h * DH + 32 * qd, q0);
        tma_reduce_add_2d(&tm_dq, stage + 32 * 128, h * DH + 32 * qd, q0 + 32);
        bulk_commit();
      }
      __syncwarp();
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  } else {
    const int qd = warp & 3;
    const int half = (warp - 8) >> 2;   // query columns [32 half, 32 half + 32) of each block
    const int krow = qd * 32 + lane;    // key row within the block == TMEM lane
    const bool key_ok = krow < kv_rows;
    const int kt = kt_base + krow;
    const uint32_t lane_off = static_cast<uint32_t>(qd * 32) << 16;
    const int tid = threadIdx.x - 256;  // 0..255
    uint8_t* ds_rows = smem + C::kOffDS + krow * 128;
    float nl = INFINITY, nd = 0.f;
    auto fetch = [&](int i) {
      const int q = q_lo + i * BQ + tid;
      const bool ok = tid < BQ && i < nq && q < q_hi;
      nl = ok ? p.lse[static_cast<long>(h) * p.n + q] : INFINITY;
      nd = ok ? p.D[static_cast<long>(h) * p.n + q] : 0.f;
    };
    fetch(0);
    const float c2 = p.scale_log2, sc = p.scale;
    for (int i = 0; i < nq; ++i) {
      const int q0 = q_lo + i * BQ;
      float* st_lse = stat + (i & 1) * 2 * BQ;
      float* st_nd = st_lse + BQ;
      if (tid < BQ) {
        st_lse[tid] = nl * kLog2e;
        st_nd[tid] = -nd * sc;
      }
      named_bar_sync(1, 32 * kSmxWarps);
      fetch(i + 1);
      const int col0 = 32 * half;
      const int vis0 = own ? kt - (q0 - seg_off) : 0;  // first visible block column of this key
      mbar_wait(&s_full[i & 1], (i >> 1) & 1);
      mbar_wait(dp_full, i & 1);
      tc_fence_after();
      const uint32_t sbuf = t_S + (i & 1) * BQ;
      float sv[32], dp[32];
      {
        uint32_t r[16], r2[16], r3[16], r4[16];
        tmem_ld16(sbuf + col0 + lane_off, r);
        tmem_ld16(sbuf + col0 + 16 + lane_off, r2);
        tmem_ld16(t_dP + col0 + lane_off, r3);
        tmem_ld16(t_dP + col0 + 16 + lane_off, r4);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          sv[e] = __uint_as_float(r[e]);
          sv[16 + e] = __uint_as_float(r2[e]);
          dp[e] = __uint_as_float(r3[e]);
          dp[16 + e] = __uint_as_float(r4[e]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dp_free);  // dP^T_i in registers: dP^T_{i+1} may overwrite it
      {
        const int lo = key_ok ? vis0 - col0 : 32;
        if (__any_sync(0xffffffff, lo > 0)) {
#pragma unroll
          for (int c = 0; c < 32; ++c) sv[c] = c >= lo ? sv[c] : -INFINITY;
        }
      }
      uint32_t wp[16], wd[16];
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        const float4 lz = *reinterpret_cast<const float4*>(st_lse + col0 + c);
        const float4 dz = *reinterpret_cast<const float4*>(st_nd + col0 + c);
        const float2 c22 = make_float2(c2, c2), sc2 = make_float2(sc, sc);
        const float2 xa = __ffma2_rn(make_float2(sv[c], sv[c + 1]), c22, make_float2(-lz.x, -lz.y));
        const float2 xb = __ffma2_rn(make_float2(sv[c + 2], sv[c + 3]), c22, make_float2(-lz.z, -lz.w));
        const float2 pa = make_float2(ex2_approx(xa.x), ex2_approx(xa.y));
        const float2 pb = make_float2(ex2_approx(xb.x), ex2_approx(xb.y));
        const float2 da = __fmul2_rn(pa, __ffma2_rn(make_float2(dp[c], dp[c + 1]), sc2, make_float2(dz.x, dz.y)));
        const float2 db = __fmul2_rn(pb, __ffma2_rn(make_float2(dp[c + 2], dp[c + 3]), sc2, make_float2(dz.z, dz.w)));
        wp[c / 2] = pack_bf16x2(pa.x, pa.y);
        wp[c / 2 + 1] = pack_bf16x2(pb.x, pb.y);
        wd[c / 2] = pack_bf16x2(da.x, da.y);
        wd[c / 2 + 1] = pack_bf16x2(db.x, db.y);
      }
      // P^T (bf16 pairs) into 16 columns this warp loaded itself: [0, 16) (half 0) / [32, 48) (half 1)
      tmem_st16(sbuf + col0 + lane_off, wp);
      // dS^T (scaled) -> smem tile i % 2 (once dK_{i-2} / dQ^T_{i-2} have read it): row krow, 16-byte
      // chunks 4 half .. 4 half + 3 of the 128-byte (64-query) row
      if (i >= 2) mbar_wait(&ds_free[i & 1], ((i - 2) >> 1) & 1);
      uint8_t* ds_row = ds_rows + (i & 1) * C::kDSBytes;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<uint4*>(ds_row + (((4 * half + c) ^ (krow & 7)) * 16)) =
            make_uint4(wd[4 * c], wd[4 * c + 1], wd[4 * c + 2], wd[4 * c + 3]);
      tmem_st_wait();
      fence_proxy_async_smem();  // dS^T generic-proxy stores -> visible to the tensor core (async proxy)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[i & 1]);
    }
    mbar_wait(acc_done, 0);
    tc_fence_after();
    float* dkr = (own ? p.dk : p.dk_pre) + static_cast<long>(kv0 + krow) * p.lddkv + h * DH;
    float* dvr = (own ? p.dv : p.dv_pre) + static_cast<long>(kv0 + krow) * p.lddkv + h * DH;
    const bool direct = it2.y == 2 && p.kv16 != nullptr;
    __nv_bfloat16* k16 = direct ? p.kv16 + static_cast<long>(kv0 + krow - p.r0) * p.ldkv16 + h * DH : nullptr;
#pragma unroll
    for (int c = half * (DH / 2); c < (half + 1) * (DH / 2); c += 16) {
      uint32_t rk[16], rv[16];
      tmem_ld16(t_dK + c + lane_off, rk);
      tmem_ld16(t_dV + c + lane_off, rv);
      tmem_ld_wait();
      if (key_ok && direct) {  // the row's only writer: bf16 straight into the packed operand
        uint32_t wk[8], wv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          wk[e] = pack_bf16x2(__uint_as_float(rk[2 * e]), __uint_as_float(rk[2 * e + 1]));  // scale is in dS
          wv[e] = pack_bf16x2(__uint_as_float(rv[2 * e]), __uint_as_float(rv[2 * e + 1]));
        }
        uint4* pk = reinterpret_cast<uint4*>(k16 + c);
        uint4* pv = reinterpret_cast<uint4*>(k16 + p.H * DH + c);
        pk[0] = make_uint4(wk[0], wk[1], wk[2], wk[3]);
        pk[1] = make_uint4(wk[4], wk[5], wk[6], wk[7]);
        pv[0] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        pv[1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
      } else if (key_ok) {
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          red_add_v4_f32(dkr + c + e, __uint_as_float(rk[e]), __uint_as_float(rk[e + 1]), __uint_as_float(rk[e + 2]),
                         __uint_as_float(rk[e + 3]));
          red_add_v4_f32(dvr + c + e, __uint_as_float(rv[e]), __uint_as_float(rv[e + 1]), __uint_as_float(rv[e + 2]),
                         __uint_as_float(rv[e + 3]));
        }
      }
    }
  }
  pdl_trigger_late();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// D[h][r] = rowsum(dO * O) over head h's dh columns (the softmax-backward correction term): one
// thread per 8 columns (16-byte loads), a group of dh/8 lanes per (row, head) reduces with shuffles.
// The same thread zeroes its 8 columns of the fp32 dQ accumulator the fused kernel reduces into (no
// separate memset between the two launches).
__global__ void attn_bwd_pre_kernel(const __nv_bfloat16* __restrict__ dO, const __nv_bfloat16* __restrict__ O,
                                    long ld, float* __restrict__ D, float* __restrict__ dq, long lddq, int n, int H,
                                    int dh) {
  pdl_wait();
  pdl_trigger();
  const long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int gpr = dh / 8;  // threads per (row, head): 8 or 16
  const int cols8 = H * gpr;
  const long r = t / cols8;
  const int j = static_cast<int>(t - r * cols8);
  float s = 0.f;
  if (r < n) {
    float4* z = reinterpret_cast<float4*>(dq + r * lddq + j * 8);
    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    const uint4 x = *reinterpret_cast<const uint4*>(dO + r * ld + j * 8);
    const uint4 y = *reinterpret_cast<const uint4*>(O + r * ld + j * 8);
    const __nv_bfloat162* xa = reinterpret_cast<const __nv_bfloat162*>(&x);
    const __nv_bfloat162* ya = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 p = __bfloat1622float2(xa[i]), q = __bfloat1622float2(ya[i]);
      s += p.x * q.x + p.y * q.y;
    }
  }
  for (int o = gpr / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  if (r < n && (j % gpr) == 0) D[static_cast<long>(j / gpr) * n + r] = s;
}

// dh = 64: the fused kernel; dQ partials are reduced into a.dq (fp32 [n x lddq], zeroed by the D pre-pass)
void launch_bwd_fused(const AttnBwdArgs& a, long rows_cap, const int4* kv_items, const int2* kv_items2, int n_kv,
                      cudaStream_t stream) {
#ifndef TT_EXP_BWD_NS
#define TT_EXP_BWD_NS 3  // Q / dO ring depth (experiment builds may change it)
#endif
  constexpr int NS = TT_EXP_BWD_NS;
  using C = FusedCfg<NS>;
  if (n_kv <= 0) return;
  if (!a.dq) throw std::invalid_argument("fused attention backward: needs the fp32 dQ accumulator");
  const int d = a.H * 64;
  CUtensorMap tq, tdo, tk, tv, tdq;
  make_tmap_bf16(&tq, a.q, d, a.n, a.ldq, 64, 128);
  make_tmap_bf16(&tdo, a.dO, d, a.n, a.ldq, 64, 128);
  make_tmap_bf16(&tk, a.k, d, rows_cap, a.ldkv, 64, 128);
  make_tmap_bf16(&tv, a.v, d, rows_cap, a.ldkv, 64, 128);
  make_tmap_f32_sw128(&tdq, a.dq, d, a.n, a.lddq);
  BwdParams p{a.lse, a.D, a.dq, a.lddq, a.dk, a.dv, a.lddkv, a.dk_pre ? a.dk_pre : a.dk,
              a.dv_pre ? a.dv_pre : a.dv, a.n, a.S, a.H, a.pbase, a.r0 < 0 ? a.S : a.r0, kv_items, kv_items2, a.scale,
              a.scale * kLog2e, a.dkv16, a.lddkv16};
  ensure_smem_attr(reinterpret_cast<const void*>(fa_bwd_fused_kernel<NS>), C::kSmem);
  launch_k(fa_bwd_fused_kernel<NS>, dim3(n_kv, a.H), dim3(kThreadsFused), C::kSmem, stream, tq, tdo, tk, tv, tdq, p);
}

// dh = 128: the fused kernel with 64-query blocks; dQ partials reduced into a.dq (fp32, zeroed by the D pre-pass)
void launch_bwd_fused128(const AttnBwdArgs& a, long rows_cap, const int4* kv_items, const int2* kv_items2, int n_kv,
                         cudaStream_t stream) {
  constexpr int NS = 3;
  using C = Fused128Cfg<NS>;
  if (n_kv <= 0) return;
  const int d = a.H * 128;
  CUtensorMap tq, tdo, tk, tv, tdq;
  make_tmap_bf16(&tq, a.q, d, a.n, a.ldq, 64, C::BQ);
  make_tmap_bf16(&tdo, a.dO, d, a.n, a.ldq, 64, C::BQ);
  make_tmap_bf16(&tk, a.k, d, rows_cap, a.ldkv, 64, 128);
  make_tmap_bf16(&tv, a.v, d, rows_cap, a.ldkv, 64, 128);
  make_tmap_f32_sw128(&tdq, a.dq, d, a.n, a.lddq);
  BwdParams p{a.lse, a.D, a.dq, a.lddq, a.dk, a.dv, a.lddkv, a.dk_pre ? a.dk_pre : a.dk,
              a.dv_pre ? a.dv_pre : a.dv, a.n, a.S, a.H, a.pbase, a.r0 < 0 ? a.S : a.r0, kv_items, kv_items2, a.scale,
              a.scale * kLog2e, a.dkv16, a.lddkv16};
  ensure_smem_attr(reinterpret_cast<const void*>(fa_bwd_fused128_kernel<NS>), C::kSmem);
  launch_k(fa_bwd_fused128_kernel<NS>, dim3(n_kv, a.H), dim3(kThreadsFused), C::kSmem, stream, tq, tdo, tk, tv, tdq, p);
}

}  // namespace

#if TT_TRACE
extern "C" int tt_debug_trace_read(long long* out, long n) {
  const long cap = static_cast<long>(kTrCtas) * kTrBlocks * kTrEv;
  if (n > cap) n = cap;
  return cudaMemcpyFromSymbol(out, g_tt_trace, n * sizeof(long long)) == cudaSuccess ? 0 : 1;
}
extern "C" int tt_debug_trace_clear() {
  static long long zeros[kTrCtas][kTrBlocks][kTrEv];
  return cudaMemcpyToSymbol(g_tt_trace, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 1;
}
#endif

void attn_bwd_pre(const AttnBwdArgs& a, cudaStream_t stream) {
  const long threads = static_cast<long>(a.n) * a.H * (a.dh / 8);
  if (a.ldq % 8 != 0) throw std::invalid_argument("attention backward: dO/O pitch must be a multiple of 8");
  if (!a.dq || a.lddq % 4 != 0 || a.lddq < static_cast<long>(a.H) * a.dh)
    throw std::invalid_argument("attention backward: dQ accumulator missing or its pitch not a multiple of 4");
  if (threads > 0)
    launch_k(attn_bwd_pre_kernel, dim3(static_cast<unsigned>((threads + 255) / 256)), dim3(256), 0, stream, a.dO, a.o,
             a.ldq, a.D, a.dq, a.lddq, a.n, a.H, a.dh);
}

void attn_bwd_sm100(const AttnBwdArgs& a, long rows_cap, const int4* kv_items, const int2* kv_items2, int n_kv,
                    cudaStream_t stream) {
  attn_bwd_pre(a, stream);
  if (a.dh == 64) return launch_bwd_fused(a, rows_cap, kv_items, kv_items2, n_kv, stream);
  if (a.dh == 128) return launch_bwd_fused128(a, rows_cap, kv_items, kv_items2, n_kv, stream);
  throw std::invalid_argument("attention: head_dim must be 64 or 128");
}

}  // namespace ttb
