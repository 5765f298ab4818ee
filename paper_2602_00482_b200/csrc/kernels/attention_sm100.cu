// tcgen05 / TMEM / TMA segment attention forward over the device KV stack (sm_100a).
//
// Replaces detail::attention_probs + the PV loop (model.hpp:298-321, 386-408). One CTA = one
// (128-query block of one segment, head). Keys are the stack prefix rows [0, S) (full) followed by
// the segment's own rows (causal); no tree mask is materialised.
//
// Roles (192 threads):
//   warp 0      TMA producer: Q once, then K/V blocks into an NS-stage ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//                 S_j = Q K_j^T  (M=128, N=BKV, K=dh)  -> TMEM S[j%2]   (fp32)
//                 O  += P_j V_j  (M=128, N=dh,  K=BKV) -> TMEM O        (fp32)
//   warps 2..5  softmax, one query row per thread (TMEM lane): online max/sum in the log2 domain,
//               P_j (bf16) into 128B-swizzled smem (the UMMA K-major A layout), O rescale in TMEM
// Barriers: q_full, kv_full/kv_empty[NS], s_full[2], p_full[2], pv_done.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <stdexcept>

#include "attention.h"
#include "gemm.h"
#include "launch.cuh"
#include "sm100.cuh"

#ifndef TT_TRACE
#define TT_TRACE 0
#endif
// Resource experiments (tools/attn_fwd_ab.sh builds only; timings, not results): 1 no exponentials
// (p = x), 2 no P store to TMEM, 3 no PV MMAs, 4 no row max (base 0)
#ifndef TT_EXP_FWD
#define TT_EXP_FWD 0
#endif
#if TT_TRACE
// pipeline trace of the forward (debug library only, -DTT_TRACE=1): [cta][block][event] clock64
constexpr int kFTrCtas = 64, kFTrBlocks = 32, kFTrEv = 8;
__device__ long long g_tt_ftrace[kFTrCtas][kFTrBlocks][kFTrEv];
__device__ long long g_tt_fcta[kFTrCtas][4];  // start, all warps past setup, softmax done, end
#define TT_FCTA(ev)                                                                      \
  do {                                                                                   \
    if (blockIdx.y == 0 && blockIdx.x < kFTrCtas) g_tt_fcta[blockIdx.x][(ev)] = clock64(); \
  } while (0)
extern "C" int tt_debug_fcta_read(long long* out) {
  return cudaMemcpyFromSymbol(out, g_tt_fcta, sizeof(g_tt_fcta)) == cudaSuccess ? 0 : 1;
}
#define TT_FTR(ev, j)                                                                                      \
  do {                                                                                                     \
    if (blockIdx.y == 0 && blockIdx.x < kFTrCtas && (j) < kFTrBlocks) g_tt_ftrace[blockIdx.x][(j)][(ev)] = clock64(); \
  } while (0)
extern "C" int tt_debug_ftrace_read(long long* out, long n) {
  const long cap = static_cast<long>(kFTrCtas) * kFTrBlocks * kFTrEv;
  if (n > cap) n = cap;
  return cudaMemcpyFromSymbol(out, g_tt_ftrace, n * sizeof(long long)) == cudaSuccess ? 0 : 1;
}
#else
#define TT_FTR(ev, j) \
  do {                \
  } while (0)
#define TT_FCTA(ev) \
  do {              \
  } while (0)
#endif

namespace ttb {

namespace {

constexpr int kBQ = 128;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
constexpr float kRescaleThreshold = 8.0f;  // log2 units: P stays <= 256
__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// SPL softmax warps per TMEM lane quadrant, each owning BKV / SPL columns of S_j with its own running
// max / sum and its own O accumulator. Warp 0 TMA, warp 1 S-MMA issuer, warps 2 .. 2 + 4 SPL - 1
// softmax, warp 2 + 4 SPL PV-MMA issuer.
template <int DH, int BKV, int NS, int SPL>
struct FwdCfg {
  static constexpr int kSmxWarps = 4 * SPL;
  static constexpr int kPvWarp = 2 + kSmxWarps;
  static constexpr int kThreads = 32 * (kPvWarp + 1);
  static constexpr int HC = BKV / SPL;  // S columns per softmax warp
  // S / P TMEM buffers: the S issuer runs NB-1 blocks ahead of the softmax (TMEM: NB S buffers + SPL O)
  static constexpr int NB = SPL == 2 ? 3 : 2;
  static constexpr int kQBytes = kBQ * DH * 2;
  static constexpr int kKVBytes = BKV * DH * 2;           // one K (or V) tile
  static constexpr int kOffK = kQBytes;
  static constexpr int kOffV = kOffK + NS * kKVBytes;
  static constexpr int kOffX = kOffV + NS * kKVBytes;  // end-of-row combine: per-split running max and sum
  static constexpr int kOffBar = kOffX + 2 * SPL * kBQ * 4;  // [m_0 .. m_SPL-1, l_0 .. l_SPL-1] x 128 rows
  static constexpr int kSmem = kOffBar + 256 + 1024;
  static constexpr int kOCol = (NB * BKV + DH - 1) / DH * DH;
  // SPL O accumulators (one per softmax split, each on its own running max): kOCol + s DH
  static constexpr int kTmemCols = (kOCol + SPL * DH) <= 256 ? 256 : 512;
  static_assert(kOCol + SPL * DH <= 512 && NS >= NB, "fwd kernel: TMEM / K-V ring too small");
  static_assert(HC % 32 == 0, "fwd kernel: 32-column multiples per softmax warp");
  static constexpr uint32_t kIdescS = make_idesc_bf16(128, BKV, false, false);
  static constexpr uint32_t kIdescO = make_idesc_bf16(128, DH, false, true);
};

struct FwdParams {
  __nv_bfloat16* o;
  long ldo;
  float* lse;
  int n, S, H;
  int pbase, r0;  // prefix rows [pbase, pbase + S); own rows from r0
  const int4* qblocks;
  float scale_log2;
};

// POLY: of every 4 element pairs, how many take 2^x on the FMA pipe (ex2_poly2) instead of MUFU:
// at dh=64 one exponential per 4*dh MMA FLOPs makes the MUFU (16/clk/SM) the bottleneck.
template <int DH, int BKV, int NS, int POLY, int SPL>
__global__ void __launch_bounds__(FwdCfg<DH, BKV, NS, SPL>::kThreads, 1)
    fa_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, FwdParams p) {
  using C = FwdCfg<DH, BKV, NS, SPL>;
  constexpr int kSmxWarps = C::kSmxWarps;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* q_full = bars;
  // separate K and V rings: a K slot frees when S_j completes, a V slot when PV_j does, so the
  // loads for S_{j+NB} never wait on the PV MMA just issued
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + NS;
  uint64_t* v_full = k_empty + NS;
  uint64_t* v_empty = v_full + NS;
  uint64_t* s_full = v_empty + NS;  // [NB]
  uint64_t* p_full = s_full + C::NB;  // [NB]
  // PV_j completion -> pv_done[j % NB]: per-buffer barriers keep the parity waits unambiguous (the
  // softmax may run up to NB-1 PV MMAs ahead of their completion)
  uint64_t* pv_done = p_full + C::NB;  // [NB]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + C::NB);

  const int warp = warp_id_sync();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TT_FCTA(0);
  const int4 blk = p.qblocks[blockIdx.x];
  const int q_start = blk.x, q_end = blk.y, seg_off = blk.z;
  const int h = blockIdx.y;
  const int S = p.S;
  const int n_pre = (S + BKV - 1) / BKV;
  const int own_rows = q_end - seg_off;
  const int n_own = (own_rows + BKV - 1) / BKV;
  const int nblk = n_pre + n_own;
  auto kv_row0 = [&](int j) { return j < n_pre ? p.pbase + j * BKV : p.r0 + seg_off + (j - n_pre) * BKV; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < C::NB; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], kSmxWarps);
      mbar_init(&pv_done[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // predecessor grid complete (launch.cuh); TMEM held before the successor may start
  pdl_trigger_early();
  if (threadIdx.x == 0) TT_FCTA(1);
  constexpr int NB = C::NB;
  const uint32_t tmem_S = tmem;              // NB x BKV columns
  // O (N = DH) at a DH-aligned column (dh 128: 256, not 192)
  const uint32_t tmem_O = tmem + C::kOCol;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, C::kQBytes);
#pragma unroll
      for (int pn = 0; pn < DH / 64; ++pn) tma_load_2d(&tm_q, q_full, smem + pn * (kBQ * 128), h * DH + pn * 64, q_start);
      for (int j = 0; j < nblk; ++j) {
        const int st = j % NS;
        const uint32_t ph = (j / NS) & 1;
        const int r0 = kv_row0(j);
        uint8_t* ks = smem + C::kOffK + st * C::kKVBytes;
        uint8_t* vs = smem + C::kOffV + st * C::kKVBytes;
        mbar_wait(&k_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&k_full[st], C::kKVBytes);
#pragma unroll
        for (int pn = 0; pn < DH / 64; ++pn) tma_load_2d(&tm_k, &k_full[st], ks + pn * (BKV * 128), h * DH + pn * 64, r0);
        mbar_wait(&v_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&v_full[st], C::kKVBytes);
#pragma unroll
        for (int pn = 0; pn < DH / 64; ++pn) tma_load_2d(&tm_v, &v_full[st], vs + pn * (BKV * 128), h * DH + pn * 64, r0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ S issuer
    // S_j = Q K_j^T into TMEM buffer j % NB once PV_{j-NB} (which read P_{j-NB} from it) is done.
    // Two issuing warps (S and PV): an mbarrier wait in an issuing thread costs ~180 clk with MMAs in
    // flight (tools/umma_probe.cu), so each dependency chain gets its own issuer.
    const uint64_t dK16 = make_sdesc_sw128(smem_u32(smem), 16, 1024);  // K-major tiles
    mbar_wait(q_full, 0);
    for (int j = 0; j < nblk; ++j) {
      const int st = j % NS;
      if (j >= NB) mbar_wait(&pv_done[(j - NB) % NB], ((j - NB) / NB) & 1);
      mbar_wait(&k_full[st], (j / NS) & 1);
      tc_fence_after();
      if (lane == 0) {
        TT_FTR(0, j);
        const uint32_t k_off = C::kOffK + st * C::kKVBytes;
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint64_t da = sdesc_add(dK16, (k / 4) * (kBQ * 128) + (k % 4) * 32);
          const uint64_t db = sdesc_add(sdesc_add(dK16, k_off), (k / 4) * (BKV * 128) + (k % 4) * 32);
          umma_bf16_ss(tmem_S + (j % NB) * BKV, da, db, C::kIdescS, k > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[j % NB]);
        umma_commit(&k_empty[st]);
      }
      __syncwarp();
    }
  } else if (warp == C::kPvWarp) {
    // ------------------------------------------------------------------ PV issuer
    // O_h += P_j[:, keys of half h] V_j[keys of half h]: each softmax half runs its own max / sum, so its
    // keys accumulate into their own O (combined once at the end). A = P_j from TMEM (bf16 pairs at
    // columns h*BKV/2 + ...)
    const uint64_t dVmn = make_sdesc_sw128(smem_u32(smem), BKV * 128, 1024);  // V read MN-major
    for (int j = 0; j < nblk; ++j) {
      mbar_wait(&p_full[j % NB], (j / NB) & 1);
      mbar_wait(&v_full[j % NS], (j / NS) & 1);
      tc_fence_after();
      if (lane == 0) {
        TT_FTR(1, j);
        const int st = j % NS;
        const uint32_t v_off = C::kOffV + st * C::kKVBytes;
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          constexpr int KPS = BKV / 16 / SPL;  // k-steps per softmax split
          const int hk = k / KPS, kl = k % KPS;  // split owning these keys, k-step within it
          if (TT_EXP_FWD != 3)
          umma_bf16_ts(tmem_O + hk * DH, tmem_S + (j % NB) * BKV + packed_col<BKV / SPL>(k),
                       sdesc_add(sdesc_add(dVmn, v_off), k * 2048), C::kIdescO, (j > 0 || kl > 0) ? 1u : 0u);
        }
        umma_commit(&v_empty[st]);
        umma_commit(&pv_done[j % NB]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------------ softmax
    // One query row per TMEM lane; the two warps on a lane quadrant split the BKV columns (half) and
    // each keeps its own running max / sum and its own O accumulator (no per-block max exchange);
    // the halves are combined once at the end.
    const int quad = warp & 3;
    const int half = (warp - 2) / 4;  // the column split (0 .. SPL-1)
    const int rloc = quad * 32 + lane;  // row within the tile == TMEM lane
    const int row = q_start + rloc;
    const int t = row - seg_off;        // local query index within the segment
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int bar_id = 2 + quad;
    float* xch = reinterpret_cast<float*>(smem + C::kOffX);
    constexpr int HC = C::HC;
    // m_used: the exponent base actually applied (log2 domain). It only moves when the running max
    // exceeds it by more than kRescaleThreshold (P <= 2^8 then), so O in TMEM is rescaled rarely.
    float m_used = -INFINITY, l = 0.f;
    const float c2 = p.scale_log2;
    for (int j = 0; j < nblk; ++j) {
      if (warp == 2 && lane == 0) TT_FTR(7, j);
      // try_wait first (~90 clk when S_j is already complete, the common case) rather than test_wait
      // (~150 clk; B300_MICROARCH mbarrier latencies): this wait is on every block's critical path
#if TT_EXP_FWD == 5  // experiment builds only: the test_wait-first variant
      mbar_wait_fast(&s_full[j % NB], (j / NB) & 1);
#else
      mbar_wait(&s_full[j % NB], (j / NB) & 1);
#endif
      tc_fence_after();
      if (warp == 2 && lane == 0) TT_FTR(2, j);
      float s[HC];
#pragma unroll
      for (int c = 0; c < HC; c += 16) {
        uint32_t r[16];
        tmem_ld16(tmem_S + (j % NB) * BKV + half * HC + c + lane_off, r);
#pragma unroll
        for (int i = 0; i < 16; ++i) s[c + i] = __uint_as_float(r[i]);
      }
      tmem_ld_wait();
      if (warp == 2 && lane == 0) TT_FTR(3, j);
      const bool pre = j < n_pre;
      // key index of this half's column 0 (prefix row / own local)
      const int base = (pre ? j * BKV : (j - n_pre) * BKV) + half * HC;
      const int lim = pre ? (S - base) : (t - base + 1);   // valid columns are [0, lim)
      if (__any_sync(0xffffffff, lim < HC)) {
#pragma unroll
        for (int i = 0; i < HC; ++i) s[i] = i < lim ? s[i] : -INFINITY;
      }
      // row max as a 3-ary tree (depth 4 at HC = 64 instead of a 32-long dependent chain)
      float mx;
      {
        constexpr int N1 = (HC + 2) / 3;
        float t1[N1];
#pragma unroll
        for (int i = 0; i < N1; ++i)
          t1[i] = fmax3f(s[3 * i], 3 * i + 1 < HC ? s[3 * i + 1] : s[3 * i], 3 * i + 2 < HC ? s[3 * i + 2] : s[3 * i]);
        constexpr int N2 = (N1 + 2) / 3;
        float t2[N2];
#pragma unroll
        for (int i = 0; i < N2; ++i)
          t2[i] = fmax3f(t1[3 * i], 3 * i + 1 < N1 ? t1[3 * i + 1] : t1[3 * i], 3 * i + 2 < N1 ? t1[3 * i + 2] : t1[3 * i]);
        mx = t2[0];
#pragma unroll
        for (int i = 1; i < N2; i += 2) mx = fmax3f(mx, t2[i], i + 1 < N2 ? t2[i + 1] : t2[i]);
      }
      const float m_new = TT_EXP_FWD == 4 ? 0.f : fmaxf(m_used, mx * c2);
      if (warp == 2 && lane == 0) TT_FTR(4, j);
      const bool resc = m_new > m_used + kRescaleThreshold;
      float corr = 1.f;
      if (resc) {
        corr = ex2_approx(m_used - m_new);  // 0 on the first block (m_used = -inf)
        m_used = m_new;
        l *= corr;
      }
      const float mb = m_used == -INFINITY ? 0.f : m_used;
      float2 rs2 = make_float2(0.f, 0.f);
      const float2 c22 = make_float2(c2, c2), nmb2 = make_float2(-mb, -mb);
      // P_j (bf16 pairs) into the first HC/2 columns of this half's OWN S_j columns [half*HC, +HC)
      // (the other half may still be reading its S columns): the A operand of PV_j
      uint32_t w[HC / 2];
#pragma unroll
      for (int cch = 0; cch < HC / 8; ++cch) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          // paired FP32 (FFMA2 / FADD2): x = s*c - m ; p = 2^x ; row sum += p
          const float2 x = __ffma2_rn(make_float2(s[cch * 8 + 2 * e], s[cch * 8 + 2 * e + 1]), c22, nmb2);
          const float2 pe = TT_EXP_FWD == 1 ? x : (e < POLY ? ex2_poly2(x) : make_float2(ex2_approx(x.x), ex2_approx(x.y)));
          rs2 = __fadd2_rn(rs2, pe);
          w[cch * 4 + e] = pack_bf16x2(pe.x, pe.y);
        }
      }
      if (warp == 2 && lane == 0) TT_FTR(5, j);
#pragma unroll
      for (int c = 0; c < (TT_EXP_FWD == 2 ? 0 : HC / 2); c += 16)
        tmem_st16(tmem_S + (j % NB) * BKV + half * HC + c + lane_off, *reinterpret_cast<uint32_t(*)[16]>(&w[c]));
      const float rs = rs2.x + rs2.y;
      l += rs;
      if (j > 0 && __any_sync(0xffffffff, resc)) {
        // O_half (from PV_{j-1}) must be final before this warp rescales it
        mbar_wait(&pv_done[(j - 1) % NB], ((j - 1) / NB) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < DH; c += 16) {
          uint32_t r[16];
          tmem_ld16(tmem_O + half * DH + c + lane_off, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * corr);
          tmem_st16(tmem_O + half * DH + c + lane_off, r);
        }
      }
      tmem_st_wait();  // P (and any O rescale) in TMEM before the PV issuer is released
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[j % NB]);
      if (lane == 0 && warp == 2) TT_FTR(6, j);

    }
    if (warp == 2 && lane == 0) TT_FCTA(2);
    // combine the splits: m = max_s m_s; l = sum_s l_s 2^(m_s - m); O = sum_s O_s 2^(m_s - m) / l
    float* lb = xch;
    lb[half * kBQ + rloc] = m_used;
    lb[(SPL + half) * kBQ + rloc] = l;
    named_bar_sync(bar_id, 32 * SPL);
    float ms[SPL], ls[SPL];
    float m = -INFINITY;
#pragma unroll
    for (int q = 0; q < SPL; ++q) {
      ms[q] = lb[q * kBQ + rloc];
      ls[q] = lb[(SPL + q) * kBQ + rloc];
      m = fmaxf(m, ms[q]);
    }
    float lt = 0.f, f[SPL];
#pragma unroll
    for (int q = 0; q < SPL; ++q) {
      f[q] = ms[q] == -INFINITY ? 0.f : ex2_approx(ms[q] - m);
      lt += ls[q] * f[q];
    }
    mbar_wait(&pv_done[(nblk - 1) % NB], ((nblk - 1) / NB) & 1);
    tc_fence_after();
    const float inv_l = 1.f / lt;
#pragma unroll
    for (int q = 0; q < SPL; ++q) f[q] *= inv_l;
    // tcgen05.ld is .sync.aligned: every lane executes it (convergently); only valid rows store.
    const bool row_ok = row < q_end;
    __nv_bfloat16* orow = p.o + static_cast<long>(row) * p.ldo + h * DH;
#pragma unroll
    for (int c = half * (DH / SPL); c < (half + 1) * (DH / SPL); c += 16) {
      float o[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] = 0.f;
#pragma unroll
      for (int q = 0; q < SPL; ++q) {
        uint32_t r[16];
        tmem_ld16(tmem_O + q * DH + c + lane_off, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) o[i] = fmaf(__uint_as_float(r[i]), f[q], o[i]);
      }
      if (row_ok) {
        uint4 w0, w1;
        w0.x = pack_bf16x2(o[0], o[1]);
        w0.y = pack_bf16x2(o[2], o[3]);
        w0.z = pack_bf16x2(o[4], o[5]);
        w0.w = pack_bf16x2(o[6], o[7]);
        w1.x = pack_bf16x2(o[8], o[9]);
        w1.y = pack_bf16x2(o[10], o[11]);
        w1.z = pack_bf16x2(o[12], o[13]);
        w1.w = pack_bf16x2(o[14], o[15]);
        *reinterpret_cast<uint4*>(orow + c) = w0;
        *reinterpret_cast<uint4*>(orow + c + 8) = w1;
      }
    }
    if (half == 0 && row_ok) p.lse[static_cast<long>(h) * p.n + row] = (m + log2f(lt)) * 0.6931471805599453f;
  }
  pdl_trigger_late();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TT_FCTA(3);
  if (warp == 1) tmem_dealloc(tmem, C::kTmemCols);
}

template <int DH, int BKV, int NS, int POLY, int SPL>
void launch_fwd(const AttnFwdArgs& a, long rows_cap, cudaStream_t stream) {
  using C = FwdCfg<DH, BKV, NS, SPL>;
  CUtensorMap tq, tk, tv;
  const int d = a.H * DH;
  make_tmap_bf16(&tq, a.q, d, a.n, a.ldq, 64, kBQ);
  make_tmap_bf16(&tk, a.k, d, rows_cap, a.ldkv, 64, BKV);
  make_tmap_bf16(&tv, a.v, d, rows_cap, a.ldkv, 64, BKV);
  ensure_smem_attr(reinterpret_cast<const void*>(fa_fwd_kernel<DH, BKV, NS, POLY, SPL>), C::kSmem);
  FwdParams p{a.o, a.ldo, a.lse, a.n, a.S, a.H, a.pbase, a.r0 < 0 ? a.S : a.r0, a.qblocks, a.scale * kLog2e};
  dim3 grid(a.nqb, a.H);
  launch_k(fa_fwd_kernel<DH, BKV, NS, POLY, SPL>, grid, dim3(C::kThreads), C::kSmem, stream, tq, tk, tv, p);
}

}  // namespace

// Forward with 128-query blocks (qblocks built with kFwdBlockQ rows). rows_cap = stack rows. dh 64: all
// exponentials on the MUFU (c2 leaf batch: 0.416 ms vs 0.420 / 0.429 with one / two pairs in four on the
// FMA pipe, tools/attn_fwd_ab.sh; round 1, before the max tree, measured +5-8% for one in four).
void attn_fwd_sm100(const AttnFwdArgs& a, long rows_cap, cudaStream_t stream) {
  if (a.nqb == 0) return;
  // dh 64: two softmax warps per lane quadrant (four, with 32 columns each and two S buffers, measured
  // 0.433 vs 0.410 ms on the c2 leaf batch)
#ifndef TT_EXP_FWD_POLY
#define TT_EXP_FWD_POLY 0  // experiment builds only (tools/attn_fwd_ab.sh)
#endif
  if (a.dh == 64) return launch_fwd<64, 128, 3, TT_EXP_FWD_POLY, 2>(a, rows_cap, stream);
  if (a.dh == 128) return launch_fwd<128, 64, 3, 1, 2>(a, rows_cap, stream);
  throw std::invalid_argument("attention: head_dim must be 64 or 128");
}

}  // namespace ttb
