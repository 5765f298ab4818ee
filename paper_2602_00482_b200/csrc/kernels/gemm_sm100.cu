// Persistent warp-specialised tcgen05 GEMM for sm_100a (bf16 operands, fp32 TMEM accumulators).
//
//   C[M x N] (op)= A[M x K] * B[N x K]^T
//
// A(m,k) is K-major (ptr[m*lda + k]) or MN-major (ptr[k*lda + m]); same for B(n,k).
// The three transformer GEMM shapes of forward_segment / backward_segment map onto it as
//   Y  = X W       (matrix.hpp:37-48 `matmul`)            : A K-major,  B MN-major
//   dX = dY W^T    (matrix.hpp:50-62 `matmul_transposed`)  : A K-major,  B K-major
//   dW += X^T dY   (matrix.hpp:64-77 `accumulate_outer`)   : A MN-major, B MN-major
//
// Roles: warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer, then 8 or 16 epilogue warps
// (TMEM -> registers -> fused op -> smem -> TMA store; 2 or 4 warps per TMEM lane quadrant split the
// tile's columns: 16 where the epilogue's per-element work is the critical path, see epi_warps).
// Smem ring of STAGES {A,B} tiles (128B swizzle); two TMEM accumulator slots so the epilogue of tile
// i overlaps the main loop of tile i+1. Split-K partials reduce through TMA reduce-add.
//
// CG = 2 (M >= 256): a CTA pair (cluster of 2 on one TPC) computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 issued by the leader CTA: each CTA stages its own 128 rows of A and HALF
// of B (BN/2), TMA completions of both CTAs land on the leader's full barrier, MMA completions are
// multicast to both CTAs' barriers, and each CTA's TMEM holds its 128 accumulator rows. Per CTA this
// halves the B operand traffic through shared memory.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "gemm.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace ttb {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
// warp 0 TMA, warp 1 MMA, then EPW = 8 or 16 epilogue warps: EPW / 4 per TMEM lane quadrant, each
// taking every (EPW / 4)-th 32-column chunk of its quadrant's 32 rows. 16 (at most 96 registers per
// thread) for the epilogues whose per-element work is the critical path at K = 896 (epi_warps), 8
// (164 registers, two staging slots per warp) otherwise.
constexpr int kMaxThreads = 64 + 32 * 16;
constexpr int threads_of(int epw) { return 64 + 32 * epw; }

template <int BN, int CG, int EPW>
struct Cfg {
  static constexpr int BNC = BN / CG;  // B rows (K-major) / columns (MN-major) staged per CTA
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BNC * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // epilogue staging slots (4 KB) per warp: 2 with 8 warps (a store drains while the next chunk is
  // staged), 1 with 16; 1 for the single-CTA 256-wide tile, whose 48 KB operand stages would
  // otherwise drop to 3
  static constexpr int kSlots = (EPW == 16 || (CG == 1 && BN == 256)) ? 1 : 2;
  static constexpr int kStagingBytes = EPW * kSlots * 4096;
  static constexpr int kStageBudget = 227 * 1024 - kStagingBytes - 2048;
  static constexpr int kStages = kStageBudget / kStageBytes > 8 ? 8 : kStageBudget / kStageBytes;
  static constexpr int kAccStride = BN == 224 ? 256 : BN;  // TMEM columns between the accumulator slots
  static constexpr int kTmemCols = 2 * kAccStride <= 256 ? 256 : 512;  // two slots (power of 2)
  static constexpr int kOffBar = kStages * kStageBytes;
  static constexpr int kOffStage = kOffBar + 1024;  // epilogue staging
  static constexpr int kSmem = kOffStage + kStagingBytes + 1024 /*align*/;
  static_assert(kSmem <= 227 * 1024, "GEMM smem budget");
  static_assert(BNC % 64 == 0 || CG == 1 || BN == 224, "2-CTA MN-major B needs 64-column halves");
};

// ---- CTA-pair (cluster of 2) helpers
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Relaxed remote arrive: these barriers only order TMEM / smem reuse (already fenced by
// tcgen05.wait + fence::before_thread_sync), not the arriving thread's global stores.
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA into this CTA's smem, completion bytes counted on the leader CTA's barrier (cluster address)
__device__ __forceinline__ void tma_load_2d_2sm(const void* tmap, uint32_t bar_cluster, void* smem_dst, int32_t x,
                                                int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_ss_2cta(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                  uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// completion of the pair's MMAs -> arrive on the barrier at this offset in both CTAs
__device__ __forceinline__ void umma_commit_2cta(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
template <int CG>
__device__ __forceinline__ void tmem_alloc_cg(uint32_t* smem_result, uint32_t ncols) {
  if constexpr (CG == 1) {
    tmem_alloc(smem_result, ncols);
  } else {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::);
  }
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc_cg(uint32_t taddr, uint32_t ncols) {
  if constexpr (CG == 1) tmem_dealloc(taddr, ncols);
  else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

// sigmoid(u) = 0.5 tanh(u/2) + 0.5 on a pair: one MUFU op per element (tanh.approx, max rel err ~2^-11
// < bf16 ulp), the affine parts on FMUL2 / FFMA2
__device__ __forceinline__ float2 fast_sigmoid2(float2 u) {
  const float2 hu = __fmul2_rn(u, make_float2(0.5f, 0.5f));
  float2 t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t.x) : "f"(hu.x));
  asm("tanh.approx.f32 %0, %1;" : "=f"(t.y) : "f"(hu.y));
  return __ffma2_rn(t, make_float2(0.5f, 0.5f), make_float2(0.5f, 0.5f));
}
// bf16 pair (lo = element 0) -> two floats, exact
__device__ __forceinline__ float2 unpack_bf16x2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

// ---- epilogue helpers (one thread = one accumulator row; 32 columns per call)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// tcgen05.wait::ld that also names the destination registers of the pending load, so no use of
// them can be scheduled above the wait
__device__ __forceinline__ void tmem_ld_wait_regs(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// ---- TMA-store epilogue
// Each epilogue warp drains its 32 accumulator rows in 32-column chunks: the chunk is written (one
// row per thread) into a per-warp shared-memory slot in the swizzled layout of an output tensor map
// and written back by ONE cp.async.bulk.tensor store (or cp.reduce.async.bulk .add for accumulating
// modes), so the LSU never issues the 32-rows-by-16-bytes scattered stores that capped the direct
// epilogue at ~16 B/clk/SM. Operands the epilogue reads (residual, SiLU input) arrive by TMA into the
// same slot. Two slots per warp: the store of chunk c drains while chunk c+1 is being produced.
// fp32 chunk: 32 rows x 128 B, SWIZZLE_128B (16-byte unit u of row r at u ^ (r & 7));
// bf16 chunk: 32 rows x 64 B, SWIZZLE_64B (unit u of row r at u ^ ((r >> 1) & 3)).
__device__ __forceinline__ uint32_t sw128_off(int r, int u) { return r * 128 + ((u ^ (r & 7)) << 4); }
__device__ __forceinline__ uint32_t sw64_off(int r, int u) { return r * 64 + ((u ^ ((r >> 1) & 3)) << 4); }

__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* smem_src, int32_t x, int32_t y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(smem_src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const void* tmap, const void* smem_src, int32_t x, int32_t y) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(smem_src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Epilogue warps per CTA: 16 for the epilogues whose per-element work is the GEMM's critical path at
// K = 896 (SiLU' with its operand load, the LM-head logits with the softmax statistics), 8 otherwise
// (profiles/r2/gemm_epilogue_ab.txt).
inline int epi_warps(int mode, int bn, int cg) {
  return (mode == EPI_DSILU || mode == EPI_STORE_BF16_STATS) && !(cg == 1 && bn == 256) ? 16 : 8;
}

__device__ __forceinline__ bool epi_f32_out(int mode) {
  return mode == EPI_STORE_F32 || mode == EPI_STORE_F32_STATS || mode == EPI_ADD_F32 || mode == EPI_RESID_F32 ||
         mode == EPI_ADD_F32_T;
}

// This thread's row (lane) of a 32-column chunk -> the warp's staging slot `buf`.
__device__ __forceinline__ void epi_stage(const EpiParams& epi, const uint32_t (&r)[32], uint8_t* buf, int lane,
                                          int row, int M, int n0, int N) {
  const float alpha = epi.alpha;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    const float2 a = __fmul2_rn(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), make_float2(alpha, alpha));
    v[i] = a.x;
    v[i + 1] = a.y;
  }
  switch (epi.mode) {
    case EPI_STORE_F32_STATS:
    case EPI_STORE_BF16_STATS: {
      // per-row (max, sum exp(v - max)) of this 32-column group (columns >= N excluded): 3-input max,
      // then 2^(v log2e - mx log2e) as one FFMA + MUFU per element, paired adds
      constexpr float kL2e = 1.4426950408889634f;
      float mx;
      if (n0 + 32 <= N) {
        mx = fmax3f(v[0], v[1], v[2]);
#pragma unroll
        for (int i = 3; i < 31; i += 2) mx = fmax3f(mx, v[i], v[i + 1]);
        mx = fmaxf(mx, v[31]);
      } else {
        mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (n0 + i < N) mx = fmaxf(mx, v[i]);
      }
      if (row < M) {
        const float nm = -mx * kL2e;
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float e0 = n0 + i < N ? ex2_approx(fmaf(v[i], kL2e, nm)) : 0.f;
          const float e1 = n0 + i + 1 < N ? ex2_approx(fmaf(v[i + 1], kL2e, nm)) : 0.f;
          acc = __fadd2_rn(acc, make_float2(e0, e1));
        }
        reinterpret_cast<float2*>(epi.out2)[static_cast<long>(row) * epi.ldo2 + n0 / 32] = make_float2(mx, acc.x + acc.y);
      }
      if (epi.mode == EPI_STORE_BF16_STATS) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          *reinterpret_cast<uint4*>(buf + sw64_off(lane, u)) =
              make_uint4(pack_bf16x2(v[8 * u] - mx, v[8 * u + 1] - mx), pack_bf16x2(v[8 * u + 2] - mx, v[8 * u + 3] - mx),
                         pack_bf16x2(v[8 * u + 4] - mx, v[8 * u + 5] - mx),
                         pack_bf16x2(v[8 * u + 6] - mx, v[8 * u + 7] - mx));
        break;
      }
    }
      [[fallthrough]];
    case EPI_STORE_F32:
    case EPI_ADD_F32:
#pragma unroll
      for (int u = 0; u < 8; ++u)
        *reinterpret_cast<float4*>(buf + sw128_off(lane, u)) =
            make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
      break;
    case EPI_ADD_F32_T:  // staged transposed: 32 columns x 32 rows (128B swizzled), conflict-free
#pragma unroll
      for (int c = 0; c < 32; ++c)
        *reinterpret_cast<float*>(buf + sw128_off(c, lane >> 2) + (lane & 3) * 4) = v[c];
      break;
    case EPI_RESID_F32:  // out = resid + acc (model.hpp:427-428,447-448); resid chunk already in buf
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float4* p = reinterpret_cast<float4*>(buf + sw128_off(lane, u));
        const float4 o = *p;
        *p = make_float4(o.x + v[4 * u], o.y + v[4 * u + 1], o.z + v[4 * u + 2], o.w + v[4 * u + 3]);
      }
      break;
    case EPI_STORE_BF16:
#pragma unroll
      for (int u = 0; u < 4; ++u)
        *reinterpret_cast<uint4*>(buf + sw64_off(lane, u)) =
            make_uint4(pack_bf16x2(v[8 * u], v[8 * u + 1]), pack_bf16x2(v[8 * u + 2], v[8 * u + 3]),
                       pack_bf16x2(v[8 * u + 4], v[8 * u + 5]), pack_bf16x2(v[8 * u + 6], v[8 * u + 7]));
      break;
    case EPI_SILU:  // h (bf16) -> buf, silu(h) (bf16) -> buf + 2048 (model.hpp:443-444)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        // h rounded to bf16 once, silu of the rounded value; pairs on FMUL2 / FFMA2
        uint32_t hw[4], sw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          hw[i] = pack_bf16x2(v[8 * u + 2 * i], v[8 * u + 2 * i + 1]);
          const float2 hh = unpack_bf16x2(hw[i]);
          const float2 sv = __fmul2_rn(hh, fast_sigmoid2(hh));
          sw[i] = pack_bf16x2(sv.x, sv.y);
        }
        *reinterpret_cast<uint4*>(buf + sw64_off(lane, u)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(buf + 2048 + sw64_off(lane, u)) = make_uint4(sw[0], sw[1], sw[2], sw[3]);
      }
      break;
    case EPI_DSILU:  // out = acc * silu'(h) (model.hpp:526-528); h chunk (bf16) already in buf
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint4* p = reinterpret_cast<uint4*>(buf + sw64_off(lane, u));
        const uint4 hw = *p;
        // silu'(h) = s (1 + h (1 - s)), s = sigmoid(h), on pairs
        const uint32_t hws[4] = {hw.x, hw.y, hw.z, hw.w};
        uint32_t gw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 hh = unpack_bf16x2(hws[i]);
          const float2 sg = fast_sigmoid2(hh);
          const float2 oms = __ffma2_rn(sg, make_float2(-1.f, -1.f), make_float2(1.f, 1.f));
          const float2 gr = __fmul2_rn(sg, __ffma2_rn(hh, oms, make_float2(1.f, 1.f)));
          const float2 g = __fmul2_rn(make_float2(v[8 * u + 2 * i], v[8 * u + 2 * i + 1]), gr);
          gw[i] = pack_bf16x2(g.x, g.y);
        }
        *p = make_uint4(gw[0], gw[1], gw[2], gw[3]);
      }
      break;
    default:
      break;
  }
}

#ifndef TT_TRACE
#define TT_TRACE 0
#endif
#if TT_TRACE  // trace build only (make trace; tools/gemm_trace.py): per-warp, per-tile clock64 events
constexpr int kGtCtas = 4, kGtTiles = 48, kGtEv = 8;
__device__ long long g_gemm_trace[kGtCtas][kMaxThreads / 32][kGtTiles][kGtEv];
#define GT_TR(ev, ti)                                                                                       \
  do {                                                                                                      \
    if (blockIdx.x < kGtCtas && (ti) < kGtTiles) g_gemm_trace[blockIdx.x][warp][(ti)][(ev)] = clock64();    \
  } while (0)
#define GT_ADD(ev, ti, v)                                                                                   \
  do {                                                                                                      \
    if (blockIdx.x < kGtCtas && (ti) < kGtTiles) g_gemm_trace[blockIdx.x][warp][(ti)][(ev)] += (v);         \
  } while (0)
#define GT_CLK() clock64()
#else
#define GT_TR(ev, ti) \
  do {                \
  } while (0)
#define GT_ADD(ev, ti, v) \
  do {                    \
  } while (0)
#define GT_CLK() 0LL
#endif

template <int BN, int CG, bool A_MN, bool B_MN, int EPW>
__global__ void __launch_bounds__(threads_of(EPW), 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                const __grid_constant__ CUtensorMap tm_o0, const __grid_constant__ CUtensorMap tm_o1,
                const __grid_constant__ CUtensorMap tm_o2, const __grid_constant__ CUtensorMap tm_x, int M, int N,
                int K, int splits, EpiParams epi) {
  using C = Cfg<BN, CG, EPW>;
  static_assert(!B_MN || CG == 1 || C::BNC % 64 == 0, "BN = 224 pairs need a K-major B (112-row halves)");
  constexpr int TM = BM * CG;  // tile rows (per CTA pair when CG = 2)
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;  // cluster id / count
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* tfull_bar = empty_bar + C::kStages;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;          // [2]
  uint64_t* ld_bar = tempty_bar + 2;  // [EPW][4]: TMA loads of epilogue operands into the slots
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ld_bar + 4 * EPW);

  const int warp = warp_id_sync();
  const int lane = threadIdx.x & 31;

  const int num_m = (M + TM - 1) / TM;
  const int num_n = (N + BN - 1) / BN;
  const int kb_total = (K + BK - 1) / BK;
  const int kb_per = (kb_total + splits - 1) / splits;
  const int num_tiles = num_m * num_n * splits;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], CG);  // leader: its own arrive.expect_tx + the peer's arrive
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], EPW * CG);  // leader: epilogue warps of both CTAs
    }
    for (int s = 0; s < 4 * EPW; ++s) mbar_init(&ld_bar[s], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg<CG>(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();     // predecessor grid complete: operands / epilogue inputs are final (launch.cuh)
  pdl_trigger_early();  // TMEM held: the successor may start its prologue

  // Rasterisation: the concurrently running tiles should share the LARGER operand's panels so it
  // streams from HBM once while the smaller one stays L2-resident: n-fastest when A (M x K) is the
  // bigger operand (activations x weights), m-fastest otherwise (e.g. the LM head's 150K-wide B).
  const bool n_fast = static_cast<long>(M) > static_cast<long>(N);
  auto tile_coords = [&](int t, int& m_blk, int& n_blk, int& kb0, int& kb1) {
    const int per = num_m * num_n;
    const int split = t / per;
    const int rem = t - split * per;
    if (n_fast) {
      m_blk = rem / num_n;
      n_blk = rem - m_blk * num_n;
    } else {
      n_blk = rem / num_m;
      m_blk = rem - n_blk * num_m;
    }
    kb0 = split * kb_per;
    kb1 = min(kb_total, kb0 + kb_per);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int ti = 0;
      for (int t = cid; t < num_tiles; t += ncl, ++ti) {
        int m_blk, n_blk, kb0, kb1;
        tile_coords(t, m_blk, n_blk, kb0, kb1);
        const int m0 = m_blk * TM + static_cast<int>(rank) * BM;         // this CTA's A rows
        const int n0 = n_blk * BN + static_cast<int>(rank) * C::BNC;     // this CTA's B half
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (kb == kb0) GT_TR(0, ti);
          if (kb == kb1 - 1) GT_TR(1, ti);
          uint8_t* sa = smem + stage * C::kStageBytes;
          uint8_t* sb = sa + C::kABytes;
          const int k0 = kb * BK;
          if constexpr (CG == 1) {
            mbar_arrive_expect_tx(&full_bar[stage], C::kStageBytes);
            if constexpr (!A_MN) {
              tma_load_2d(&tmap_a, &full_bar[stage], sa, k0, m0);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j) tma_load_2d(&tmap_a, &full_bar[stage], sa + j * 8192, m0 + j * 64, k0);
            }
            if constexpr (!B_MN) {
              tma_load_2d(&tmap_b, &full_bar[stage], sb, k0, n0);
            } else {
#pragma unroll
              for (int j = 0; j < C::BNC / 64; ++j)
                tma_load_2d(&tmap_b, &full_bar[stage], sb + j * 8192, n0 + j * 64, k0);
            }
          } else {
            const uint32_t fb = mapa_shared(smem_u32(&full_bar[stage]), 0);  // the leader's full barrier
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * C::kStageBytes);
            else mbar_arrive_remote(fb);
            if constexpr (!A_MN) {
              tma_load_2d_2sm(&tmap_a, fb, sa, k0, m0);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j) tma_load_2d_2sm(&tmap_a, fb, sa + j * 8192, m0 + j * 64, k0);
            }
            if constexpr (!B_MN) {
              tma_load_2d_2sm(&tmap_b, fb, sb, k0, n0);
            } else {
#pragma unroll
              for (int j = 0; j < C::BNC / 64; ++j) tma_load_2d_2sm(&tmap_b, fb, sb + j * 8192, n0 + j * 64, k0);
            }
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA only)
    if (!leader) goto mma_done;
    {
    constexpr uint32_t idesc = make_idesc_bf16(TM, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int ti = 0;
    for (int t = cid; t < num_tiles; t += ncl, ++ti) {
      int m_blk, n_blk, kb0, kb1;
      tile_coords(t, m_blk, n_blk, kb0, kb1);
      if (lane == 0) GT_TR(0, ti);
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      if (lane == 0) GT_TR(1, ti);
      const uint32_t d_tmem = tmem_base + acc * C::kAccStride;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t sb = sa + C::kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t da, db;
            if constexpr (!A_MN) da = make_sdesc_sw128(sa + k * 32, 16, 1024);
            else da = make_sdesc_sw128(sa + k * 2048, 8192, 1024);
            if constexpr (!B_MN) db = make_sdesc_sw128(sb + k * 32, 16, 1024);
            else db = make_sdesc_sw128(sb + k * 2048, 8192, 1024);
            if constexpr (CG == 1) umma_bf16_ss(d_tmem, da, db, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            else umma_bf16_ss_2cta(d_tmem, da, db, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          if constexpr (CG == 1) umma_commit(&empty_bar[stage]);
          else umma_commit_2cta(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) {
        if constexpr (CG == 1) umma_commit(&tfull_bar[acc]);
        else umma_commit_2cta(&tfull_bar[acc]);
        GT_TR(2, ti);
      }
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    }
  mma_done:;
  } else {
    // ------------------------------------------------------------ epilogue
    // Each warp drains 32 TMEM lanes (rows) x BN/kEG columns in 32-column chunks. The TMEM load of
    // chunk c+1 is in flight while chunk c is staged; the accumulator slot is handed back to the MMA
    // warp as soon as its last chunk is in registers; stores drain asynchronously (TMA).
    constexpr int EG = EPW / 4;  // epilogue warps per TMEM lane quadrant
    constexpr int SL = C::kSlots;  // staging slots per warp
    const int quad = warp & 3;             // TMEM lane quadrant this warp may access
    const int grp = (warp - 2) / 4;        // which 32-column chunks of the tile this warp handles
    constexpr int NCHT = BN / 32;          // chunks per tile; warp group g takes chunks g, g + EG, ...
    constexpr int NCH = (NCHT + EG - 1) / EG;  // chunk slots per warp (the last may be empty)
    constexpr int CS = 32 * EG;           // columns between a warp's consecutive chunks
    const int ew = warp - 2;
    uint8_t* stg = smem + C::kOffStage + ew * (SL * 4096);
    uint64_t* wld = ld_bar + 4 * ew;
    const int mode = epi.mode;
    const bool need_ld = mode == EPI_RESID_F32 || mode == EPI_DSILU;
    const uint32_t ld_bytes = epi_f32_out(mode) ? 4096u : 2048u;
    // SiLU' epilogue (bf16 operand in, bf16 out, in place): all NCH chunks' operands fit in the slots
    const bool whole_tile_ld = mode == EPI_DSILU && NCH <= 4 && SL * 4096 >= NCH * 2048;
    // residual epilogue (fp32 operand, 4 KB per chunk): two chunks loaded ahead, one per slot
    const bool two_ahead = need_ld && !whole_tile_ld && SL == 2;
    uint32_t gc = 0;        // chunks staged by this warp: slot = gc & 1
    bool pf = false;        // SiLU' operand chunks 0 .. NCH-2 of this tile were prefetched by the last one
    uint32_t ld_phase = 0;  // per-slot parity of the operand-load barriers
    bool ld_ahead = false;  // the current chunk's operand load was issued during the previous chunk
    int acc = 0;
    uint32_t acc_phase = 0;
    int ti = 0;
    for (int t = cid; t < num_tiles; t += ncl, ++ti) {
      int m_blk, n_blk, kb0, kb1;
      tile_coords(t, m_blk, n_blk, kb0, kb1);
      const int row0 = m_blk * TM + static_cast<int>(rank) * BM + quad * 32;  // this warp's first row
      const int n_base = n_blk * BN + grp * 32;  // this warp's first chunk; chunk c at n_base + CS c
      auto chunk_ok = [&](int c) { return EG * c + grp < NCHT && n_base + CS * c < N; };
      if (whole_tile_ld) {
        // every chunk's bf16 operand (2 KB) gets its own quarter slot: all loads issued before the
        // accumulator wait (all but the last already at the end of the previous tile, see below)
        if (lane == 0) {
          bulk_wait_read<0>();
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
            if ((!pf || ch == NCH - 1) && chunk_ok(ch)) {
              mbar_arrive_expect_tx(&wld[ch], 2048u);
              tma_load_2d(&tm_x, &wld[ch], stg + ch * 2048, n_base + CS * ch, row0);
            }
        }
        __syncwarp();
        pf = false;
      } else if (two_ahead) {
        if (lane == 0) {
          bulk_wait_read<0>();
#pragma unroll
          for (int k = 0; k < 2 && k < NCH; ++k)
            if (chunk_ok(k)) {
              const int sl = static_cast<int>((gc + k) & 1);
              mbar_arrive_expect_tx(&wld[sl], ld_bytes);
              tma_load_2d(&tm_x, &wld[sl], stg + sl * 4096, n_base + CS * k, row0);
            }
        }
        __syncwarp();
      } else if (need_ld && !ld_ahead && chunk_ok(0)) {
        // the tile's first epilogue operand chunk loads while its main loop still runs
        const int slot = SL == 2 ? static_cast<int>(gc & 1) : 0;
        if (lane == 0) {
          bulk_wait_read<SL - 1>();
          mbar_arrive_expect_tx(&wld[slot], ld_bytes);
          tma_load_2d(&tm_x, &wld[slot], stg + slot * 4096, n_base, row0);
        }
        __syncwarp();
        ld_ahead = true;
      }
      if (lane == 0) GT_TR(0, ti);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      if (lane == 0) GT_TR(1, ti);
      const uint32_t t_row = tmem_base + acc * C::kAccStride + grp * 32 + (static_cast<uint32_t>(quad * 32) << 16);
      uint32_t rr[2][32];
      tmem_ld32(t_row, rr[0]);
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int n0 = n_base + CS * ch;
        const bool active = chunk_ok(ch);  // warp-uniform
        const int slot = whole_tile_ld ? ch : (SL == 2 ? static_cast<int>(gc & 1) : 0);
        uint8_t* buf = whole_tile_ld ? stg + ch * 2048 : stg + slot * 4096;
        int blk = 0, xc = n0;
        if (epi.split_w > 0) {
          blk = n0 / epi.split_w;
          xc = n0 - blk * epi.split_w;
        }
        // the chunk's accumulator columns first (the last chunk hands the slot back to the MMA warp),
        // then the staging slot: a slow store drain does not hold the accumulator
        long long gt0 = GT_CLK();
        tmem_ld_wait_regs(rr[ch & 1]);
        if (lane == 0) GT_ADD(6, ti, GT_CLK() - gt0);
        if (ch + 1 < NCH) {
          tmem_ld32(t_row + (ch + 1) * CS, rr[(ch + 1) & 1]);
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 1) mbar_arrive(&tempty_bar[acc]);
            else mbar_arrive_remote(mapa_shared(smem_u32(&tempty_bar[acc]), 0));  // the leader's slot barrier
            GT_TR(2, ti);
          }
        }
        if (active && !ld_ahead && !whole_tile_ld && !two_ahead) {
          if (lane == 0) {
            gt0 = GT_CLK();
            bulk_wait_read<SL - 1>();  // the store that last used this slot has read it
            GT_ADD(7, ti, GT_CLK() - gt0);
          }
          __syncwarp();
          if (need_ld && lane == 0) {
            mbar_arrive_expect_tx(&wld[slot], ld_bytes);
            tma_load_2d(&tm_x, &wld[slot], buf, n0, row0);
          }
        }
        ld_ahead = false;
        if (active) {
          if (need_ld) {
            gt0 = GT_CLK();
            mbar_wait(&wld[slot], (ld_phase >> slot) & 1);
            ld_phase ^= 1u << slot;
            if (lane == 0) GT_ADD(4, ti, GT_CLK() - gt0);
          }
          gt0 = GT_CLK();
          epi_stage(epi, rr[ch & 1], buf, lane, row0 + lane, M, n0, N);
          if (lane == 0) GT_ADD(5, ti, GT_CLK() - gt0);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            const CUtensorMap* tm = blk == 0 ? &tm_o0 : (blk == 1 ? &tm_o1 : &tm_o2);
            if (mode == EPI_ADD_F32) tma_reduce_add_2d(tm, buf, xc, row0);
            else if (mode == EPI_ADD_F32_T) tma_reduce_add_2d(tm, buf, row0, n0);
#if defined(TT_EXP_SILU_NOSTORE)  // experiment builds only: the SiLU epilogue computes and stages, stores nothing
            else if (mode != EPI_SILU) tma_store_2d(tm, buf, xc, row0);
#else
            else tma_store_2d(tm, buf, xc, row0);
#endif
#if !defined(TT_EXP_SILU_ONESTORE) && !defined(TT_EXP_SILU_NOSTORE)
            if (mode == EPI_SILU) tma_store_2d(&tm_x, buf + 2048, n0, row0);
#endif
            bulk_commit();
            GT_TR(3, ti);  // the tile's last store issued (overwritten per chunk)
          }
          ++gc;
          // operand epilogues (residual / SiLU input): start the next chunk's TMA load now, into the
          // other slot once its previous store has been read, so it overlaps this chunk's tail
          if (two_ahead) {
            // this chunk's slot takes chunk ch + 2 once the store just issued has read it
            if (ch + 2 < NCH && chunk_ok(ch + 2)) {
              const int ns = static_cast<int>((gc + 1) & 1);  // == slot (gc was incremented)
              if (lane == 0) {
                bulk_wait_read<0>();
                mbar_arrive_expect_tx(&wld[ns], ld_bytes);
                tma_load_2d(&tm_x, &wld[ns], stg + ns * 4096, n0 + 2 * CS, row0);
              }
              __syncwarp();
            }
          } else if (SL == 2 && need_ld && !whole_tile_ld && ch + 1 < NCH && chunk_ok(ch + 1)) {
            const int ns = static_cast<int>(gc & 1);
            if (lane == 0) {
              bulk_wait_read<1>();
              mbar_arrive_expect_tx(&wld[ns], ld_bytes);
              tma_load_2d(&tm_x, &wld[ns], stg + ns * 4096, n0 + CS, row0);
            }
            __syncwarp();
            ld_ahead = true;
          }
        }
      }
      if (whole_tile_ld && NCH >= 2 && t + ncl < num_tiles) {
        // At K = 896 the main loop is short and this epilogue is the GEMM's critical path, so the next
        // tile's SiLU' operand must not start loading only when that tile starts: chunks 0 .. NCH-2 load
        // now, into quarter slots whose stores (all but this tile's last) have been read
        int m2, n2, k0n, k1n;
        tile_coords(t + ncl, m2, n2, k0n, k1n);
        const int row0n = m2 * TM + static_cast<int>(rank) * BM + quad * 32;
        const int n_basen = n2 * BN + grp * 32;
        if (lane == 0) {
          if (chunk_ok(NCH - 1)) bulk_wait_read<1>();  // the last group is chunk NCH-1's store
          else bulk_wait_read<0>();
#pragma unroll
          for (int ch = 0; ch < NCH - 1; ++ch)
            if (EG * ch + grp < NCHT && n_basen + CS * ch < N) {
              mbar_arrive_expect_tx(&wld[ch], 2048u);
              tma_load_2d(&tm_x, &wld[ch], stg + ch * 2048, n_basen + CS * ch, row0n);
            }
        }
        __syncwarp();
        pf = true;
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait_all();  // stores complete before the CTA (and its smem) retires
  }

  pdl_trigger_late();
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();  // the peer's MMAs into this CTA's TMEM are complete
  if (warp == 1) tmem_dealloc_cg<CG>(tmem_base, C::kTmemCols);
}

// ---------------------------------------------------------------- host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

}  // namespace

// 2-D bf16 tensor map: inner dimension `inner` (contiguous), outer `outer`, row pitch `ld` elements.
void make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                    uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

void make_tmap_f32_sw128(CUtensorMap* map, const void* ptr, uint64_t width, uint64_t rows, uint64_t ld) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (ld * 4) % 16 != 0)
    throw std::invalid_argument("fp32 tensor map: pointer / pitch must be 16-byte aligned");
  cuuint64_t dims[2] = {width, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled (f32 sw128) failed (" + std::to_string(int(r)) + ")");
}

// 2-D fp32 tensor map (no swizzle): inner x outer elements, row pitch ld elements (multiple of 4).
void make_tmap_f32_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                      uint32_t box_inner, uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled (f32) failed (" + std::to_string(int(r)) + ")");
}

namespace {


// Output / epilogue-operand tensor map: [rows x width] elements (fp32 or bf16), row pitch ld elements,
// 32 x 32 boxes in the swizzled staging layout of the epilogue (128B rows fp32, 64B rows bf16).
void make_tmap_epi(CUtensorMap* map, const void* ptr, bool f32, uint64_t width, uint64_t rows, uint64_t ld) {
  const uint64_t esz = f32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (ld * esz) % 16 != 0)
    throw std::invalid_argument("gemm epilogue: output pointer / pitch must be 16-byte aligned");
  cuuint64_t dims[2] = {width, rows};
  cuuint64_t strides[1] = {ld * esz};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                               const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled (epilogue) failed (" + std::to_string(int(r)) + ")");
}

template <int BN, int CG, bool A_MN, bool B_MN, int EPW>
void launch_epw(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const EpiParams& epi, int splits,
                cudaStream_t stream) {
  using C = Cfg<BN, CG, EPW>;
  CUtensorMap ta, tb;
  if (!A_MN) make_tmap_bf16(&ta, A.ptr, K, M, A.ld, 64, BM);
  else make_tmap_bf16(&ta, A.ptr, M, K, A.ld, 64, 64);
  if (!B_MN) make_tmap_bf16(&tb, B.ptr, K, N, B.ld, 64, C::BNC);
  else make_tmap_bf16(&tb, B.ptr, N, K, B.ld, 64, 64);
  ensure_smem_attr(reinterpret_cast<const void*>(gemm_kernel<BN, CG, A_MN, B_MN, EPW>), C::kSmem);
  const int g_num_sms = device_sm_count();
  const int kb_total = (K + BK - 1) / BK;
  if (splits < 1) splits = 1;
  if (splits > kb_total) splits = kb_total;
  const int per = (kb_total + splits - 1) / splits;
  splits = (kb_total + per - 1) / per;  // no empty split
  const int tiles = ((M + BM * CG - 1) / (BM * CG)) * ((N + BN - 1) / BN) * splits;
  const int max_clusters = g_num_sms / CG;
  const int grid = (tiles < max_clusters ? tiles : max_clusters) * CG;
  EpiParams e = epi;
  if (splits > 1) e.atomic = 1;
  // output tensor maps (and the epilogue operand map: silu output / dsilu input / residual input)
  const bool f32 = e.mode == EPI_STORE_F32 || e.mode == EPI_STORE_F32_STATS || e.mode == EPI_ADD_F32 ||
                   e.mode == EPI_RESID_F32 || e.mode == EPI_ADD_F32_T;
  if (e.mode == EPI_ADD_F32_T && e.split_w > 0) throw std::invalid_argument("gemm epilogue: transposed add takes no split_w");
  if (e.split_w > 0 && (e.split_w % 32 != 0 || e.mode == EPI_SILU || e.mode == EPI_DSILU || e.mode == EPI_RESID_F32))
    throw std::invalid_argument("gemm epilogue: split_w must be a multiple of 32 (store / add modes only)");
  CUtensorMap to[3], tx;
  std::memset(to, 0, sizeof(to));
  std::memset(&tx, 0, sizeof(tx));
  const uint64_t width = e.split_w > 0 ? static_cast<uint64_t>(e.split_w) : static_cast<uint64_t>(N);
  const int nout = e.split_w > 0 ? (N + e.split_w - 1) / e.split_w : 1;
  if (nout > 3) throw std::invalid_argument("gemm epilogue: at most 3 column blocks");
  if (e.mode == EPI_ADD_F32_T) make_tmap_epi(&to[0], e.out[0], true, M, N, e.ldo[0]);  // [N][M] output
  else
    for (int i = 0; i < nout; ++i) make_tmap_epi(&to[i], e.out[i], f32, width, M, e.ldo[i]);
  if (e.mode == EPI_SILU) make_tmap_epi(&tx, e.out2, false, N, M, e.ldo2);
  if (e.mode == EPI_DSILU) make_tmap_epi(&tx, e.aux, false, N, M, e.ld_aux);
  if (e.mode == EPI_RESID_F32) make_tmap_epi(&tx, e.resid, true, N, M, e.ld_resid);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads_of(EPW));
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_attr(attr, 1);
  check_launch(cudaLaunchKernelEx(&cfg, gemm_kernel<BN, CG, A_MN, B_MN, EPW>, ta, tb, to[0], to[1], to[2], tx, M, N, K,
                                  splits, e),
               "gemm launch");
}

template <int BN, int CG, bool A_MN, bool B_MN>
void launch(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const EpiParams& epi, int splits,
            cudaStream_t stream) {
  if constexpr (!(CG == 1 && BN == 256)) {
    if (epi_warps(epi.mode, BN, CG) == 16) return launch_epw<BN, CG, A_MN, B_MN, 16>(A, B, M, N, K, epi, splits, stream);
  }
  launch_epw<BN, CG, A_MN, B_MN, 8>(A, B, M, N, K, epi, splits, stream);
}

}  // namespace

int g_gemm_2cta = 1;
void gemm_set_2cta(int on) { g_gemm_2cta = on; }

// CTA pairs (256-row tiles) unless padding M to 256 wastes more than ~5% (e.g. M = 896); up to 15%
// when the GEMM has many waves of pair tiles anyway (e.g. the LM-head dW: 896 x 151936), where the
// pair's halved operand traffic outweighs the padding (profiles/r1: 0.556 -> 0.513 ms).
bool gemm_use_2cta(int M, int N) {
  if (!g_gemm_2cta || M < 256) return false;
  if (g_gemm_2cta == 2) return true;  // debug / measurement: always pair tiles
  constexpr int waste_pct = 5;  // allowed M padding in %
  const long padded = (M + 255) / 256 * 256;
  if ((padded - M) * 100 <= static_cast<long>(M) * waste_pct) return true;
  const int g_num_sms = device_sm_count();
  const long pair_tiles = (padded / 256) * ((N + 255) / 256);
  return (padded - M) * 100 <= static_cast<long>(M) * 15 && pair_tiles >= 4L * (g_num_sms / 2);
}

// 2-CTA tile width: 256 unless its padding waste outweighs the halved per-CTA B traffic
// 2-CTA tile width from a wave model: time ~ waves x per-tile cost, with a 128-wide pair tile ~60%
// more expensive per column than a 256-wide one (twice the A re-reads per FLOP, shorter MMAs, half
// the B staging per CTA). Measured (profiles/r1/gemm_shapes_bn2.log, profiles/r2/gemm_bn2.txt): N = 896
// at M = 32768 runs 17-22% faster with 256-wide tiles despite 12.5% padding; the c3 QKV weight
// gradient (1536 x 4608 x 8192) 911 -> 1373 TF/s with 256 (3 waves of 128-wide tiles modelled at
// 1.25 had picked 128); M = 4864, N = 896 runs the same either way.
int g_gemm_force_bn2 = 0;  // debug entry only (tt_debug_gemm_force_bn2): 0 = modelled
void gemm_force_bn2(int bn) { g_gemm_force_bn2 = bn; }

int gemm_pick_bn2(int M, int N) {
  if (g_gemm_force_bn2 == 128 || g_gemm_force_bn2 == 256) return g_gemm_force_bn2;
  const int g_num_sms = device_sm_count();
  const long pairs = std::max(1, g_num_sms / 2);
  const long m_tiles = (M + 255) / 256;
  auto cost = [&](int bn, double f) {
    const long tiles = m_tiles * ((N + bn - 1) / bn);
    return static_cast<double>((tiles + pairs - 1) / pairs) * bn * f;
  };
  return cost(256, 1.0) <= cost(128, 1.6) ? 256 : 128;
}

int g_gemm_force_bn1 = 0;  // debug entry only (tt_debug_gemm_force_bn1): 0 = modelled
void gemm_force_bn1(int bn) { g_gemm_force_bn1 = bn; }

int gemm_pick_bn(int N, bool b_mn_major) {
  (void)b_mn_major;  // 128/192/256 are all multiples of the 64-element MN atom
  if (g_gemm_force_bn1 == 128 || g_gemm_force_bn1 == 192 || g_gemm_force_bn1 == 256) return g_gemm_force_bn1;
  // padded columns weighted by the per-tile overhead of narrower tiles (smem operand traffic); 128-wide
  // at 1.25 (profiles/r2/gemm_bn2.txt: the c2 W_o weight gradient 896 x 896 x 32768 runs at 965 TF/s
  // with 128-wide tiles, 1035 with 192, 1074 with 256)
  int best = 256;
  double best_cost = 0;
  for (int bn : {256, 192, 128}) {
    const double f = bn == 256 ? 1.0 : (bn == 192 ? 1.04 : 1.25);
    const double cost = static_cast<double>((N + bn - 1) / bn) * bn * f;
    if (bn == 256 || cost < best_cost) {
      best = bn;
      best_cost = cost;
    }
  }
  return best;
}

#if TT_TRACE
extern "C" int tt_debug_gemm_trace_read(long long* out, long n) {
  const long sz = static_cast<long>(sizeof(g_gemm_trace) / sizeof(long long));
  return cudaMemcpyFromSymbol(out, g_gemm_trace, (n < sz ? n : sz) * sizeof(long long)) == cudaSuccess ? 0 : -1;
}
extern "C" int tt_debug_gemm_trace_clear() {
  static long long zero[sizeof(g_gemm_trace) / sizeof(long long)];
  return cudaMemcpyToSymbol(g_gemm_trace, zero, sizeof(zero)) == cudaSuccess ? 0 : -1;
}
#endif

void gemm_bf16(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const EpiParams& epi, int splits,
               cudaStream_t stream) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  if (N % 16 != 0) throw std::invalid_argument("gemm_bf16: N must be a multiple of 16");
  if (splits > 1 && epi.mode != EPI_ADD_F32 && epi.mode != EPI_ADD_F32_T)
    throw std::invalid_argument("gemm_bf16: split-K needs EPI_ADD_F32");
  if (epi.mode == EPI_ADD_F32 && epi.split_w == 0 && gemm_prefer_transposed(M, N, K)) {
    // C += A B^T  <=>  C^T += B A^T with a transposed epilogue (operand views swap roles unchanged)
    EpiParams et = epi;
    et.mode = EPI_ADD_F32_T;
    return gemm_bf16(B, A, N, M, K, et, gemm_choose_splits(N, M, K), stream);
  }
  const bool amn = A.mn_major, bmn = B.mn_major;
#define TTB_DISPATCH(BN_, CG_)                                                                      \
  if (!amn && bmn) return launch<BN_, CG_, false, true>(A, B, M, N, K, epi, splits, stream);  \
  if (!amn && !bmn) return launch<BN_, CG_, false, false>(A, B, M, N, K, epi, splits, stream); \
  if (amn && bmn) return launch<BN_, CG_, true, true>(A, B, M, N, K, epi, splits, stream);     \
  return launch<BN_, CG_, true, false>(A, B, M, N, K, epi, splits, stream);
  if (!bmn && N % 256 != 0 && N % 224 == 0 && gemm_use_2cta(M, N)) {
    // N = 896 (d of the 0.5B shape): 4 x 224 columns instead of 3.5 x 256 (12.5% padding); each CTA
    // stages 112 rows of the K-major B
    if (!amn) return launch<224, 2, false, false>(A, B, M, N, K, epi, splits, stream);
    return launch<224, 2, true, false>(A, B, M, N, K, epi, splits, stream);
  }
  if (gemm_use_2cta(M, N)) {
    // CTA pairs: 256-row tiles; BN 128 or 256 (each CTA stages a 64-aligned half of B)
    if (gemm_pick_bn2(M, N) == 256) {
      TTB_DISPATCH(256, 2)
    } else {
      TTB_DISPATCH(128, 2)
    }
  }
  const int bn = gemm_pick_bn(N, B.mn_major);
  if (bn == 256) {
    TTB_DISPATCH(256, 1)
  } else if (bn == 192) {
    TTB_DISPATCH(192, 1)
  } else {
    TTB_DISPATCH(128, 1)
  }
#undef TTB_DISPATCH
}

int gemm_choose_splits(int M, int N, int K) {
  const int g_num_sms = device_sm_count();
  const bool two = gemm_use_2cta(M, N);
  const int bn = two ? gemm_pick_bn2(M, N) : gemm_pick_bn(N, true);
  // Time model: waves of (tile, K/s) items at ~9 TFLOP/s per SM, plus the fp32 reduce-add of every
  // split's partial output through L2 (~2.5 TB/s). Splits pay when the tiles leave units idle: 49
  // tiles on 148 SMs (3 splits = one wave), or 104 pair tiles on 74 pairs (2 waves, the second 40%
  // full; 2 splits = 3 half-length waves: the LM-head dX at 6656 loss rows); never for outputs whose
  // reduce traffic dominates (the LM-head dW: 896 x 151936 fp32).
  const long units = two ? g_num_sms / 2 : g_num_sms;
  const long tiles = (two ? (M + 2 * BM - 1) / (2 * BM) : (M + BM - 1) / BM) * static_cast<long>((N + bn - 1) / bn);
  const int kb = (K + BK - 1) / BK;
  if (kb < 8) return 1;
  const double unit_rate = (two ? 2.0 : 1.0) * 9e12;
  const double tile_flops = 2.0 * (two ? 2 * BM : BM) * bn * static_cast<double>(K);
  auto cost = [&](int sp) {
    const double waves = static_cast<double>((tiles * sp + units - 1) / units);
    const double red = sp > 1 ? sp * static_cast<double>(M) * N * 4.0 / 2.5e12 : 0.0;
    return waves * tile_flops / sp / unit_rate + red;
  };
  int best_s = 1;
  double best = cost(1);
  for (int sp = 2; sp <= 16 && sp <= kb / 4; ++sp) {
    const double c = cost(sp);
    if (c < best * 0.98) {  // a split must buy a clear win
      best = c;
      best_s = sp;
    }
  }
  return best_s;
}

// Wave model of one launch in SM-seconds: waves x (per-unit tile FLOPs / K-split) / unit rate, with the
// narrower tiles' per-FLOP overhead (pick_bn / pick_bn2 weights) and the split reduce traffic.
static double gemm_est_cost(int M, int N, int K) {
  const int g_num_sms = device_sm_count();
  const bool two = gemm_use_2cta(M, N);
  const int bn = two ? gemm_pick_bn2(M, N) : gemm_pick_bn(N, true);
  const double f = two ? (bn == 256 ? 1.0 : 1.6) : (bn == 256 ? 1.0 : (bn == 192 ? 1.04 : 1.25));
  const long units = two ? g_num_sms / 2 : g_num_sms;
  const long tiles = (two ? (M + 2 * BM - 1) / (2 * BM) : (M + BM - 1) / BM) * static_cast<long>((N + bn - 1) / bn);
  const int sp = gemm_choose_splits(M, N, K);
  const double waves = static_cast<double>((tiles * sp + units - 1) / units);
  const double tile_flops = 2.0 * (two ? 2 * BM : BM) * bn * static_cast<double>(K) / sp;
  const double red = sp > 1 ? sp * static_cast<double>(M) * N * 4.0 / 2.5e12 : 0.0;
  return waves * tile_flops * f / ((two ? 2.0 : 1.0) * 9e12) + red;
}

// Measured (profiles/r1): dW_out 4864 x 896 x 32768 ran at 763 TFLOP/s as 133 128-wide pair tiles
// on 74 pairs (1.8 waves), its transpose 896 x 4864 at 1234 as 133 single-CTA 128 x 256 tiles in
// one wave. Transpose only on a clear (>10%) modelled win; gemm_set_transpose (test hook): 0 = never,
// 1 = modelled (default), 2 = always.
static int g_gemm_transpose = 1;
void gemm_set_transpose(int mode) { g_gemm_transpose = mode; }

bool gemm_prefer_transposed(int M, int N, int K) {
  const int mode = g_gemm_transpose;
  if (mode == 0 || M % 16 != 0 || N % 16 != 0 || M == N) return false;
  if (mode == 2) return true;  // force (tests)
  const int g_num_sms = device_sm_count();
  return gemm_est_cost(N, M, K) < 0.9 * gemm_est_cost(M, N, K);
}

}  // namespace ttb
