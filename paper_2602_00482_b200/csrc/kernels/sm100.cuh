// sm_100a primitives: mbarrier, TMA (cp.async.bulk.tensor), tcgen05 (MMA, TMEM alloc/ld),
// UMMA shared-memory / instruction descriptors. Raw inline PTX, no CUTLASS dependency.
//
// Descriptor bit layouts follow the PTX ISA "tcgen05 matrix descriptors" and
// "instruction descriptor" tables (kind::f16): see DESIGN.md §Kernels.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

namespace ttb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 1024-byte aligned base of the dynamic shared memory (the SWIZZLE_128B atom alignment). Pointer
// arithmetic on the __shared__ array (not a uintptr_t round trip) keeps the shared address space
// visible to the compiler, so accesses through it compile to LDS/STS rather than generic LD/ST.
__device__ __forceinline__ uint8_t* align_smem_1024(uint8_t* raw) {
  return raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint32_t mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok;
}
// Non-blocking probe of the phase (mbarrier.test_wait): the fast path of a wait whose phase has most
// likely completed already (try_wait costs ~200 clk even then).
__device__ __forceinline__ uint32_t mbar_test_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Blocking wait on the phase with the given parity. A wait that does not complete within ~4 s is a
// pipeline bug: report the barrier and trap (the launch fails loudly instead of hanging the GPU).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity);
// The same with a non-blocking test first (consumers that usually find the phase complete).
__device__ __forceinline__ void mbar_wait_fast(uint64_t* bar, uint32_t parity) {
  if (mbar_test_wait(smem_u32(bar), parity)) return;
  mbar_wait(bar, parity);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const uint64_t t0 = globaltimer_ns();
  while (!mbar_try_wait(addr, parity)) {
    if (globaltimer_ns() - t0 > 4000000000ull) {
      printf("ttb: mbarrier timeout bar=0x%x parity=%u block=(%d,%d) thread=%d\n", addr, parity, blockIdx.x,
             blockIdx.y, threadIdx.x);
      __trap();
    }
  }
}

// ---------------------------------------------------------------- programmatic dependent launch
// (kernels/launch.cuh): block until the predecessor grid has completed and its writes are visible (a
// no-op when launched without the PDL attribute); let the successor grid start its prologue.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// TMEM-holding kernels release their successor either right after the prologue (early) or when the
// CTA's work is done (late, TT_PDL_LATE=1 experiment builds).
#ifndef TT_PDL_LATE
#define TT_PDL_LATE 0
#endif
__device__ __forceinline__ void pdl_trigger_early() {
  if (!TT_PDL_LATE) pdl_trigger();
}
__device__ __forceinline__ void pdl_trigger_late() {
  if (TT_PDL_LATE) pdl_trigger();
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(const void* tmap, uint64_t* bar, void* smem_dst, int32_t x,
                                            int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_result, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accum). Issued by one thread.
__device__ __forceinline__ void umma_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T  (A operand from TMEM, e.g. P in attention).
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns: thread t of the warp gets lane (quadrant*32+t).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- UMMA descriptors
// Shared-memory matrix descriptor, SWIZZLE_128B (layout type 2), sm_100 version bit (46) = 1.
//   K-major  tile: rows of 128 B (64 bf16 along K), 8-row atoms 1024 B apart  -> SBO = 1024, LBO unused.
//   MN-major tile: 64-element MN atoms (128 B) stacked over K rows (128 B apart); 8-K-row groups
//                  SBO apart (1024 B); successive MN atoms LBO apart.
__device__ __forceinline__ uint64_t make_sdesc_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version = 1 (Blackwell)
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

// Descriptor of (the address of desc) + off bytes: the start-address field holds addr >> 4 in its low
// 14 bits and shared-memory addresses stay below 2^18, so a plain add never carries out of it. Lets
// an MMA issuer build every descriptor from one precomputed base with a single integer add.
__device__ __forceinline__ uint64_t sdesc_add(uint64_t desc, uint32_t off_bytes) { return desc + (off_bytes >> 4); }

// Instruction descriptor, kind::f16: A,B bf16, D fp32.
__host__ __device__ constexpr uint32_t make_idesc_bf16(int M, int N, bool a_mn_major, bool b_mn_major) {
  return (1u << 4)                                   // c_format = F32
         | (1u << 7)                                 // a_format = BF16
         | (1u << 10)                                // b_format = BF16
         | ((a_mn_major ? 1u : 0u) << 15)            // a_major
         | ((b_mn_major ? 1u : 0u) << 16)            // b_major
         | ((static_cast<uint32_t>(N) >> 3) << 17)   // n_dim
         | ((static_cast<uint32_t>(M) >> 4) << 24);  // m_dim
}

// TMEM column of the bf16 A-operand k-step k (16 elements = 8 packed columns) when two softmax
// warps each own HALF columns of a fp32 buffer and pack their bf16 results into the start of their own
// half: elements [h*HALF, (h+1)*HALF) sit at columns h*HALF + (e - h*HALF)/2.
template <int HALF>
__device__ __forceinline__ uint32_t packed_col(int k) {
  return static_cast<uint32_t>((k * 16 / HALF) * HALF + (k * 16 % HALF) / 2);
}

// ---------------------------------------------------------------- exp2
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA/ALU pipes (no MUFU): round-to-nearest split x = j + f, f in [-0.5, 0.5] via the
// 1.5*2^23 magic add, cubic minimax 2^f (max rel err 7.5e-5, far below bf16's 3.9e-3), exponent
// added as an integer. Used for a fraction of the softmax exponentials so the MUFU (16/clk/SM) and
// FMA (128/clk/SM) pipes share the load. x < -126 (incl. -inf) -> 0.
__device__ __forceinline__ float ex2_poly(float x) {
  const float xc = fmaxf(x, -126.0f);
  const float t = xc + 12582912.0f;  // 0x1.8p23: low mantissa bits = round(xc)
  const float j = t - 12582912.0f;
  const float f = xc - j;
  const float pz = fmaf(fmaf(fmaf(0.05517084f, f, 0.24260935f), f, 0.69326096f), f, 0.99992818f);
  const int ji = __float_as_int(t) - 0x4B400000;
  const float r = __int_as_float(__float_as_int(pz) + (ji << 23));
  return x < -126.0f ? 0.0f : r;
}

// Paired variant on FFMA2/FADD2 (two exponentials per issue of each step). x is clamped to
// [-126, +inf) so masked (-inf) inputs give ~2^-126 instead of 0 — below every bf16/fp32 sum they
// enter. The exponent add uses (t_bits << 23): the 1.5*2^23 bias bits vanish mod 2^32.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.0f);
  x.y = fmaxf(x.y, -126.0f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.0f, 12582912.0f));
  const float2 j = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = __ffma2_rn(j, make_float2(-1.0f, -1.0f), x);
  float2 pz = __ffma2_rn(make_float2(0.05517084f, 0.05517084f), f, make_float2(0.24260935f, 0.24260935f));
  pz = __ffma2_rn(pz, f, make_float2(0.69326096f, 0.69326096f));
  pz = __ffma2_rn(pz, f, make_float2(0.99992818f, 0.99992818f));
  return make_float2(__int_as_float(__float_as_int(pz.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(pz.y) + (__float_as_int(t.y) << 23)));
}
// 3-input max (FMNMX3, sm_100+).
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// ---------------------------------------------------------------- misc
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void red_add_v4_f32(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ void red_add_v2_f32(float* addr, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ int warp_id_sync() { return __shfl_sync(0xffffffff, threadIdx.x / 32, 0); }
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t"
      ".reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}

}  // namespace ttb
