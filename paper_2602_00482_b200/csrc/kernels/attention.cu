// Segment attention over the device KV-prefix stack (replaces detail::attention_probs + the PV
// loop, model.hpp:298-321,386-408, and the attention backward, model.hpp:546-604).
//
// A segment batch holds one or more sibling segments that share the stack prefix rows [0, S).
// Query row r of segment i (batch-local offset seg_off, local index t = r - seg_off) attends to
// stack rows [0, S) (full) and to its own rows [S+seg_off, S+seg_off+t] (causal) — no tree mask
// is ever materialised. Heads are packed in columns (head h = cols [h*dh, (h+1)*dh)).
//
// First version: flash-attention-2 style tiling on mma.sync.m16n8k16 (bf16 -> fp32) with
// ldmatrix + cp.async; forward writes O (bf16) and the log-sum-exp per (head, row); backward is
// KV-block parallel: each CTA owns 64 stack rows and loops over the query blocks that see them,
// accumulating dK/dV in registers and adding them into the fp32 dK/dV stack once (red.add),
// dQ via fp32 atomics.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <stdexcept>

#include "attention.h"
#include "sm100.cuh"

namespace ttb {

namespace {

constexpr int kThreads = 128;
constexpr int kBQ = 64;
constexpr int kBK = 64;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = smem_u32(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Load `rows_valid` rows of a [64 x DH] bf16 tile (global row pitch ld) into smem [64][DH+8];
// invalid rows are zero-filled.
template <int DH>
__device__ __forceinline__ void load_tile(__nv_bfloat16 (*dst)[DH + 8], const __nv_bfloat16* src, long ld,
                                          int rows_valid) {
  constexpr int kChunks = DH / 8;  // 16B chunks per row
  for (int i = threadIdx.x; i < 64 * kChunks; i += kThreads) {
    const int r = i / kChunks, c = (i % kChunks) * 8;
    const bool ok = r < rows_valid;
    cp_async16(&dst[r][c], ok ? src + static_cast<long>(r) * ld + c : src, ok);
  }
}

// ---------------------------------------------------------------------------- forward
template <int DH>
__global__ void __launch_bounds__(kThreads) attn_fwd_kernel(AttnFwdArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  using Tile = __nv_bfloat16[kBQ][DH + 8];
  Tile& Qs = *reinterpret_cast<Tile*>(smem_raw);
  Tile* Ks = reinterpret_cast<Tile*>(smem_raw + sizeof(Tile));      // [2]
  Tile* Vs = reinterpret_cast<Tile*>(smem_raw + 3 * sizeof(Tile));  // [2]

  const int4 blk = a.qblocks[blockIdx.x];
  const int q_start = blk.x, q_end = blk.y, seg_off = blk.z;
  const int h = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int g = lane >> 2, c4 = lane & 3;
  const int S = a.S;
  const long col0 = static_cast<long>(h) * DH;

  // KV block list: prefix blocks then own blocks up to the diagonal of this q-block.
  const int n_pre = (S + kBK - 1) / kBK;
  const int own_rows = q_end - seg_off;  // keys needed: own local [0, own_rows)
  const int n_own = (own_rows + kBK - 1) / kBK;
  const int n_blocks = n_pre + n_own;
  const int t_lo = q_start - seg_off;  // smallest query local index in this block

  auto kv_block = [&](int b, long& row0, int& valid, int& kt0) {
    if (b < n_pre) {
      row0 = static_cast<long>(a.pbase) + static_cast<long>(b) * kBK;
      valid = min(kBK, S - b * kBK);
      kt0 = -1;
    } else {
      const int ob = b - n_pre;
      row0 = static_cast<long>(a.r0 < 0 ? S : a.r0) + seg_off + ob * kBK;
      valid = min(kBK, own_rows - ob * kBK);
      kt0 = ob * kBK;
    }
  };
  auto issue_kv = [&](int b, int buf) {
    long row0;
    int valid, kt0;
    kv_block(b, row0, valid, kt0);
    load_tile<DH>(Ks[buf], a.k + row0 * a.ldkv + col0, a.ldkv, valid);
    load_tile<DH>(Vs[buf], a.v + row0 * a.ldkv + col0, a.ldkv, valid);
  };

  load_tile<DH>(Qs, a.q + static_cast<long>(q_start) * a.ldq + col0, a.ldq, q_end - q_start);
  issue_kv(0, 0);
  cp_async_commit();

  uint32_t qf[DH / 16][4];
  float o[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  const float sl2 = a.scale * kLog2e;
  const int t_row0 = t_lo + warp * 16 + g;  // local query index of accumulator row g
  const int t_row1 = t_row0 + 8;

  for (int b = 0; b < n_blocks; ++b) {
    if (b + 1 < n_blocks) {
      issue_kv(b + 1, (b + 1) & 1);
      cp_async_commit();
      cp_async_wait_1();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    if (b == 0) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk)
        ldsm_x4(qf[kk], &Qs[warp * 16 + (lane & 15)][kk * 16 + (lane >> 4) * 8]);
    }
    long row0;
    int valid, kt0;
    kv_block(b, row0, valid, kt0);
    const int buf = b & 1;
    // ---- S = Q K^T (16 x 64 per warp)
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t kb[4];
        ldsm_x4(kb, &Ks[buf][np * 16 + (lane & 7) + ((lane >> 4) << 3)][kk * 16 + ((lane >> 3) & 1) * 8]);
        mma16816(s[2 * np], qf[kk], kb[0], kb[1]);
        mma16816(s[2 * np + 1], qf[kk], kb[2], kb[3]);
      }
    }
    // ---- mask + online softmax (log2 domain)
    float bmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = j * 8 + c4 * 2 + (e & 1);
        const int trow = (e < 2) ? t_row0 : t_row1;
        bool ok = key < valid;
        if (kt0 >= 0) ok = ok && (kt0 + key <= trow);
        const float v = ok ? s[j][e] * sl2 : -INFINITY;
        s[j][e] = v;
        bmax[e >> 1] = fmaxf(bmax[e >> 1], v);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      bmax[r] = fmaxf(bmax[r], __shfl_xor_sync(0xffffffff, bmax[r], 1));
      bmax[r] = fmaxf(bmax[r], __shfl_xor_sync(0xffffffff, bmax[r], 2));
    }
    float corr[2], mref[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float mn = fmaxf(m_r[r], bmax[r]);
      mref[r] = mn == -INFINITY ? 0.f : mn;
      corr[r] = exp2f(m_r[r] - mref[r]);
      m_r[r] = mn;
    }
    float rsum[2] = {0.f, 0.f};
    uint32_t pf[4][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float p0 = exp2f(s[j][0] - mref[0]), p1 = exp2f(s[j][1] - mref[0]);
      const float p2 = exp2f(s[j][2] - mref[1]), p3 = exp2f(s[j][3] - mref[1]);
      rsum[0] += p0 + p1;
      rsum[1] += p2 + p3;
      pf[j >> 1][(j & 1) * 2 + 0] = pack_bf16x2(p0, p1);
      pf[j >> 1][(j & 1) * 2 + 1] = pack_bf16x2(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rsum[r] += __shfl_xor_sync(0xffffffff, rsum[r], 1);
      rsum[r] += __shfl_xor_sync(0xffffffff, rsum[r], 2);
      l_r[r] = l_r[r] * corr[r] + rsum[r];
    }
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    // ---- O += P V   (A = P from registers; pf[kstep] = {a0,a1,a2,a3})
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t afr[4] = {pf[ks][0], pf[ks][1], pf[ks][2], pf[ks][3]};
#pragma unroll
      for (int np = 0; np < DH / 16; ++np) {
        uint32_t vb[4];
        ldsm_x4_t(vb, &Vs[buf][ks * 16 + (lane & 15)][np * 16 + (lane >> 4) * 8]);
        mma16816(o[2 * np], afr, vb[0], vb[1]);
        mma16816(o[2 * np + 1], afr, vb[2], vb[3]);
      }
    }
    __syncthreads();
  }
  // ---- epilogue: O / l, LSE
  const float inv0 = 1.f / l_r[0], inv1 = 1.f / l_r[1];
  const int r0 = q_start + warp * 16 + g, r1 = r0 + 8;
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) {
    const long c = col0 + i * 8 + c4 * 2;
    if (r0 < q_end)
      *reinterpret_cast<uint32_t*>(a.o + static_cast<long>(r0) * a.ldo + c) = pack_bf16x2(o[i][0] * inv0, o[i][1] * inv0);
    if (r1 < q_end)
      *reinterpret_cast<uint32_t*>(a.o + static_cast<long>(r1) * a.ldo + c) = pack_bf16x2(o[i][2] * inv1, o[i][3] * inv1);
  }
  if (c4 == 0) {
    const float ln2 = 0.6931471805599453f;
    if (r0 < q_end) a.lse[static_cast<long>(h) * a.n + r0] = (m_r[0] + log2f(l_r[0])) * ln2;
    if (r1 < q_end) a.lse[static_cast<long>(h) * a.n + r1] = (m_r[1] + log2f(l_r[1])) * ln2;
  }
}

// ---------------------------------------------------------------------------- backward
// smem: Ks, Vs, Qs, dOs : [64][DH+8] bf16 ; dSs [64 keys][64+8 queries] bf16 ; lse2, D : [64] f32
template <int DH>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_kernel(AttnBwdArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  using Tile = __nv_bfloat16[64][DH + 8];
  using STile = __nv_bfloat16[64][64 + 8];
  Tile& Ks = *reinterpret_cast<Tile*>(smem_raw);
  Tile& Vs = *reinterpret_cast<Tile*>(smem_raw + sizeof(Tile));
  Tile& Qs = *reinterpret_cast<Tile*>(smem_raw + 2 * sizeof(Tile));
  Tile& dOs = *reinterpret_cast<Tile*>(smem_raw + 3 * sizeof(Tile));
  STile& dSs = *reinterpret_cast<STile*>(smem_raw + 4 * sizeof(Tile));
  float* lse_s = reinterpret_cast<float*>(smem_raw + 4 * sizeof(Tile) + sizeof(STile));
  float* D_s = lse_s + 64;

  const int4 it = a.items[blockIdx.x];
  const int2 it2 = a.items2[blockIdx.x];
  const long kv0 = it.x;
  const int kv_valid = it.y, q_lo = it.z, q_hi = it.w;
  const int seg_off = it2.x;
  const bool own = it2.y != 0;
  const int kt_base = own ? static_cast<int>(kv0 - (a.r0 < 0 ? a.S : a.r0) - seg_off) : 0;  // local key of row 0
  const int h = blockIdx.y;
  const long col0 = static_cast<long>(h) * DH;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int g = lane >> 2, c4 = lane & 3;
  const float sl2 = a.scale * kLog2e;

  load_tile<DH>(Ks, a.k + kv0 * a.ldkv + col0, a.ldkv, kv_valid);
  load_tile<DH>(Vs, a.v + kv0 * a.ldkv + col0, a.ldkv, kv_valid);
  cp_async_commit();

  float dk[DH / 8][4], dv[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;

  const int key_r0 = warp * 16 + g, key_r1 = key_r0 + 8;  // accumulator rows (keys) of this thread

  for (int q0 = q_lo; q0 < q_hi; q0 += kBQ) {
    const int qn = min(kBQ, q_hi - q0);
    load_tile<DH>(Qs, a.q + static_cast<long>(q0) * a.ldq + col0, a.ldq, qn);
    load_tile<DH>(dOs, a.dO + static_cast<long>(q0) * a.ldq + col0, a.ldq, qn);
    cp_async_commit();
    for (int i = threadIdx.x; i < 64; i += kThreads) {
      const bool ok = i < qn;
      lse_s[i] = ok ? a.lse[static_cast<long>(h) * a.n + q0 + i] * kLog2e : INFINITY;
      D_s[i] = ok ? a.D[static_cast<long>(h) * a.n + q0 + i] : 0.f;
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- S^T = K Q^T  and  dP^T = V dO^T   (16 keys x 64 queries per warp)
    float st[8][4], dpt[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[j][e] = dpt[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
      uint32_t ka[4], va[4];
      ldsm_x4(ka, &Ks[warp * 16 + (lane & 15)][kk * 16 + (lane >> 4) * 8]);
      ldsm_x4(va, &Vs[warp * 16 + (lane & 15)][kk * 16 + (lane >> 4) * 8]);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t qb[4], ob[4];
        ldsm_x4(qb, &Qs[np * 16 + (lane & 7) + ((lane >> 4) << 3)][kk * 16 + ((lane >> 3) & 1) * 8]);
        ldsm_x4(ob, &dOs[np * 16 + (lane & 7) + ((lane >> 4) << 3)][kk * 16 + ((lane >> 3) & 1) * 8]);
        mma16816(st[2 * np], ka, qb[0], qb[1]);
        mma16816(st[2 * np + 1], ka, qb[2], qb[3]);
        mma16816(dpt[2 * np], va, ob[0], ob[1]);
        mma16816(dpt[2 * np + 1], va, ob[2], ob[3]);
      }
    }
    // ---- P^T, dS^T
    uint32_t pa[4][4], dsa[4][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float p[4], ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = j * 8 + c4 * 2 + (e & 1);
        const int key = (e < 2) ? key_r0 : key_r1;
        bool ok = key < kv_valid && qi < qn;
        if (own) ok = ok && (kt_base + key <= q0 + qi - seg_off);
        p[e] = ok ? exp2f(st[j][e] * sl2 - lse_s[qi]) : 0.f;
        ds[e] = p[e] * (dpt[j][e] - D_s[qi]);
      }
      pa[j >> 1][(j & 1) * 2 + 0] = pack_bf16x2(p[0], p[1]);
      pa[j >> 1][(j & 1) * 2 + 1] = pack_bf16x2(p[2], p[3]);
      dsa[j >> 1][(j & 1) * 2 + 0] = pack_bf16x2(ds[0], ds[1]);
      dsa[j >> 1][(j & 1) * 2 + 1] = pack_bf16x2(ds[2], ds[3]);
      // stash dS^T (keys x queries) for the dQ product
      *reinterpret_cast<uint32_t*>(&dSs[key_r0][j * 8 + c4 * 2]) = dsa[j >> 1][(j & 1) * 2 + 0];
      *reinterpret_cast<uint32_t*>(&dSs[key_r1][j * 8 + c4 * 2]) = dsa[j >> 1][(j & 1) * 2 + 1];
    }
    // ---- dV += P^T dO ; dK += dS^T Q   (k = queries)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int np = 0; np < DH / 16; ++np) {
        uint32_t ob[4], qb[4];
        ldsm_x4_t(ob, &dOs[ks * 16 + (lane & 15)][np * 16 + (lane >> 4) * 8]);
        ldsm_x4_t(qb, &Qs[ks * 16 + (lane & 15)][np * 16 + (lane >> 4) * 8]);
        mma16816(dv[2 * np], pa[ks], ob[0], ob[1]);
        mma16816(dv[2 * np + 1], pa[ks], ob[2], ob[3]);
        mma16816(dk[2 * np], dsa[ks], qb[0], qb[1]);
        mma16816(dk[2 * np + 1], dsa[ks], qb[2], qb[3]);
      }
    }
    __syncthreads();
    // ---- dQ[q0 + 16w .. +16] += dS K * scale, in 32-column chunks
    {
      uint32_t af[4][4];
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        // A[m = query][k = key] from dSs stored [key][query]: transposed 8x8 loads
        const int key = ks * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int qq = warp * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4_t(af[ks], &dSs[key][qq]);
      }
      const int qr0 = q0 + warp * 16 + g, qr1 = qr0 + 8;
#pragma unroll
      for (int cc = 0; cc < DH / 32; ++cc) {
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
          for (int np = 0; np < 2; ++np) {
            uint32_t kb[4];
            ldsm_x4_t(kb, &Ks[ks * 16 + (lane & 15)][cc * 32 + np * 16 + (lane >> 4) * 8]);
            mma16816(acc[2 * np], af[ks], kb[0], kb[1]);
            mma16816(acc[2 * np + 1], af[ks], kb[2], kb[3]);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const long c = col0 + cc * 32 + i * 8 + c4 * 2;
          if (qr0 < q0 + qn) {
            atomicAdd(a.dq + static_cast<long>(qr0) * a.lddq + c, acc[i][0] * a.scale);
            atomicAdd(a.dq + static_cast<long>(qr0) * a.lddq + c + 1, acc[i][1] * a.scale);
          }
          if (qr1 < q0 + qn) {
            atomicAdd(a.dq + static_cast<long>(qr1) * a.lddq + c, acc[i][2] * a.scale);
            atomicAdd(a.dq + static_cast<long>(qr1) * a.lddq + c + 1, acc[i][3] * a.scale);
          }
        }
      }
    }
    __syncthreads();
  }
  // ---- add dK (scaled) / dV into the fp32 stack rows this CTA owns
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) {
    const long c = col0 + i * 8 + c4 * 2;
    if (key_r0 < kv_valid) {
      float* pk = a.dk + (kv0 + key_r0) * a.lddkv + c;
      float* pv = a.dv + (kv0 + key_r0) * a.lddkv + c;
      atomicAdd(pk, dk[i][0] * a.scale);
      atomicAdd(pk + 1, dk[i][1] * a.scale);
      atomicAdd(pv, dv[i][0]);
      atomicAdd(pv + 1, dv[i][1]);
    }
    if (key_r1 < kv_valid) {
      float* pk = a.dk + (kv0 + key_r1) * a.lddkv + c;
      float* pv = a.dv + (kv0 + key_r1) * a.lddkv + c;
      atomicAdd(pk, dk[i][2] * a.scale);
      atomicAdd(pk + 1, dk[i][3] * a.scale);
      atomicAdd(pv, dv[i][2]);
      atomicAdd(pv + 1, dv[i][3]);
    }
  }
}

// D[h][r] = sum_c dO[r, h*dh+c] * O[r, h*dh+c]
// D[h][r] = rowsum(dO * O) over head h's dh columns: one thread per 8 columns (16-byte loads), a
// group of dh/8 lanes per (row, head) reduces with shuffles.
__global__ void attn_bwd_pre_kernel(const __nv_bfloat16* __restrict__ dO, const __nv_bfloat16* __restrict__ O,
                                    long ld, float* __restrict__ D, int n, int H, int dh) {
  const long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int gpr = dh / 8;  // threads per (row, head): 8 or 16
  const int cols8 = H * gpr;
  const long r = t / cols8;
  const int j = static_cast<int>(t - r * cols8);
  float s = 0.f;
  if (r < n) {
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

template <int DH>
size_t fwd_smem() {
  return 5 * sizeof(__nv_bfloat16) * kBQ * (DH + 8);
}
template <int DH>
size_t bwd_smem() {
  return 4 * sizeof(__nv_bfloat16) * 64 * (DH + 8) + sizeof(__nv_bfloat16) * 64 * 72 + 2 * 64 * sizeof(float);
}

}  // namespace

void attn_fwd(const AttnFwdArgs& a, cudaStream_t stream) {
  if (a.nqb == 0) return;
  dim3 grid(a.nqb, a.H);
  if (a.dh == 64) {
    static bool once = (cudaFuncSetAttribute(attn_fwd_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(fwd_smem<64>())),
                        true);
    (void)once;
    attn_fwd_kernel<64><<<grid, kThreads, fwd_smem<64>(), stream>>>(a);
  } else if (a.dh == 128) {
    static bool once = (cudaFuncSetAttribute(attn_fwd_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(fwd_smem<128>())),
                        true);
    (void)once;
    attn_fwd_kernel<128><<<grid, kThreads, fwd_smem<128>(), stream>>>(a);
  } else {
    throw std::invalid_argument("attention: head_dim must be 64 or 128");
  }
}

void attn_bwd_pre(const AttnBwdArgs& a, cudaStream_t stream) {
  const long threads = static_cast<long>(a.n) * a.H * (a.dh / 8);
  if (a.ldq % 8 != 0) throw std::invalid_argument("attention backward: dO/O pitch must be a multiple of 8");
  if (threads > 0)
    attn_bwd_pre_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(a.dO, a.o, a.ldq, a.D, a.n,
                                                                                         a.H, a.dh);
}

void attn_bwd(const AttnBwdArgs& a, cudaStream_t stream) {
  attn_bwd_pre(a, stream);
  if (a.nitems == 0) return;
  dim3 grid(a.nitems, a.H);
  if (a.dh == 64) {
    static bool once = (cudaFuncSetAttribute(attn_bwd_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(bwd_smem<64>())),
                        true);
    (void)once;
    attn_bwd_kernel<64><<<grid, kThreads, bwd_smem<64>(), stream>>>(a);
  } else if (a.dh == 128) {
    static bool once = (cudaFuncSetAttribute(attn_bwd_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(bwd_smem<128>())),
                        true);
    (void)once;
    attn_bwd_kernel<128><<<grid, kThreads, bwd_smem<128>(), stream>>>(a);
  } else {
    throw std::invalid_argument("attention: head_dim must be 64 or 128");
  }
}

}  // namespace ttb
