// HBM-bound kernels of the push/pop path: embedding + positional encoding, RMSNorm fwd/bwd,
// fused weighted cross-entropy over a vocab row, stack pop (dK/dV consume + zero), embedding
// gradient scatter, parameter layout conversion / init. 128-bit coalesced accesses throughout.
#include <algorithm>
#include <cstdlib>
#include <cuda_bf16.h>
#include <stdexcept>
#include <cuda_runtime.h>

#include "elementwise.h"
#include "gemm.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace ttb {

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffff, v, o));
  return v;
}
// Block-wide sum for blockDim.x == 256; returns the total to every thread.
__device__ __forceinline__ float block_sum256(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = l < 8 ? red[l] : 0.f;
  return warp_sum(t);
}

// x[r] = E[tok[r]] + PE[pos[r]]  (model.hpp:363-369, add_positional_encoding :239-248)
__global__ void embed_pe_kernel(const int32_t* __restrict__ tok, const int32_t* __restrict__ pos,
                                const __nv_bfloat16* __restrict__ emb, const float* __restrict__ pe,
                                float* __restrict__ x, int d) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  const int r = blockIdx.x;
  const long e0 = static_cast<long>(tok[r]) * d, p0 = static_cast<long>(pos[r]) * d, x0 = static_cast<long>(r) * d;
  for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
    const uint2 eb = *reinterpret_cast<const uint2*>(emb + e0 + c);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&eb.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&eb.y));
    const float4 p = *reinterpret_cast<const float4*>(pe + p0 + c);
    *reinterpret_cast<float4*>(x + x0 + c) = make_float4(a.x + p.x, a.y + p.y, b.x + p.z, b.y + p.w);
  }
}

// inv = 1/sqrt(mean(x^2)+eps); y = x*inv*g (bf16)   (rms_inv model.hpp:250-256; apply :377-380)
// WPR warps per row (8 / WPR rows per 256-thread block); each lane holds VPT float4 column groups
// (c = (lr + 32 WPR k) * 4) in registers, so x is read from HBM once. WPR > 1 keeps VPT <= 16 for
// rows wider than 4096 (the sum of squares is then combined across the row's warps in smem).
template <int VPT, int WPR = 1>
__global__ void __launch_bounds__(256) rmsnorm_fwd_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                                                          float* __restrict__ inv, __nv_bfloat16* __restrict__ y, int n,
                                                          int d) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  constexpr int STRIDE = 32 * WPR;
  __shared__ float red[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * (8 / WPR) + warp / WPR;
  const int lr = (warp % WPR) * 32 + lane;
  const bool valid = row < n;
  if (WPR == 1 && !valid) return;
  const float* xr = x + static_cast<long>(row) * d;
  float4 v[VPT];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = (lr + STRIDE * k) * 4;
    v[k] = (valid && c < d) ? __ldcs(reinterpret_cast<const float4*>(xr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    s += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
  }
  s = warp_sum(s);
  if constexpr (WPR > 1) {
    if (lane == 0) red[warp] = s;
    __syncthreads();
    s = 0.f;
#pragma unroll
    for (int j = 0; j < WPR; ++j) s += red[(warp / WPR) * WPR + j];
    if (!valid) return;
  }
  const float iv = 1.0f / sqrtf(s / static_cast<float>(d) + 1e-6f);
  if (lr == 0) inv[row] = iv;
  __nv_bfloat16* yr = y + static_cast<long>(row) * d;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = (lr + STRIDE * k) * 4;
    if (c < d) {
      const float4 g = __ldg(reinterpret_cast<const float4*>(gain + c));
      uint2 o;
      o.x = pack_bf16x2(v[k].x * iv * g.x, v[k].y * iv * g.y);
      o.y = pack_bf16x2(v[k].z * iv * g.z, v[k].w * iv * g.w);
      *reinterpret_cast<uint2*>(yr + c) = o;
    }
  }
}

// rmsnorm_backward (model.hpp:258-271), WPR warps per row, row groups strided over a ~2-wave grid:
//   gx = gres + gy*g*inv - x*(sum(gy*g*x)*inv^3/d);  ggain += sum_rows gy*x*inv
// Each lane of a row group owns VPT float4 columns (c = (lr + 32 WPR k) * 4, lr = lane within the
// group); the row is held in registers, the dot product is reduced across the group's warps through
// shared memory (double-buffered, one barrier per row step), the gain-gradient partial stays in
// registers for all of the group's rows, is reduced across the block in shared memory and lands with
// one red.global.add.v4 per column group. WPR > 1 keeps VPT <= 8 for wide rows (d = 3584: one warp
// per row needed 28 float4 per lane, 254 registers, 8 warps per SM and 1.6 TB/s).
template <int VPT, int WPR>
__global__ void __launch_bounds__(256) rmsnorm_bwd_kernel(const float* __restrict__ gy, const float* __restrict__ x,
                                                          const float* __restrict__ inv, const float* __restrict__ gain,
                                                          const float* gres, float* gx, __nv_bfloat16* __restrict__ gxb,
                                                          float* __restrict__ ggain, int n, int d) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  constexpr int RPB = 8 / WPR;     // rows per block step
  constexpr int STRIDE = 32 * WPR;  // float4 column stride between a lane's groups
  extern __shared__ float gsum[];  // [d]
  __shared__ float red[2][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rloc = warp / WPR, lr = (warp % WPR) * 32 + lane;
  for (int c = threadIdx.x; c < d; c += 256) gsum[c] = 0.f;
  float4 gacc[VPT], av[VPT], bv[VPT];
#pragma unroll
  for (int k = 0; k < VPT; ++k) gacc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  int step = 0;
  for (int base = blockIdx.x * RPB; base < n; base += gridDim.x * RPB, ++step) {
    const int r = base + rloc;
    const bool valid = r < n;
    const long o = static_cast<long>(r) * d;
    const float iv = valid ? inv[r] : 0.f;
    float dot = 0.f;
    if (valid) {
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int c = (lr + k * STRIDE) * 4;
        if (c < d) {
          const float4 a = __ldcs(reinterpret_cast<const float4*>(gy + o + c));
          const float4 b = *reinterpret_cast<const float4*>(x + o + c);
          const float4 g = __ldg(reinterpret_cast<const float4*>(gain + c));
          dot += a.x * g.x * b.x + a.y * g.y * b.y + a.z * g.z * b.z + a.w * g.w * b.w;
          av[k] = a;
          bv[k] = b;
        }
      }
    }
    dot = warp_sum(dot);
    if constexpr (WPR > 1) {
      if (lane == 0) red[step & 1][warp] = dot;
      __syncthreads();
      dot = 0.f;
#pragma unroll
      for (int j = 0; j < WPR; ++j) dot += red[step & 1][rloc * WPR + j];
    }
    if (!valid) continue;
    const float scale = dot * iv * iv * iv / static_cast<float>(d);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = (lr + k * STRIDE) * 4;
      if (c < d) {
        const float4 a = av[k], b = bv[k];
        const float4 g = __ldg(reinterpret_cast<const float4*>(gain + c));
        float4 res = gres ? *reinterpret_cast<const float4*>(gres + o + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        res.x += a.x * g.x * iv - b.x * scale;
        res.y += a.y * g.y * iv - b.y * scale;
        res.z += a.z * g.z * iv - b.z * scale;
        res.w += a.w * g.w * iv - b.w * scale;
        *reinterpret_cast<float4*>(gx + o + c) = res;
        uint2 pb;
        pb.x = pack_bf16x2(res.x, res.y);
        pb.y = pack_bf16x2(res.z, res.w);
        *reinterpret_cast<uint2*>(gxb + o + c) = pb;
        gacc[k].x += a.x * b.x * iv;
        gacc[k].y += a.y * b.y * iv;
        gacc[k].z += a.z * b.z * iv;
        gacc[k].w += a.w * b.w * iv;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = (lr + k * STRIDE) * 4;
    if (c < d) {
      atomicAdd(gsum + c, gacc[k].x);
      atomicAdd(gsum + c + 1, gacc[k].y);
      atomicAdd(gsum + c + 2, gacc[k].z);
      atomicAdd(gsum + c + 3, gacc[k].w);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x * 4; c < d; c += 1024) red_add_v4_f32(ggain + c, gsum[c], gsum[c + 1], gsum[c + 2], gsum[c + 3]);
}

template <int VPT, int WPR>
void launch_rmsnorm_bwd(const float* gy, const float* x, const float* inv, const float* gain, const float* gres,
                        float* gx, __nv_bfloat16* gxb, float* ggain, int n, int d, cudaStream_t s) {
  constexpr int RPB = 8 / WPR;
  static const int per_sm = [] {  // resident blocks per SM (registers bound it), one wave of them
    int b = 2;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rmsnorm_bwd_kernel<VPT, WPR>, 256, 8192 * sizeof(float));
    return std::max(1, b);
  }();
  const int blocks = std::min((n + RPB - 1) / RPB, 148 * per_sm);
  launch_k(rmsnorm_bwd_kernel<VPT, WPR>, dim3(blocks), dim3(256), d * sizeof(float), s, gy, x, inv, gain, gres, gx, gxb, ggain, n, d);
}

// rmsnorm_backward fed by TMA (rows up to 4096 columns): a persistent block per SM streams each of its
// rows' gy / x / gres into an NST-deep shared-memory ring with cp.async.bulk (mbarrier complete_tx);
// NCW consumer warps take the rows round-robin (warp w: the block's rows k = w (mod NCW); NST is a
// multiple of NCW, so stage k % NST belongs to warp k % NCW and is used in order — no warp can wait on
// a stage's next phase while its current one is pending). Each consumer warp refills the stage it just
// read with its row k + NST (TT_NORM_SELFLOAD): the single producer thread of the first version spent
// an empty-barrier wait and three bulk copies per row for all ~221 rows of an SM, which at the
// power-capped in-step clock (~1.46 GHz) held the c2 kernel at 4.1-4.7 TB/s; self-refilling runs it
// at 5.5 TB/s in-step (profiles/r2/rmsnorm_selfload_ab.txt). The
// ring keeps ~170 KB of rows in flight per SM independently of the consumers' reduce-then-store
// latency, which is what bounded the register version (one HBM round trip for gy / x, a second for
// gres, 16 warps per SM: 4.1-4.5 TB/s). Each consumer reads its row from shared memory twice (dot
// product, then outputs) instead of holding it in registers; the gain sits in registers (VPT <= 16) or
// in shared memory (GS, wider rows); the gain-gradient partials stay in registers for all of a warp's
// rows and leave through shared memory + one red.global.add.v4 per column group.
__device__ __forceinline__ void bulk_load_1d(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

#ifndef TT_NORM_SELFLOAD
#define TT_NORM_SELFLOAD 1  // consumer warps refill their own ring stages (0: one producer thread; A/B)
#endif
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
constexpr int kNormTmaThreads = 288;  // up to 8 consumer warps + warp 8 (the producer of TT_NORM_SELFLOAD=0 builds)

// GyT: fp32 gy, or bf16 gy (the grad_normed outputs of the dX GEMMs: 2 of the 18 bytes per element)
template <int VPT, bool GS, typename GyT = float>
__global__ void __launch_bounds__(kNormTmaThreads, 1)
    rmsnorm_bwd_tma_kernel(const GyT* __restrict__ gy, const float* __restrict__ x, const float* __restrict__ inv,
                           const float* __restrict__ gain, const float* gres, float* gx, __nv_bfloat16* __restrict__ gxb,
                           float* __restrict__ ggain, int n, int d, int nst, int ncw) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int row_bytes = d * 4;
  const int gy_bytes = d * static_cast<int>(sizeof(GyT));
  const int stage_bytes = gy_bytes + (gres ? 2 : 1) * row_bytes;  // [gy | x | gres]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + nst;
  float* gsum = reinterpret_cast<float*>(empty + nst);  // [d]
  float* gsm = gsum + d;                                 // [d] gain copy (GS)
  uint8_t* ring = smem_raw + ((nst * 16 + 2 * d * 4 + 127) / 128) * 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    gsum[c] = 0.f;
    if (GS) gsm[c] = gain[c];
  }
  __syncthreads();
  const int rows_mine = n > static_cast<int>(blockIdx.x) ? (n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // row k's gy / x / gres into stage k % nst (one thread)
  auto issue = [&](int k) {
    const int st = k % nst;
    const long r = blockIdx.x + static_cast<long>(k) * gridDim.x;
    uint8_t* b = ring + static_cast<long>(st) * stage_bytes;
    mbar_arrive_expect_tx(&full[st], stage_bytes);
    bulk_load_1d(b, gy + r * d, gy_bytes, &full[st]);
    bulk_load_1d(b + gy_bytes, x + r * d, row_bytes, &full[st]);
    if (gres) bulk_load_1d(b + gy_bytes + row_bytes, gres + r * d, row_bytes, &full[st]);
  };
#if TT_NORM_SELFLOAD
  // every consumer warp refills its own stages (stage k % nst belongs to warp k % ncw): no producer
  // thread serialising ~221 rows x (empty wait + 3 bulk copies) per launch, no empty barriers; warp 8
  // idles
  if (warp < ncw && lane == 0)
    for (int k = warp; k < rows_mine && k < nst; k += ncw) issue(k);
#else
  if (warp == 8 && lane == 0) {  // the single producer (A/B builds)
    for (int k = 0; k < rows_mine; ++k) {
      mbar_wait(&empty[k % nst], ((k / nst) & 1) ^ 1);
      issue(k);
    }
  }
#endif
  if (warp < ncw) {
    float4 g[GS ? 1 : VPT], gacc[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = (lane + 32 * k) * 4;
      if constexpr (!GS) g[k] = c < d ? __ldg(reinterpret_cast<const float4*>(gain + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
      gacc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    auto gain4 = [&](int q, int c) {
      if constexpr (GS) return *reinterpret_cast<const float4*>(gsm + c);
      else return g[q];
    };
    for (int k = warp; k < rows_mine; k += ncw) {
      const int st = k % nst;
      const long r = blockIdx.x + static_cast<long>(k) * gridDim.x;
      const float iv = inv[r];  // issued before the wait: its latency overlaps the ring
      mbar_wait(&full[st], (k / nst) & 1);
      const uint8_t* stage = ring + static_cast<long>(st) * stage_bytes;
      const GyT* sgy = reinterpret_cast<const GyT*>(stage);
      const float* sx = reinterpret_cast<const float*>(stage + gy_bytes);
      const float* sres = sx + d;
      auto gy4 = [&](int c) {
        if constexpr (sizeof(GyT) == 4) {
          return *reinterpret_cast<const float4*>(sgy + c);
        } else {
          const uint2 w = *reinterpret_cast<const uint2*>(sgy + c);
          return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u), __uint_as_float(w.y << 16),
                             __uint_as_float(w.y & 0xffff0000u));
        }
      };
      float dot = 0.f;
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        const int c = (lane + 32 * q) * 4;
        if (c < d) {
          const float4 a = gy4(c);
          const float4 b = *reinterpret_cast<const float4*>(sx + c);
          const float4 gq = gain4(q, c);
          dot += a.x * gq.x * b.x + a.y * gq.y * b.y + a.z * gq.z * b.z + a.w * gq.w * b.w;
        }
      }
      dot = warp_sum(dot);
      const float scale = dot * iv * iv * iv / static_cast<float>(d);
      float* gxr = gx + r * d;
      __nv_bfloat16* gxbr = gxb + r * d;
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        const int c = (lane + 32 * q) * 4;
        if (c < d) {
          const float4 a = gy4(c);
          const float4 b = *reinterpret_cast<const float4*>(sx + c);
          const float4 gq = gain4(q, c);
          float4 res = gres ? *reinterpret_cast<const float4*>(sres + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          res.x += a.x * gq.x * iv - b.x * scale;
          res.y += a.y * gq.y * iv - b.y * scale;
          res.z += a.z * gq.z * iv - b.z * scale;
          res.w += a.w * gq.w * iv - b.w * scale;
          __stcs(reinterpret_cast<float4*>(gxr + c), res);
          uint2 pb;
          pb.x = pack_bf16x2(res.x, res.y);
          pb.y = pack_bf16x2(res.z, res.w);
          *reinterpret_cast<uint2*>(gxbr + c) = pb;
          gacc[q].x += a.x * b.x * iv;
          gacc[q].y += a.y * b.y * iv;
          gacc[q].z += a.z * b.z * iv;
          gacc[q].w += a.w * b.w * iv;
        }
      }
#if TT_NORM_SELFLOAD
      // this warp's reads of the stage are done: refill it with row k + nst (generic-proxy reads
      // ordered before the async-proxy writes)
      fence_async_shared();
      __syncwarp();
      if (lane == 0 && k + nst < rows_mine) issue(k + nst);
#else
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
#endif
    }
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int c = (lane + 32 * q) * 4;
      if (c < d) {
        atomicAdd(gsum + c, gacc[q].x);
        atomicAdd(gsum + c + 1, gacc[q].y);
        atomicAdd(gsum + c + 2, gacc[q].z);
        atomicAdd(gsum + c + 3, gacc[q].w);
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x * 4; c < d; c += 4 * blockDim.x)
    red_add_v4_f32(ggain + c, gsum[c], gsum[c + 1], gsum[c + 2], gsum[c + 3]);
}

template <int VPT, bool GS, typename GyT = float>
void launch_rmsnorm_bwd_tma(const GyT* gy, const float* x, const float* inv, const float* gain, const float* gres,
                            float* gx, __nv_bfloat16* gxb, float* ggain, int n, int d, cudaStream_t s) {
  constexpr int kSmemMax = 227 * 1024;
  const int stage_bytes = d * static_cast<int>(sizeof(GyT)) + (gres ? 2 : 1) * d * 4;
  const int head = ((16 * 32 + 2 * d * 4 + 127) / 128) * 128;  // barriers (<= 32 stages) + gsum + gain copy
  const int fit = std::min(32, (kSmemMax - head - 1024) / stage_bytes);
  // consumer warps: 8 when 8 stages fit, else 4 / 2 (stage k % nst must belong to warp k % ncw)
  const int ncw = fit >= 8 ? 8 : (fit >= 4 ? 4 : 2);
  const int nst = fit / ncw * ncw;
  if (nst < 2) throw std::invalid_argument("rmsnorm backward: row too wide for the TMA ring");
  const int smem = ((nst * 16 + 2 * d * 4 + 127) / 128) * 128 + nst * stage_bytes;
  ensure_smem_attr(reinterpret_cast<const void*>(rmsnorm_bwd_tma_kernel<VPT, GS, GyT>), kSmemMax);
  const int blocks = std::min(n, device_sm_count());
  launch_k(rmsnorm_bwd_tma_kernel<VPT, GS, GyT>, dim3(blocks), dim3(kNormTmaThreads), smem, s, gy, x, inv, gain, gres, gx, gxb, ggain, n, d, nst, ncw);
}

// Weighted NLL over one vocab row with several (target, weight) pairs (weighted_nll,
// model.hpp:643-677, extended to multi-target rows):
//   loss += sum_j w_j (lse - l[t_j])  (fp64);  dl = (sum_j w_j) softmax(l) - sum_j w_j onehot(t_j)  (bf16)
__device__ __forceinline__ float4 ld_evict_last_f4(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// Persistent: one 1024-thread CTA per SM walks rows. Pass 1 streams the row with an L2 evict_last
// policy (the ~148 rows in flight fit in the 126 MB L2), pass 2 re-reads it from L2 (evict_first)
// and writes dlogits, so HBM sees each logit once. With `stats` (per-32-column (max, sum) from the
// LM-head GEMM epilogue) pass 1 reads only the statistics.
// 512 threads, 4 CTAs (rows) per SM; the write pass keeps 4 float4 loads per thread in flight
// (64 KB per SM) — one float4 per thread is far too little memory-level parallelism for HBM.
constexpr int kCeThreads = 512;
// OutT = bf16: the tree step's dlogits (operand of the head GEMMs); float: the standalone
// weighted_nll's fp32 grad_logits (LossResult::grad_logits, model.hpp:637-640).
template <typename OutT>
__device__ __forceinline__ void st_grad4(OutT* p, float a, float b, float c, float d);
template <>
__device__ __forceinline__ void st_grad4<__nv_bfloat16>(__nv_bfloat16* p, float a, float b, float c, float d) {
  *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16x2(a, b), pack_bf16x2(c, d));
}
template <>
__device__ __forceinline__ void st_grad4<float>(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void st_grad1(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
__device__ __forceinline__ void st_grad1(float* p, float v) { *p = v; }

template <typename OutT>
__global__ void __launch_bounds__(kCeThreads, 4) ce_kernel(const float* __restrict__ logits, int m, long V,
                                                  const int32_t* __restrict__ pair_off,
                                                  const int32_t* __restrict__ tgt, const double* __restrict__ w,
                                                  OutT* __restrict__ dl, double* __restrict__ loss,
                                                  const float2* __restrict__ stats, int n_groups) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  __shared__ float red[32];
  __shared__ float s_lse;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  const int wi = threadIdx.x >> 5, ln = threadIdx.x & 31;
  for (int r = blockIdx.x; r < m; r += gridDim.x) {
    const float* lr = logits + static_cast<long>(r) * V;
    float mx = -INFINITY, s = 0.f;
    if (stats) {
      const float2* sr = stats + static_cast<long>(r) * n_groups;
      for (int g = threadIdx.x; g < n_groups; g += kCeThreads) {
        const float2 ms = sr[g];
        if (ms.x > mx) {
          s = s * __expf(mx - ms.x) + ms.y;
          mx = ms.x;
        } else {
          s += ms.y * __expf(ms.x - mx);
        }
      }
    } else {
      for (long c = threadIdx.x * 4; c < V; c += 4 * kCeThreads) {
        const float4 v = ld_evict_last_f4(lr + c, pol);
        const float vm = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
        if (vm > mx) {
          s *= __expf(mx - vm);
          mx = vm;
        }
        s += __expf(v.x - mx) + __expf(v.y - mx) + __expf(v.z - mx) + __expf(v.w - mx);
      }
    }
    // combine (max, sum) across the block
    float gm = warp_max(mx);
    if (ln == 0) red[wi] = gm;
    __syncthreads();
    gm = warp_max(ln < kCeThreads / 32 ? red[ln] : -INFINITY);
    __syncthreads();
    s = (mx == -INFINITY) ? 0.f : s * __expf(mx - gm);
    s = warp_sum(s);
    if (ln == 0) red[wi] = s;
    __syncthreads();
    if (wi == 0) {
      const float t = warp_sum(ln < kCeThreads / 32 ? red[ln] : 0.f);
      if (ln == 0) s_lse = gm + logf(t);
    }
    __syncthreads();
    const float lse = s_lse;
    const int p0 = pair_off[r], p1 = pair_off[r + 1];
    float wsum = 0.f;
    for (int p = p0; p < p1; ++p) wsum += static_cast<float>(w[p]);
    OutT* dr = dl + static_cast<long>(r) * V;
    constexpr int U = 4;
    constexpr long kStep = 4L * kCeThreads;
    for (long c0 = threadIdx.x * 4; c0 < V; c0 += U * kStep) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long c = c0 + u * kStep;
        v[u] = c < V ? __ldcs(reinterpret_cast<const float4*>(lr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long c = c0 + u * kStep;
        if (c >= V) break;
        st_grad4(dr + c, wsum * __expf(v[u].x - lse), wsum * __expf(v[u].y - lse), wsum * __expf(v[u].z - lse),
                 wsum * __expf(v[u].w - lse));
      }
    }
    // target columns: - sum_j w_j onehot(t_j), rewritten after the streaming pass (one thread per
    // distinct target; the block barrier orders it after the pass's store of that column)
    __syncthreads();
    for (int p = p0 + static_cast<int>(threadIdx.x); p < p1; p += kCeThreads) {
      const long t = tgt[p];
      bool first = true;
      float wt = 0.f;
      for (int q = p0; q < p1; ++q)
        if (tgt[q] == t) {
          first = first && q >= p;
          wt += static_cast<float>(w[q]);
        }
      if (first) st_grad1(dr + t, wsum * __expf(lr[t] - lse) - wt);
    }
    if (threadIdx.x == 0) {
      double acc = 0.0;
      for (int p = p0; p < p1; ++p) acc += w[p] * (static_cast<double>(lse) - static_cast<double>(lr[tgt[p]]));
      atomicAdd(loss, acc);
    }
    __syncthreads();  // red / s_lse reuse by the next row
  }
}

// weighted_nll over bf16 logits stored relative to their 32-column group max (the LM-head GEMM's
// EPI_STORE_BF16_STATS epilogue): l = y + m_g. The row's lse comes from the per-group (m_g, s_g)
// statistics alone; the streaming pass reads 2 B per logit (8 per 16-byte load, all in one group)
// and writes the bf16 dlogits. Same multi-target semantics as ce_kernel.
__global__ void __launch_bounds__(kCeThreads, 4)
    ce_bf16_kernel(const __nv_bfloat16* __restrict__ y, int m, long V, const int32_t* __restrict__ pair_off,
                   const int32_t* __restrict__ tgt, const double* __restrict__ w, __nv_bfloat16* __restrict__ dl,
                   double* __restrict__ loss, const float2* __restrict__ stats, int n_groups) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  __shared__ float red[32];
  __shared__ float s_lse;
  constexpr float kL2e = 1.4426950408889634f;
  const int wi = threadIdx.x >> 5, ln = threadIdx.x & 31;
  for (int r = blockIdx.x; r < m; r += gridDim.x) {
    const __nv_bfloat16* yr = y + static_cast<long>(r) * V;
    const float2* sr = stats + static_cast<long>(r) * n_groups;
    float mx = -INFINITY, s = 0.f;
    for (int g = threadIdx.x; g < n_groups; g += kCeThreads) {
      const float2 ms = sr[g];
      if (ms.x > mx) {
        s = s * __expf(mx - ms.x) + ms.y;
        mx = ms.x;
      } else {
        s += ms.y * __expf(ms.x - mx);
      }
    }
    float gm = warp_max(mx);
    if (ln == 0) red[wi] = gm;
    __syncthreads();
    gm = warp_max(ln < kCeThreads / 32 ? red[ln] : -INFINITY);
    __syncthreads();
    s = (mx == -INFINITY) ? 0.f : s * __expf(mx - gm);
    s = warp_sum(s);
    if (ln == 0) red[wi] = s;
    __syncthreads();
    if (wi == 0) {
      const float t = warp_sum(ln < kCeThreads / 32 ? red[ln] : 0.f);
      if (ln == 0) s_lse = gm + logf(t);
    }
    __syncthreads();
    const float lse = s_lse;
    const int p0 = pair_off[r], p1 = pair_off[r + 1];
    float wsum = 0.f;
    for (int p = p0; p < p1; ++p) wsum += static_cast<float>(w[p]);
    __nv_bfloat16* dr = dl + static_cast<long>(r) * V;
    constexpr int U = 4;
    constexpr long kStep = 8L * kCeThreads;
    for (long c0 = threadIdx.x * 8; c0 < V; c0 += U * kStep) {
      uint4 v[U];
      float off[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long c = c0 + u * kStep;
        v[u] = c < V ? __ldcs(reinterpret_cast<const uint4*>(yr + c)) : make_uint4(0, 0, 0, 0);
        off[u] = c < V ? (sr[c >> 5].x - lse) * kL2e : 0.f;  // p = 2^((y + m_g - lse) log2e)
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long c = c0 + u * kStep;
        if (c >= V) break;
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
        uint32_t o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          o[i] = pack_bf16x2(wsum * ex2_approx(fmaf(f.x, kL2e, off[u])), wsum * ex2_approx(fmaf(f.y, kL2e, off[u])));
        }
        __stcs(reinterpret_cast<uint4*>(dr + c), make_uint4(o[0], o[1], o[2], o[3]));
      }
    }
    // target columns, after the streaming pass (the barrier orders it after that pass's store)
    __syncthreads();
    for (int p = p0 + static_cast<int>(threadIdx.x); p < p1; p += kCeThreads) {
      const long t = tgt[p];
      bool first = true;
      float wt = 0.f;
      for (int q = p0; q < p1; ++q)
        if (tgt[q] == t) {
          first = first && q >= p;
          wt += static_cast<float>(w[q]);
        }
      if (first) st_grad1(dr + t, wsum * __expf(__bfloat162float(yr[t]) + sr[t >> 5].x - lse) - wt);
    }
    if (threadIdx.x == 0) {
      double acc = 0.0;
      for (int p = p0; p < p1; ++p) {
        const long t = tgt[p];
        const double lt = static_cast<double>(__bfloat162float(yr[t])) + static_cast<double>(sr[t >> 5].x);
        acc += w[p] * (static_cast<double>(lse) - lt);
      }
      atomicAdd(loss, acc);
    }
    __syncthreads();
  }
}

__global__ void gather_rows_bf16_kernel(const __nv_bfloat16* __restrict__ src, const int32_t* __restrict__ idx,
                                        __nv_bfloat16* __restrict__ dst, int d) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  const int i = blockIdx.x;
  const uint4* s = reinterpret_cast<const uint4*>(src + static_cast<long>(idx[i]) * d);
  uint4* o = reinterpret_cast<uint4*>(dst + static_cast<long>(i) * d);
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) o[c] = s[c];
}

__global__ void scatter_rows_f32_kernel(const float* __restrict__ src, const int32_t* __restrict__ idx,
                                        float* __restrict__ dst, int d) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  const int i = blockIdx.x;
  const float4* s = reinterpret_cast<const float4*>(src + static_cast<long>(i) * d);
  float4* o = reinterpret_cast<float4*>(dst + static_cast<long>(idx[i]) * d);
  for (int c = threadIdx.x; c < d / 4; c += blockDim.x) o[c] = s[c];
}

// Stack pop of one layer: dqkv[r] = [dQ[r] | dK[r] | dV[r]] (bf16), then zero the consumed
// dK/dV stack rows (KVGrad::add_rows consumer + frame release, model.hpp:193-206).
// Grid-stride over 8-column chunks (two 16-byte loads per fp32 stream, one 16-byte bf16 store): at
// d = 896 a block-per-row layout left a quarter of the threads idle and paid one CTA per 3.5 KB row.
// DQ: pack dQ (leaf batches: dK / dV were written into the operand by the attention backward);
// KV: pack and consume dK / dV.
__device__ __forceinline__ void zero8(float* p) {
  reinterpret_cast<float4*>(p)[0] = make_float4(0.f, 0.f, 0.f, 0.f);
  reinterpret_cast<float4*>(p)[1] = make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ uint4 ld8_bf16(const float* p) {
  const float4 a = __ldcs(reinterpret_cast<const float4*>(p)), b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
  return make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w));
}
template <bool DQ, bool KV>
__global__ void __launch_bounds__(256) pack_dqkv_kernel(const float* __restrict__ dq, float* __restrict__ dk,
                                                        float* __restrict__ dv, __nv_bfloat16* __restrict__ out,
                                                        long n, int d) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  const int cpr = d / 8;
  const long total = n * cpr;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long r = i / cpr;
    const int c = static_cast<int>(i - r * cpr) * 8;
    const long o = r * d + c;
    __nv_bfloat16* orow = out + r * 3 * d + c;
    if (DQ) *reinterpret_cast<uint4*>(orow) = ld8_bf16(dq + o);
    if (KV) {
      *reinterpret_cast<uint4*>(orow + d) = ld8_bf16(dk + o);
      *reinterpret_cast<uint4*>(orow + 2 * d) = ld8_bf16(dv + o);
      zero8(dk + o);
      zero8(dv + o);
    }
  }
}

// dE[tok[r]] += gx[r]   (model.hpp:627-630)
__global__ void embed_grad_kernel(const float* __restrict__ gx, const int32_t* __restrict__ tok,
                                  float* __restrict__ gemb, int d) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  const int r = blockIdx.x;
  const float* s = gx + static_cast<long>(r) * d;
  float* o = gemb + static_cast<long>(tok[r]) * d;
  for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(s + c);
    red_add_v4_f32(o + c, v.x, v.y, v.z, v.w);
  }
}

// dst[c * ldd + r] = bf16(src[r * lds + c]) (parameter upload into a transposed device layout)
__global__ void f32_to_bf16_2d_t_kernel(const float* __restrict__ src, long lds, __nv_bfloat16* __restrict__ dst,
                                        long ldd, int rows, int cols) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  const long total = static_cast<long>(rows) * cols;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long c = i / rows, r = i % rows;
    dst[c * ldd + r] = __float2bfloat16_rn(src[r * lds + c]);
  }
}

__global__ void f32_to_bf16_2d_kernel(const float* __restrict__ src, long lds, __nv_bfloat16* __restrict__ dst,
                                      long ldd, int rows, int cols) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  const long total = static_cast<long>(rows) * cols;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long r = i / cols, c = i % cols;
    dst[r * ldd + c] = __float2bfloat16_rn(src[r * lds + c]);
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// N(0, std) via Box-Muller on a counter hash (seed, element index).
__global__ void init_normal_kernel(float* __restrict__ out, long n, uint64_t seed, float stdv) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const uint64_t h = mix64(seed * 0x9E3779B97F4A7C15ULL + static_cast<uint64_t>(i));
    const float u1 = (static_cast<float>(h >> 40) + 1.0f) * (1.0f / 16777217.0f);
    const float u2 = static_cast<float>((h >> 16) & 0xFFFFFF) * (1.0f / 16777216.0f);
    out[i] = stdv * sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
  }
}

__global__ void fill_kernel(float* __restrict__ out, long n, float v) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    out[i] = v;
}

}  // namespace

void k_embed_pe(const int32_t* tok, const int32_t* pos, const __nv_bfloat16* emb, const float* pe, float* x, int n,
                int d, cudaStream_t s) {
  if (n > 0) launch_k(embed_pe_kernel, dim3(n), dim3(128), 0, s, tok, pos, emb, pe, x, d);
}
void k_rmsnorm_fwd(const float* x, const float* gain, float* inv, __nv_bfloat16* y, int n, int d, cudaStream_t s) {
  if (n <= 0) return;
  const int vpt = (d + 127) / 128;
  const int blocks = (n + 7) / 8;
  if (vpt <= 2) launch_k(rmsnorm_fwd_kernel<2>, dim3(blocks), dim3(256), 0, s, x, gain, inv, y, n, d);
  else if (vpt <= 4) launch_k(rmsnorm_fwd_kernel<4>, dim3(blocks), dim3(256), 0, s, x, gain, inv, y, n, d);
  else if (vpt <= 8) launch_k(rmsnorm_fwd_kernel<8>, dim3(blocks), dim3(256), 0, s, x, gain, inv, y, n, d);
  else if (vpt <= 16) launch_k(rmsnorm_fwd_kernel<16>, dim3(blocks), dim3(256), 0, s, x, gain, inv, y, n, d);
  else if (vpt <= 32) launch_k(rmsnorm_fwd_kernel<16, 2>, dim3((n + 3) / 4), dim3(256), 0, s, x, gain, inv, y, n, d);
  else if (vpt <= 64) launch_k(rmsnorm_fwd_kernel<16, 4>, dim3((n + 1) / 2), dim3(256), 0, s, x, gain, inv, y, n, d);
  else throw std::invalid_argument("rmsnorm: d_model > 8192");
}
void k_rmsnorm_bwd(const float* gy, const float* x, const float* inv, const float* gain, const float* gres, float* gx,
                   __nv_bfloat16* gxb, float* ggain, int n, int d, cudaStream_t s) {
  if (n <= 0) return;
  const int vpt = (d + 127) / 128;  // float4 column groups per lane with one warp per row
  // (two warps per row at d = 896 measured 3.6 vs 4.2 TB/s: one warp per row up to 7 float4 per lane)
  // d <= 4096 with 16-byte rows: the TMA-fed persistent kernel; wider rows: several warps per row
  if (d % 4 == 0 && vpt <= 2) launch_rmsnorm_bwd_tma<2, false>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (d % 4 == 0 && vpt <= 4) launch_rmsnorm_bwd_tma<4, false>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (d % 4 == 0 && vpt <= 8) launch_rmsnorm_bwd_tma<8, false>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (d % 4 == 0 && vpt <= 16) launch_rmsnorm_bwd_tma<16, false>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (d % 4 == 0 && vpt <= 32) launch_rmsnorm_bwd_tma<32, true>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (vpt <= 2) launch_rmsnorm_bwd<2, 1>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (vpt <= 4) launch_rmsnorm_bwd<4, 1>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (vpt <= 7) launch_rmsnorm_bwd<7, 1>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (vpt <= 14) launch_rmsnorm_bwd<7, 2>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (vpt <= 28) launch_rmsnorm_bwd<7, 4>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (vpt <= 64) launch_rmsnorm_bwd<8, 8>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else throw std::invalid_argument("rmsnorm backward: d_model > 8192");
}
bool rmsnorm_bwd_bf16_gy_ok(int d) { return d % 8 == 0 && d <= 4096; }
void k_rmsnorm_bwd(const __nv_bfloat16* gy, const float* x, const float* inv, const float* gain, const float* gres,
                   float* gx, __nv_bfloat16* gxb, float* ggain, int n, int d, cudaStream_t s) {
  if (!rmsnorm_bwd_bf16_gy_ok(d)) throw std::invalid_argument("rmsnorm backward (bf16 gy): d_model must be a multiple of 8, <= 4096");
  if (n <= 0) return;
  const int vpt = (d + 127) / 128;
  if (vpt <= 2) launch_rmsnorm_bwd_tma<2, false>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (vpt <= 4) launch_rmsnorm_bwd_tma<4, false>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (vpt <= 8) launch_rmsnorm_bwd_tma<8, false>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else if (vpt <= 16) launch_rmsnorm_bwd_tma<16, false>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
  else launch_rmsnorm_bwd_tma<32, true>(gy, x, inv, gain, gres, gx, gxb, ggain, n, d, s);
}
void k_ce(const float* logits, int m, long V, const int32_t* pair_off, const int32_t* tgt, const double* w,
          __nv_bfloat16* dl, double* loss, cudaStream_t s, const float2* stats, int n_groups) {
  if (m > 0)
    launch_k(ce_kernel<__nv_bfloat16>, dim3(std::min(m, 148 * 4)), dim3(kCeThreads), 0, s, logits, m, V, pair_off, tgt, w, dl, loss, stats, n_groups);
}
void k_ce_bf16(const __nv_bfloat16* y, int m, long V, const int32_t* pair_off, const int32_t* tgt, const double* w,
               __nv_bfloat16* dl, double* loss, cudaStream_t s, const float2* stats, int n_groups) {
  if (V % 8 != 0) throw std::invalid_argument("k_ce_bf16: vocab_size must be a multiple of 8");
  if (m > 0)
    launch_k(ce_bf16_kernel, dim3(std::min(m, 148 * 4)), dim3(kCeThreads), 0, s, y, m, V, pair_off, tgt, w, dl, loss, stats, n_groups);
}
void k_ce_f32(const float* logits, int m, long V, const int32_t* pair_off, const int32_t* tgt, const double* w,
              float* dl, double* loss, cudaStream_t s) {
  if (m > 0)
    launch_k(ce_kernel<float>, dim3(std::min(m, 148 * 4)), dim3(kCeThreads), 0, s, logits, m, V, pair_off, tgt, w, dl, loss, nullptr, 0);
}
// dst[i] += src[i] (fp32, n % 4 == 0, 16-byte aligned)
__global__ void add_f32_kernel(float* __restrict__ dst, const float* __restrict__ src, long n4) {
  pdl_wait();  // launch.cuh: no global access before the predecessor completes
  pdl_trigger();
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    float4 a = reinterpret_cast<float4*>(dst)[i];
    const float4 b = reinterpret_cast<const float4*>(src)[i];
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
    reinterpret_cast<float4*>(dst)[i] = a;
  }
}
void k_add_f32(float* dst, const float* src, long n, cudaStream_t s) {
  if (n % 4 != 0) throw std::invalid_argument("k_add_f32: n must be a multiple of 4");
  if (n > 0)
    launch_k(add_f32_kernel, dim3(static_cast<int>(std::min<long>((n / 4 + 255) / 256, 148 * 16))), dim3(256), 0, s, dst, src, n / 4);
}
void k_gather_rows_bf16(const __nv_bfloat16* src, const int32_t* idx, __nv_bfloat16* dst, int m, int d,
                        cudaStream_t s) {
  if (m > 0) launch_k(gather_rows_bf16_kernel, dim3(m), dim3(128), 0, s, src, idx, dst, d);
}
void k_scatter_rows_f32(const float* src, const int32_t* idx, float* dst, int m, int d, cudaStream_t s) {
  if (m > 0) launch_k(scatter_rows_f32_kernel, dim3(m), dim3(128), 0, s, src, idx, dst, d);
}
static unsigned pack_grid(long n, int d) {
  const long chunks = n * (d / 8);
  return static_cast<unsigned>(std::min<long>((chunks + 255) / 256, static_cast<long>(device_sm_count()) * 8));
}
void k_pack_dqkv(const float* dq, float* dk, float* dv, __nv_bfloat16* out, int n, int d, cudaStream_t s) {
  if (d % 8 != 0) throw std::invalid_argument("pack_dqkv: d_model must be a multiple of 8");
  if (n <= 0) return;
  if (dk == nullptr)
    launch_k(pack_dqkv_kernel<true, false>, dim3(pack_grid(n, d)), dim3(256), 0, s, dq, dk, dv, out, static_cast<long>(n), d);
  else
    launch_k(pack_dqkv_kernel<true, true>, dim3(pack_grid(n, d)), dim3(256), 0, s, dq, dk, dv, out, static_cast<long>(n), d);
}
void k_pack_dkv(float* dk, float* dv, __nv_bfloat16* out, int n, int d, cudaStream_t s) {
  if (d % 8 != 0) throw std::invalid_argument("pack_dkv: d_model must be a multiple of 8");
  if (n > 0)
    launch_k(pack_dqkv_kernel<false, true>, dim3(pack_grid(n, d)), dim3(256), 0, s, nullptr, dk, dv, out,
             static_cast<long>(n), d);
}
void k_embed_grad(const float* gx, const int32_t* tok, float* gemb, int n, int d, cudaStream_t s) {
  if (n > 0) launch_k(embed_grad_kernel, dim3(n), dim3(128), 0, s, gx, tok, gemb, d);
}
void k_f32_to_bf16_2d_t(const float* src, long lds, __nv_bfloat16* dst, long ldd, int rows, int cols, cudaStream_t s) {
  const long total = static_cast<long>(rows) * cols;
  if (total > 0)
    launch_k(f32_to_bf16_2d_t_kernel, dim3(static_cast<int>(std::min<long>((total + 255) / 256, 148 * 32))), dim3(256), 0, s, src, lds, dst, ldd, rows, cols);
}
void k_f32_to_bf16_2d(const float* src, long lds, __nv_bfloat16* dst, long ldd, int rows, int cols, cudaStream_t s) {
  const long total = static_cast<long>(rows) * cols;
  if (total > 0) launch_k(f32_to_bf16_2d_kernel, dim3(static_cast<int>(std::min<long>((total + 255) / 256, 148 * 32))), dim3(256), 0, s, src, lds, dst, ldd, rows, cols);
}
void k_init_normal(float* out, long n, uint64_t seed, float stdv, cudaStream_t s) {
  if (n > 0) launch_k(init_normal_kernel, dim3(static_cast<int>(std::min<long>((n + 255) / 256, 148 * 32))), dim3(256), 0, s, out, n, seed, stdv);
}
void k_fill(float* out, long n, float v, cudaStream_t s) {
  if (n > 0) launch_k(fill_kernel, dim3(static_cast<int>(std::min<long>((n + 255) / 256, 148 * 32))), dim3(256), 0, s, out, n, v);
}

}  // namespace ttb
