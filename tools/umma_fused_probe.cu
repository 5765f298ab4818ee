// Tensor-pipe floor of the fused dh=64 attention-backward block (attention_bwd_sm100.cu): one thread
// issues, per 128-key x 128-query block, S^T (4 x M128 N128 K16, SS K-major), dP^T (same), dV (8 x
// N64, TS, B MN-major), dQ (8 x N64, SS, A and B MN-major), dK (8 x N64, SS, A K-major, B MN-major)
// with the kernel's 5 commits; variants isolate each group. Random bf16 operands. One CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_00482_b200/csrc/kernels \
//        tools/umma_fused_probe.cu -o /tmp/umma_fused_probe && /tmp/umma_fused_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace ttb;

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t bar, cb[8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&cb[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  for (int i = threadIdx.x; i < 180224 / 4; i += blockDim.x) {
    uint32_t h = (i + 1) * 2654435761u;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    const uint32_t lo = 0x3c00u ^ (h & 0x807fu), hi = 0x3c00u ^ ((h >> 16) & 0x807fu);
    reinterpret_cast<uint32_t*>(smem)[i] = lo | (hi << 16);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // smem: K 0 (16 KB), V 16 KB, Q ring 32 KB + 3 x 16, dO ring 80 KB + 3 x 16, dS 2 x 32 KB at 128 KB
  constexpr int kOffV = 16384, kOffQ = 32768, kOffDO = 81920, kOffDS = 131072;
  if (threadIdx.x == 0) {
    constexpr uint32_t idS = make_idesc_bf16(128, 128, false, false);
    constexpr uint32_t idKV = make_idesc_bf16(128, 64, false, true);
    constexpr uint32_t idQ = make_idesc_bf16(128, 64, true, true);
    const uint64_t d16 = make_sdesc_sw128(smem_u32(smem), 16, 1024);
    const uint64_t dmn = make_sdesc_sw128(smem_u32(smem), 128 * 128, 1024);
    const uint64_t dsk = make_sdesc_sw128(smem_u32(smem + kOffDS), 16, 1024);
    const uint64_t dsm = make_sdesc_sw128(smem_u32(smem + kOffDS), 128 * 128, 1024);
    const uint32_t t_S = tmem, t_dP = tmem + 256, t_dK = tmem + 384, t_dV = tmem + 448;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int st = i % 3;
      const uint32_t q_off = kOffQ + st * 16384, do_off = kOffDO + st * 16384, ds_off = (i & 1) * 32768;
      if (MODE == 0 || MODE == 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16_ss(t_S + (i & 1) * 128, sdesc_add(d16, k * 32), sdesc_add(d16, q_off + k * 32), idS, k > 0);
        umma_commit(&cb[i & 1]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16_ss(t_dP, sdesc_add(d16, kOffV + k * 32), sdesc_add(d16, do_off + k * 32), idS, k > 0);
        umma_commit(&cb[2]);
      }
      if (MODE == 0 || MODE == 2 || MODE == 3) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma_bf16_ts(t_dV, t_S + (i & 1) * 128 + 8 * k, sdesc_add(dmn, do_off + k * 2048), idKV, 1);
      }
      if (MODE == 0 || MODE == 2 || MODE == 4) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma_bf16_ss(t_S + (i & 1) * 128 + 64, sdesc_add(dsm, ds_off + k * 2048), sdesc_add(dmn, k * 2048), idQ, k > 0);
        if (MODE == 0) umma_commit(&cb[3 + (i & 1)]);
      }
      if (MODE == 0 || MODE == 2 || MODE == 5) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma_bf16_ss(t_dK, sdesc_add(dsk, ds_off + (k / 4) * 16384 + (k % 4) * 32), sdesc_add(dmn, q_off + k * 2048),
                       idKV, 1);
      }
      if (MODE == 0) {
        umma_commit(&cb[5]);
        umma_commit(&cb[6 + (i & 1)]);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int MODE>
void run(long long* d, int iters, const char* name, int mmas) {
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  probe<MODE><<<148, 128, 200000>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[1];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-44s %7.1f clk/block  %6.1f clk/MMA  %s\n", name, double(h[0]) / iters, double(h[0]) / (iters * mmas),
         cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<0>(d, 2000, "fused block (S, dP, dV, dQ, dK + 5 commits)", 32);
  run<1>(d, 2000, "S + dP only (N=128 SS)", 8);
  run<2>(d, 2000, "dV + dQ + dK (N=64)", 24);
  run<3>(d, 2000, "dV only (TS, B MN-major)", 8);
  run<4>(d, 2000, "dQ only (SS, A+B MN-major)", 8);
  run<5>(d, 2000, "dK only (SS, A K-major, B MN-major)", 8);
  return 0;
}
