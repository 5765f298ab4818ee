// TMEM load throughput probe (sm_100a): W warps per CTA (one CTA per SM) each repeatedly issue P
// tcgen05.ld.32x32b.x{16,32,64} from their lane quadrant and then one tcgen05.wait::ld; reports
// bytes read per SM clock (profiles/r2/tmem_probe.log).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_probe tools/tmem_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int X>
__device__ __forceinline__ void ldx(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ldx<16>(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(a));
}
template <>
__device__ __forceinline__ void ldx<32>(uint32_t a, uint32_t* r) {
  ldx<16>(a, r);
  ldx<16>(a + 16, r + 16);
}

template <int X, int P>
__global__ void probe(int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        static_cast<uint32_t>(__cvta_generic_to_shared(&slot))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp / 4) * 16;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[P][X];
#pragma unroll
    for (int j = 0; j < P; ++j) ldx<X>(tmem + ((j * X) & 255), r[j]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < P; ++j) acc ^= r[j][0] ^ r[j][X - 1];
  }
  __syncthreads();
  const long long t1 = clock64();
  if (acc == 0x12345678) sink[0] = acc;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int X, int P>
void run(int warps, unsigned long long* d, uint32_t* sink) {
  const int iters = 4000;
  probe<X, P><<<148, warps * 32>>>(iters, d, sink);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return; }
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double bytes = double(iters) * P * warps * 32 * X * 4;
  printf("warps %2d  %d x ld.x%-2d per wait: %6.1f B/clk/SM  (%.0f clk per wait round)\n", warps, P, X,
         bytes / double(h[0]), double(h[0]) / iters);
}

int main() {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4);
  for (int w : {4, 8, 16}) {
    run<16, 1>(w, d, sink);
    run<16, 2>(w, d, sink);
    run<16, 4>(w, d, sink);
    run<32, 2>(w, d, sink);
    run<32, 4>(w, d, sink);
    run<16, 8>(w, d, sink);
  }
  return 0;
}
