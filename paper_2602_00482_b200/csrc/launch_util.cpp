// Per-device launch helpers declared in kernels/gemm.h.
#include <cuda_runtime.h>

#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>

#include "kernels/gemm.h"

namespace ttb {

namespace {
std::mutex g_mu;
std::set<std::pair<const void*, int>> g_attr_done;
int g_sms[64] = {0};
}  // namespace

void ensure_smem_attr(const void* fn, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_attr_done.insert({fn, dev}).second) return;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    g_attr_done.erase({fn, dev});
    (void)cudaGetLastError();
    throw std::runtime_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  }
}

int device_sm_count() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int n = __atomic_load_n(&g_sms[dev], __ATOMIC_RELAXED);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    __atomic_store_n(&g_sms[dev], n, __ATOMIC_RELAXED);
  }
  return n;
}

int g_pdl = 1;
void set_pdl(int on) { g_pdl = on ? 1 : 0; }

void check_launch(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace ttb
