// Kernel launches with programmatic dependent launch (PDL, sm_90+).
//
// A step is ~40K back-to-back kernels on one stream (c2: 24 layers x 80 segment batches x ~20). With
// plain stream order each kernel's launch, CTA rasterisation and prologue (mbarrier init, TMEM
// allocation, tensor-map prefetch) start only after the previous kernel has drained. Launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, a kernel may start as soon as every CTA of its
// predecessor has executed griddepcontrol.launch_dependents; it runs its prologue and then blocks in
// griddepcontrol.wait until the predecessor grid has COMPLETED and its memory is visible. Contract
// for every kernel launched here (pdl_wait / pdl_trigger in sm100.cuh):
//   * no global-memory access (read or write) before pdl_wait();
//   * pdl_trigger() only after the CTA holds its TMEM allocation: a dependent CTA that allocated TMEM
//     on the same SM and then blocked in its wait would otherwise starve a predecessor CTA's alloc.
// Completion is transitive (a kernel completes only after its own wait returned), so the only grid
// that can still be running when a kernel passes its prologue is its immediate predecessor.
#pragma once
#include <cuda_runtime.h>

#include <utility>

#include "gemm.h"

namespace ttb {

// Fills attr[n] with the PDL attribute when enabled; returns the new attribute count.
inline unsigned pdl_attr(cudaLaunchAttribute* attr, unsigned n) {
  if (!g_pdl) return n;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n].val.programmaticStreamSerializationAllowed = 1;
  return n + 1;
}

template <typename... KArgs, typename... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = pdl_attr(attr, 0);
  check_launch(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "kernel launch");
}

}  // namespace ttb
