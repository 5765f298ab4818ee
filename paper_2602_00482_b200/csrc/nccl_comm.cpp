// NCCL plumbing of the multi-GPU step: one communicator per GPU and ONE in-place
// sum all-reduce of the flat fp32 GradientStore per step — the replacement of the reference's
// worker-order gradient reduction.
//
// libnccl is bound at run time (dlopen of libnccl.so.2, reusing an already-loaded copy, e.g. the one
// PyTorch ships) instead of at link time: the process then holds exactly one NCCL, whichever loaded
// first, and the engine library has no hard dependency on it. The API used (ncclGetUniqueId,
// ncclCommInitRank, ncclCommInitAll, ncclAllReduce, ncclCommDestroy) is stable across NCCL 2.x.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "engine.hpp"

namespace ttb {

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      err = std::string("NCCL not available: ") + (e ? e : "dlopen(libnccl.so.2) failed");
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && err.empty()) err = std::string("NCCL symbol missing: ") + name;
      return p;
    };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(sym("ncclCommInitAll"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) throw std::runtime_error(err);
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* s = nccl().error_string ? nccl().error_string(r) : "?";
    throw std::runtime_error(std::string(what) + ": " + s);
  }
}

}  // namespace

void Engine::grads_allreduce(void* comm) {
  if (!comm) throw std::invalid_argument("grads_allreduce: null communicator");
  nck(nccl().all_reduce(grads_.p, grads_.p, n_params_, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm), stream_),
      "ncclAllReduce");
  check_cuda(cudaStreamSynchronize(stream_), "grads_allreduce");
}

}  // namespace ttb

extern "C" {

int tt_nccl_unique_id(uint8_t* id_out) {
  return ttb::guarded([&] {
    if (!id_out) throw std::invalid_argument("null id_out");
    ncclUniqueId id;
    ttb::nck(ttb::nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

int tt_nccl_comm_init_rank(const uint8_t* id, int32_t nranks, int32_t rank, int32_t device, void** comm_out) {
  return ttb::guarded([&] {
    if (!id || !comm_out) throw std::invalid_argument("null id / comm_out");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("tt_nccl_comm_init_rank: bad rank");
    ttb::check_cuda(cudaSetDevice(device), "cudaSetDevice");
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t c = nullptr;
    ttb::nck(ttb::nccl().comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
    *comm_out = c;
  });
}

int tt_nccl_comm_init_all(int32_t ndev, const int32_t* devices, void** comms_out) {
  return ttb::guarded([&] {
    if (ndev < 1 || !comms_out) throw std::invalid_argument("tt_nccl_comm_init_all: bad arguments");
    std::vector<ncclComm_t> c(ndev);
    ttb::nck(ttb::nccl().comm_init_all(c.data(), ndev, devices), "ncclCommInitAll");
    for (int i = 0; i < ndev; ++i) comms_out[i] = c[i];
  });
}

int tt_nccl_comm_destroy(void* comm) {
  return ttb::guarded([&] {
    if (comm) ttb::nck(ttb::nccl().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  });
}

}  // extern "C"
