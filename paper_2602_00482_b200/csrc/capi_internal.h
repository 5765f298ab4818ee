// Error plumbing shared by the C-ABI translation units: every extern "C" entry returns a
// status code; exceptions never cross the ABI (SURVEY §8(b) C-ABI conventions).
#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../include/treetrain_b200.h"

namespace ttb {

void set_last_error(const std::string& msg);

// Non-finite loss: the SPEC's abort-on-divergence.
struct NonFiniteError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return TT_OK;
  } catch (const NonFiniteError& e) {
    set_last_error(e.what());
    return TT_ERR_NONFINITE;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return TT_ERR_INVALID_ARGUMENT;
  } catch (const std::bad_alloc& e) {
    set_last_error(std::string("out of memory: ") + e.what());
    return TT_ERR_OOM;
  } catch (const std::runtime_error& e) {
    set_last_error(e.what());
    return TT_ERR_RUNTIME;
  } catch (...) {
    set_last_error("unknown error");
    return TT_ERR_RUNTIME;
  }
}

}  // namespace ttb
