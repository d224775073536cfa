// Helpers shared by the runtime's translation units (runtime.cpp,
// runtime_mmdit.cpp). Internal: not part of the C ABI.
#pragma once

#include <sstream>

#include "runtime.h"

namespace pf {

#define PF_CUDA_CHECK(expr)                                                  \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) {                                                 \
      std::ostringstream _os;                                                \
      _os << "CUDA error " << cudaGetErrorString(_e) << " at " << __FILE__   \
          << ":" << __LINE__ << " (" #expr ")";                              \
      throw CudaError(_os.str());                                            \
    }                                                                        \
  } while (0)

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

// The stage's split-K workspace attached to a GEMM's epilogue parameters
// (skinny residual split-K itself is opt-in, kernels.cu).
inline EpiParams sk(const Stage& s, EpiParams ep) {
  ep.splitk_ws = s.splitk_ws;
  ep.splitk_ws_floats = s.splitk_ws_floats;
  ep.splitk_counters = s.splitk_counters;
  ep.splitk_counter_cap = s.splitk_counter_cap;
  return ep;
}

inline void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::ostringstream os;
    os << "CUDA error " << cudaGetErrorString(e) << " launching " << what;
    throw CudaError(os.str());
  }
}

}  // namespace pf
