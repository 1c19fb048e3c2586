// capi_common.h — error plumbing shared by the extern "C" entry points.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/fsmoe_cuda.h"

namespace fsmoe {

void set_last_error(const std::string& msg);
int config_error(const std::string& msg);     // returns FSMOE_CONFIG_ERROR
int invariant_error(const std::string& msg);  // returns FSMOE_INVARIANT_ERROR
int cuda_status(cudaError_t e, const char* where);  // 0 or FSMOE_CUDA_ERROR

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Process-wide count of kernels this library has launched (fsmoe_launch_count).
void count_launch();

}  // namespace fsmoe

#define FSMOE_CUDA_TRY(expr, where)                         \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return ::fsmoe::cuda_status(_e, where); \
  } while (0)
