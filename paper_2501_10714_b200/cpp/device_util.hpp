// device_util.hpp — small RAII helpers for the C++ drop-in's host-Matrix
// entry points: scoped device allocations on a private stream, and mapping
// of C-ABI status codes to the reference's exception types.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "fsmoe/common.hpp"
#include "fsmoe_cuda.h"

namespace fsmoe {

inline void throw_on(int rc) {
  if (rc == FSMOE_OK) return;
  std::string msg = fsmoe_last_error();
  if (rc == FSMOE_CONFIG_ERROR) throw ConfigError(msg);
  if (rc == FSMOE_INVARIANT_ERROR) throw InvariantError(msg);
  throw DeviceError(msg.empty() ? "device error" : msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

class DeviceScope {
 public:
  DeviceScope() { cuda_check(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "stream"); }
  ~DeviceScope() {
    cudaStreamSynchronize(s_);
    for (void* p : ptrs_) cudaFree(p);
    cudaStreamDestroy(s_);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;

  template <class T>
  T* alloc(long long n) {
    void* p = nullptr;
    size_t bytes = static_cast<size_t>(n > 0 ? n : 1) * sizeof(T);
    cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    ptrs_.push_back(p);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const std::vector<T>& h) {
    T* d = alloc<T>(static_cast<long long>(h.size()));
    if (!h.empty())
      cuda_check(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s_),
                 "upload");
    return d;
  }
  template <class T>
  void download(T* h, const T* d, long long n) {
    if (n <= 0) return;
    cuda_check(cudaMemcpyAsync(h, d, static_cast<size_t>(n) * sizeof(T), cudaMemcpyDeviceToHost, s_),
               "download");
    cuda_check(cudaStreamSynchronize(s_), "sync");
  }
  template <class T>
  void zero(T* d, long long n) {
    cuda_check(cudaMemsetAsync(d, 0, static_cast<size_t>(n) * sizeof(T), s_), "memset");
  }
  void* stream() const { return s_; }

 private:
  cudaStream_t s_ = nullptr;
  std::vector<void*> ptrs_;
};

}  // namespace fsmoe
