// host_once.h — per-device one-time host setup (kernel attributes).
#pragma once
#include <cuda_runtime.h>

#include <atomic>

namespace fsmoe {

// True the first time it is called for the current device with this flag:
// cudaFuncSetAttribute is per device, so a process driving several GPUs must
// set it on each.
inline bool first_on_device(std::atomic<unsigned>& seen) {
  int d = 0;
  cudaGetDevice(&d);
  const unsigned bit = 1u << (d & 31);
  return (seen.fetch_or(bit) & bit) == 0;
}

}  // namespace fsmoe
