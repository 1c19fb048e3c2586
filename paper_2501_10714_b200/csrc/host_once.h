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

// Threads per block for thread-per-token kernels: 128, or 32 when 128 would
// put the work on fewer than two blocks per SM (small token counts: spread
// the latency-bound per-token loops over every SM).
inline int per_token_block(long long T) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return (T + 127) / 128 >= 2LL * sms ? 128 : 32;
}

}  // namespace fsmoe
