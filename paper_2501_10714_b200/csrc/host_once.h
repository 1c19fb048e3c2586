// host_once.h — per-device one-time host setup (kernel attributes) and cached
// device properties, safe for a process that drives several GPUs from
// several threads.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <utility>

namespace fsmoe {

constexpr int kMaxDevices = 32;

inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d & (kMaxDevices - 1);
}

// One std::once_flag per device: cudaFuncSetAttribute is per device, and a
// second thread on the same device must not launch before the first one's
// attribute call has returned (call_once blocks it until then).
struct DeviceOnce {
  std::once_flag flag[kMaxDevices];
};

template <class F>
void once_on_device(DeviceOnce& o, F&& fn) {
  std::call_once(o.flag[current_device()], fn);
}

// SM count of the current device (cached per device).
inline int device_sms() {
  static std::atomic<int> sms[kMaxDevices];
  const int d = current_device();
  int v = sms[d].load(std::memory_order_relaxed);
  if (v <= 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    sms[d].store(v, std::memory_order_relaxed);
  }
  return v;
}

// Threads per block for thread-per-token kernels: 128, or 32 when 128 would
// put the work on fewer than two blocks per SM (small token counts: spread
// the latency-bound per-token loops over every SM).
inline int per_token_block(long long T) {
  return (T + 127) / 128 >= 2LL * device_sms() ? 128 : 32;
}

// Programmatic dependent launch (PDL). Kernels that start with
// fsmoe_dev::pdl_enter() are launched through pdl_launch() with
// cudaLaunchAttributeProgrammaticStreamSerialization: the next kernel of the
// stream is scheduled while this one drains (its prologue overlaps our tail)
// and blocks in griddepcontrol.wait until this grid has completed and its
// memory is visible. FSMOE_PDL=0 turns the attribute off (read once).
inline bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("FSMOE_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... P, typename... A>
cudaError_t pdl_launch(void (*kern)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

}  // namespace fsmoe
