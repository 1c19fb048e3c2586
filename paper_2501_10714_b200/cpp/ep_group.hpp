// ep_group.hpp — the expert-parallel communicator: one NCCL communicator over
// the ranks of one box (NVLink 5 / NVSwitch), created from a unique id that
// the host side distributes (torch.distributed is only used for that
// bootstrap broadcast). All MoE exchanges of a layer run on one comm stream
// so NCCL's issue order is the FSMoE schedule's inter-link order
// (schedule_sim.cpp:182-216).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <string>
#include <vector>

#include "fsmoe/common.hpp"

namespace fsmoe {

inline void throw_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw DeviceError(std::string(what) + ": " + ncclGetErrorString(r));
}

class EpGroup {
 public:
  EpGroup(int world, int rank, const ncclUniqueId& id, int device, int max_ctas)
      : world_(world), rank_(rank), device_(device) {
    cudaSetDevice(device);
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (max_ctas > 0) cfg.maxCTAs = max_ctas;
    nccl_check(ncclCommInitRankConfig(&comm_, world, id, rank, &cfg), "ncclCommInitRankConfig");
  }
  ~EpGroup() {
    if (comm_) ncclCommDestroy(comm_);
  }
  EpGroup(const EpGroup&) = delete;
  EpGroup& operator=(const EpGroup&) = delete;

  // Collective: every rank passes its own device allocation; returns every
  // rank's pointer to it mapped into this process (CUDA IPC over NVLink /
  // NVSwitch; [rank] is `local`). The NCCL allgather of the 64-byte handles
  // is also the barrier that orders each rank's initialisation of `local`
  // (stream `s`) before any peer can touch it.
  std::vector<void*> map_peers(void* local, cudaStream_t s) {
    cudaIpcMemHandle_t h;
    throw_cuda(cudaIpcGetMemHandle(&h, local), "cudaIpcGetMemHandle");
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    void* dbuf = nullptr;
    throw_cuda(cudaMalloc(&dbuf, hb * world_), "cudaMalloc");
    throw_cuda(cudaMemcpyAsync(static_cast<char*>(dbuf) + hb * rank_, &h, hb, cudaMemcpyHostToDevice, s),
               "cudaMemcpyAsync");
    nccl_check(ncclAllGather(static_cast<char*>(dbuf) + hb * rank_, dbuf, hb, ncclUint8, comm_, s),
               "ncclAllGather");
    std::vector<cudaIpcMemHandle_t> all(world_);
    throw_cuda(cudaMemcpyAsync(all.data(), dbuf, hb * world_, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
    throw_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    cudaFree(dbuf);
    std::vector<void*> out(world_, nullptr);
    for (int p = 0; p < world_; ++p) {
      if (p == rank_) {
        out[p] = local;
        continue;
      }
      throw_cuda(cudaIpcOpenMemHandle(&out[p], all[p], cudaIpcMemLazyEnablePeerAccess),
                 "cudaIpcOpenMemHandle");
    }
    return out;
  }
  void unmap_peers(const std::vector<void*>& ptrs) {
    for (int p = 0; p < static_cast<int>(ptrs.size()); ++p)
      if (p != rank_ && ptrs[p]) cudaIpcCloseMemHandle(ptrs[p]);
  }

  ncclComm_t comm() const { return comm_; }
  int world() const { return world_; }
  int rank() const { return rank_; }
  int device() const { return device_; }

 private:
  ncclComm_t comm_ = nullptr;
  int world_ = 1, rank_ = 0, device_ = 0;
};

}  // namespace fsmoe
