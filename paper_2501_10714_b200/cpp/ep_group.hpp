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

#include "fsmoe/common.hpp"

namespace fsmoe {

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

  ncclComm_t comm() const { return comm_; }
  int world() const { return world_; }
  int rank() const { return rank_; }
  int device() const { return device_; }

 private:
  ncclComm_t comm_ = nullptr;
  int world_ = 1, rank_ = 0, device_ = 0;
};

}  // namespace fsmoe
