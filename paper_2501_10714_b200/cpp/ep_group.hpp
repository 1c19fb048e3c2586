// ep_group.hpp — the expert-parallel group of one MoE layer.
//
// Two kinds, same interface to the layer executor:
//
// * NCCL group (production): one NCCL communicator over the ranks of one box
//   (NVLink 5 / NVSwitch), one process per GPU, created from a unique id that
//   the host side distributes (torch.distributed is only used for that
//   bootstrap broadcast). Receive buffers are shared through CUDA IPC. All
//   MoE exchanges of a layer run on one comm stream so NCCL's issue order is
//   the FSMoE schedule's inter-link order (schedule_sim.cpp:182-216).
//
// * Local group (the single-GPU multi-rank harness): P logical ranks in one
//   process on ONE device, each driven by its own host thread. Peer "maps"
//   are the other ranks' plain device pointers, collectives are host
//   barriers plus a summation kernel, and there is no NCCL or IPC. It runs
//   the peer-memory transport's producer stores and arrival flags exactly as
//   on several GPUs, so a one-GPU box verifies them. The executor calls
//   host_sync() before enqueueing any wait on a peer flag: every signal that
//   wait needs is then already enqueued (all ranks issue their exchanges in
//   the same order), so work enqueued from different threads onto the one
//   device can never wait on something queued behind it.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "fsmoe/common.hpp"
#include "fsmoe_cuda.h"

namespace fsmoe {

inline void throw_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw DeviceError(std::string(what) + ": " + ncclGetErrorString(r));
}

// Shared state of a local group: a reusable host barrier, one pointer slot
// and two events per rank.
struct LocalHub {
  explicit LocalHub(int world)
      : world(world), ptr(world, nullptr), ev_ready(world, nullptr), ev_done(world, nullptr) {}

  // Returns false when `timeout` expires first (teardown only; the barrier
  // is then left in an undefined state and must not be reused).
  bool barrier(std::chrono::milliseconds timeout = std::chrono::milliseconds(0)) {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    if (timeout.count() > 0)
      return cv.wait_for(lk, timeout, [&] { return gen != g; });
    cv.wait(lk, [&] { return gen != g; });
    return true;
  }

  const int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  std::vector<void*> ptr;
  std::vector<cudaEvent_t> ev_ready, ev_done;
};

class EpGroup {
 public:
  EpGroup(int world, int rank, const ncclUniqueId& id, int device, int max_ctas)
      : world_(world), rank_(rank), device_(device) {
    cudaSetDevice(device);
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (max_ctas > 0) cfg.maxCTAs = max_ctas;
    nccl_check(ncclCommInitRankConfig(&comm_, world, id, rank, &cfg), "ncclCommInitRankConfig");
  }
  EpGroup(std::shared_ptr<LocalHub> hub, int rank, int device)
      : world_(hub->world), rank_(rank), device_(device), hub_(std::move(hub)) {
    throw_cuda(cudaSetDevice(device), "cudaSetDevice");
    throw_cuda(cudaEventCreateWithFlags(&hub_->ev_ready[rank], cudaEventDisableTiming), "event");
    throw_cuda(cudaEventCreateWithFlags(&hub_->ev_done[rank], cudaEventDisableTiming), "event");
  }
  ~EpGroup() {
    if (comm_) ncclCommDestroy(comm_);
    if (hub_) {
      cudaEventDestroy(hub_->ev_ready[rank_]);
      cudaEventDestroy(hub_->ev_done[rank_]);
    }
    if (scratch_) cudaFree(scratch_);
  }
  EpGroup(const EpGroup&) = delete;
  EpGroup& operator=(const EpGroup&) = delete;

  bool local() const { return hub_ != nullptr; }

  // Local group: every rank has enqueued everything before this call.
  void host_sync() {
    if (hub_) hub_->barrier();
  }

  // Collective: every rank passes its own device allocation; returns every
  // rank's pointer to it usable from this process ([rank] is `local`). NCCL
  // group: CUDA IPC handles allgathered over the communicator, which is also
  // the barrier that orders each rank's initialisation of `local` (stream
  // `s`) before any peer can touch it. Local group: the pointers themselves.
  std::vector<void*> map_peers(void* local, cudaStream_t s) {
    if (hub_) {
      throw_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
      hub_->ptr[rank_] = local;
      hub_->barrier();
      std::vector<void*> out(hub_->ptr);
      hub_->barrier();
      return out;
    }
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
    if (hub_) return;
    for (int p = 0; p < static_cast<int>(ptrs.size()); ++p)
      if (p != rank_ && ptrs[p]) cudaIpcCloseMemHandle(ptrs[p]);
  }

  // Teardown barrier (no exceptions): after it, no peer maps or signals into
  // this rank's exported memory any more, so it can be freed. NCCL: a
  // one-word allreduce on `s`, synchronised; local: the host barrier (with a
  // timeout, so a rank torn down alone does not hang the process).
  void quiesce(cudaStream_t s) noexcept {
    if (hub_) {
      cudaStreamSynchronize(s);
      hub_->barrier(std::chrono::milliseconds(10000));
      return;
    }
    int* one = nullptr;
    if (cudaMalloc(&one, sizeof(int)) != cudaSuccess) return;
    if (ncclAllReduce(one, one, 1, ncclInt32, ncclSum, comm_, s) == ncclSuccess) cudaStreamSynchronize(s);
    cudaFree(one);
  }

  void group_start() {
    if (!hub_) nccl_check(ncclGroupStart(), "ncclGroupStart");
  }
  void group_end() {
    if (!hub_) nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  }

  // In-place sum over the group of n fp64 / fp32 elements, stream-ordered on
  // s. Local group: every rank sums all ranks' buffers in rank order into
  // its scratch (same bits on every rank, as NCCL's allreduce), then copies
  // the result back once every rank has read its sources.
  void allreduce_sum(void* buf, size_t n, bool f64, cudaStream_t s) {
    if (!hub_) {
      nccl_check(ncclAllReduce(buf, buf, n, f64 ? ncclFloat64 : ncclFloat32, ncclSum, comm_, s),
                 "ncclAllReduce");
      return;
    }
    const size_t bytes = n * (f64 ? 8 : 4);
    if (bytes > scratch_bytes_) {
      throw_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
      if (scratch_) cudaFree(scratch_);
      scratch_ = nullptr;
      throw_cuda(cudaMalloc(&scratch_, bytes), "cudaMalloc");
      scratch_bytes_ = bytes;
    }
    hub_->ptr[rank_] = buf;
    throw_cuda(cudaEventRecord(hub_->ev_ready[rank_], s), "eventRecord");
    hub_->barrier();
    std::vector<const void*> src(hub_->ptr.begin(), hub_->ptr.end());
    for (int p = 0; p < world_; ++p)
      throw_cuda(cudaStreamWaitEvent(s, hub_->ev_ready[p], 0), "waitEvent");
    int rc = fsmoe_sum_buffers(f64 ? FSMOE_F64 : FSMOE_F32, world_, src.data(),
                               static_cast<long long>(n), scratch_, s);
    if (rc) throw DeviceError(fsmoe_last_error());
    throw_cuda(cudaEventRecord(hub_->ev_done[rank_], s), "eventRecord");
    hub_->barrier();
    for (int p = 0; p < world_; ++p)
      throw_cuda(cudaStreamWaitEvent(s, hub_->ev_done[p], 0), "waitEvent");
    throw_cuda(cudaMemcpyAsync(buf, scratch_, bytes, cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync");
  }

  ncclComm_t comm() const {
    if (hub_) throw ConfigError("ep: a local (single-device) group has no NCCL communicator");
    return comm_;
  }
  int world() const { return world_; }
  int rank() const { return rank_; }
  int device() const { return device_; }

 private:
  ncclComm_t comm_ = nullptr;
  int world_ = 1, rank_ = 0, device_ = 0;
  std::shared_ptr<LocalHub> hub_;
  void* scratch_ = nullptr;
  size_t scratch_bytes_ = 0;
};

}  // namespace fsmoe
