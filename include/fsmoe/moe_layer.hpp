// fsmoe/moe_layer.hpp — the unified MoE module on the B200: gate -> order ->
// AlltoAll -> expert FFN (tcgen05 grouped GEMM) -> AlltoAll -> I-order,
// forward and backward, expert-parallel over NCCL with the FSMoE chunked
// pipeline (degree r_fwd / r_bwd) and gradient-allreduce slices placed in the
// backward's inter-link window (§4-5; schedule_sim.cpp:182-216).
//
// Not part of the reference library (which simulates this schedule but never
// executes it); its task kinds map 1:1 to the simulator's OpKind values.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "fsmoe/workload.hpp"

namespace fsmoe {

enum class Precision { bf16 = 0, f32 = 1 };

struct MoELayerConfig {
  int tokens = 0;      // local tokens per rank
  int model_dim = 0;   // M
  int ffn_dim = 0;     // H
  int experts = 0;     // E (global)
  int top_k = 1;
  GateKind gate = GateKind::noisy_topk;
  LayerConfig::Ffn ffn = LayerConfig::Ffn::simple;  // simple = GELU, gated3 = SwiGLU
  long long capacity = 0;  // per (rank, expert); 0 -> capacity_tokens(k, f, unlimited)
  double capacity_factor = 1.0;     // LayerConfig::capacity_factor (workload.hpp:24)
  bool unlimited_capacity = false;  // LayerConfig::unlimited_capacity (workload.hpp:25)
  int proj_dim = 0;        // cosine_topk
  std::uint64_t seed = 0;
  Precision precision = Precision::bf16;
  int r_fwd = 1;           // pipeline degrees (chunks of 128-row granules)
  int r_bwd = 1;
  int device = 0;
  long long dense_grad_elems = 0;  // optional replicated-gradient buffer (fp32)
  std::vector<long long> ar_slices;  // allreduce slice sizes (elements); empty -> one
  // EP exchange: 0 = FSMOE_EP_TRANSPORT or peer, 1 = peer stores fused into
  // the producers, 2 = ce (chunked copy-engine dispatch), 3 = nccl send/recv
  int transport = 0;
};

class EpGroup;  // NCCL communicator over the expert-parallel ranks

struct MoEParams {
  double* w_gate = nullptr;   // score weights (M x E, or proj_dim x E)
  double* w_noise = nullptr;  // M x E
  double* proj = nullptr;     // proj_dim x M
  void* w1 = nullptr;         // [E_l][N1][M]   N1 = H (simple) or 2H interleaved (gated3)
  void* w2 = nullptr;         // [E_l][M][H]
  double* g_gate = nullptr;
  double* g_noise = nullptr;
  double* g_proj = nullptr;
  float* g_w1 = nullptr;
  float* g_w2 = nullptr;
  float* dense_grad = nullptr;  // dense_grad_elems (allreduced in backward slots)
};

class MoELayer {
 public:
  MoELayer(const MoELayerConfig& cfg, EpGroup* ep);
  ~MoELayer();
  MoELayer(const MoELayer&) = delete;
  MoELayer& operator=(const MoELayer&) = delete;

  void bind(const MoEParams& p);
  // x, y, dy, dx: tokens x model_dim (bf16 or f32 per precision), device.
  void forward(const void* x, void* y, void* stream);
  void backward(const void* dy, void* dx, void* stream);

  const MoELayerConfig& config() const { return cfg_; }
  long long capacity() const { return cap_; }
  int local_experts() const { return el_; }
  int world() const { return world_; }
  // Named internal device buffers (for tests / inspection).
  void* buffer(const std::string& name, long long* bytes) const;
  long long dropped_host() const;  // synchronises
  // Measured per-phase timeline (CUDA events on both streams; Chrome trace
  // JSON with the schedule simulator's fields). Tracing synchronises each call.
  void set_trace(bool on);
  std::string trace_json() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
  MoELayerConfig cfg_;
  long long cap_ = 0;
  int el_ = 0;
  int world_ = 1;
};

}  // namespace fsmoe
