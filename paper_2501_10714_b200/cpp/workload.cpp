// workload.cpp — drop-in implementation of include/fsmoe/workload.hpp.
//
// Shape logic (validate / capacity_tokens / derive_volumes) is host-side
// arithmetic with the reference's exact semantics (proj/src/workload.cpp:
// 10-79). The routing entry points keep the reference's host-Matrix
// signatures (workload.hpp:110-132) but execute on the GPU through the C ABI
// of libfsmoe_cuda.so: inputs are uploaded, the sm_100a kernels run, results
// come back. There is no CPU implementation here.
#include "fsmoe/workload.hpp"

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>

#include "device_util.hpp"
#include "fsmoe_cuda.h"

namespace fsmoe {

void validate(const LayerConfig& cfg) {
  const std::pair<int, const char*> positive[] = {
      {cfg.batch, "batch"},         {cfg.heads, "heads"},     {cfg.seq_len, "seq_len"},
      {cfg.model_dim, "model_dim"}, {cfg.hidden_scale, "hidden_scale"},
      {cfg.experts, "experts"},     {cfg.top_k, "top_k"}};
  for (const auto& [v, name] : positive)
    if (v <= 0) throw ConfigError(std::string("layer: ") + name + " must be positive");
  if (!cfg.unlimited_capacity && cfg.capacity_factor <= 0.0)
    throw ConfigError("layer: capacity_factor must be positive");
  if (cfg.t_olp_dense_ms < 0.0) throw ConfigError("layer: t_olp_dense_ms must be nonnegative");
}

void validate(const ParallelConfig& p) {
  const std::pair<int, const char*> positive[] = {
      {p.total_gpus, "total_gpus"},           {p.gpus_per_node, "gpus_per_node"},
      {p.data_parallel, "data_parallel"},     {p.tensor_parallel, "tensor_parallel"},
      {p.expert_parallel, "expert_parallel"}, {p.expert_shard, "expert_shard"}};
  for (const auto& [v, name] : positive)
    if (v <= 0) throw ConfigError(std::string("parallel: ") + name + " must be positive");
  if (p.total_gpus % p.gpus_per_node != 0)
    throw ConfigError("parallel: total_gpus must be a multiple of gpus_per_node");
}

long long capacity_tokens(const LayerConfig& cfg) {
  validate(cfg);
  const double tokens = static_cast<double>(cfg.batch) * cfg.seq_len;
  if (cfg.unlimited_capacity) return static_cast<long long>(static_cast<double>(cfg.top_k) * tokens);
  const double v = cfg.top_k * cfg.capacity_factor * tokens / cfg.experts;
  return static_cast<long long>(std::ceil(v - 1e-9));
}

TaskVolumes derive_volumes(const LayerConfig& cfg, const ParallelConfig& pcfg) {
  validate(cfg);
  validate(pcfg);
  if (cfg.experts % pcfg.expert_parallel != 0)
    throw ConfigError("experts must divide evenly across expert_parallel groups");
  const double cap = static_cast<double>(capacity_tokens(cfg));
  const double m = cfg.model_dim;
  const double h = static_cast<double>(cfg.hidden_scale) * m;
  const double e_local = static_cast<double>(cfg.experts) / pcfg.expert_parallel;
  TaskVolumes v;
  v.capacity = static_cast<long long>(cap);
  v.a2a_elements = static_cast<double>(cfg.experts) * cap * m / pcfg.expert_shard;
  v.ag_elements = e_local * cap * m;
  v.rs_elements = v.ag_elements;
  v.gemm_macs = cap * m * h;
  v.gemm_count = cfg.ffn == LayerConfig::Ffn::gated3 ? 3 : 2;
  v.grad_elements = e_local * v.gemm_count * m * h / pcfg.expert_shard +
                    4.0 * m * m / pcfg.tensor_parallel;
  if (cfg.grad_elements_override) {
    if (*cfg.grad_elements_override < 0) throw ConfigError("grad_elements override must be >= 0");
    v.grad_elements = *cfg.grad_elements_override;
  }
  return v;
}

// --------------------------------------------------------------- routing --

namespace {

int kind_of(GateKind k) {
  switch (k) {
    case GateKind::noisy_topk: return FSMOE_GATE_NOISY_TOPK;
    case GateKind::sigmoid_topk: return FSMOE_GATE_SIGMOID_TOPK;
    case GateKind::cosine_topk: return FSMOE_GATE_COSINE_TOPK;
    case GateKind::expert_choice: return FSMOE_GATE_EXPERT_CHOICE;
  }
  return -1;
}

}  // namespace

GateOutput run_gate(const Matrix& tokens, const GateConfig& gcfg, const GateParams& params) {
  fsmoe_gate_desc d{};
  d.kind = kind_of(gcfg.kind);
  d.top_k = gcfg.top_k;
  d.seed = gcfg.seed;
  d.tokens = tokens.rows;
  d.model_dim = tokens.cols;
  d.x_dtype = FSMOE_F64;
  d.score_rows = params.score_weights.rows;
  d.score_cols = params.score_weights.cols;
  d.noise_rows = params.noise_weights.rows;
  d.noise_cols = params.noise_weights.cols;
  d.proj_rows = params.projection.rows;
  d.proj_cols = params.projection.cols;
  throw_on(fsmoe_gate_validate(&d));

  const int T = d.tokens, E = d.score_cols, k = d.top_k;
  const long long n = d.kind == FSMOE_GATE_EXPERT_CHOICE ? static_cast<long long>(E) * k
                                                         : static_cast<long long>(T) * k;
  DeviceScope dev;
  double* x = dev.upload(tokens.v);
  double* ws = dev.upload(params.score_weights.v);
  double* wn = d.kind == FSMOE_GATE_NOISY_TOPK ? dev.upload(params.noise_weights.v) : nullptr;
  double* pj = d.kind == FSMOE_GATE_COSINE_TOPK ? dev.upload(params.projection.v) : nullptr;
  int* tok = dev.alloc<int>(n);
  int* exp = dev.alloc<int>(n);
  double* w = dev.alloc<double>(n);
  int* status = dev.alloc<int>(2);
  dev.zero(status, 2);
  const size_t wsb = fsmoe_gate_workspace_size(&d);
  void* work = dev.alloc<char>(static_cast<long long>(wsb));
  throw_on(fsmoe_gate(&d, x, ws, wn, pj, tok, exp, w, nullptr, nullptr, nullptr, nullptr, status,
                      work, wsb, dev.stream()));
  throw_on(fsmoe_check_status(status, dev.stream()));

  std::vector<int> htok(n), hexp(n);
  std::vector<double> hw(n);
  dev.download(htok.data(), tok, n);
  dev.download(hexp.data(), exp, n);
  dev.download(hw.data(), w, n);
  GateOutput out;
  out.tokens = T;
  out.experts = E;
  out.picks.resize(static_cast<size_t>(n));
  for (long long i = 0; i < n; ++i) out.picks[i] = {htok[i], hexp[i], hw[i]};
  return out;
}

DispatchResult dispatch_tokens(const Matrix& tokens, const GateOutput& gate, long long capacity) {
  if (capacity <= 0) throw ConfigError("dispatch: capacity must be positive");
  const long long P = static_cast<long long>(gate.picks.size());
  const int E = gate.experts;
  DispatchResult r;
  r.experts = E;
  r.capacity = capacity;
  r.buffers = Matrix(static_cast<int>(E * capacity), tokens.cols);
  r.slot_of_pick.assign(static_cast<size_t>(P), -1);
  r.fill.assign(static_cast<size_t>(E > 0 ? E : 0), 0);
  if (E <= 0) {
    // Every pick names an unknown expert.
    if (P > 0) throw ConfigError("dispatch: pick references an unknown token or expert");
    return r;
  }
  std::vector<int> htok(P), hexp(P);
  for (long long i = 0; i < P; ++i) {
    htok[i] = gate.picks[i].token;
    hexp[i] = gate.picks[i].expert;
  }
  DeviceScope dev;
  int* tok = dev.upload(htok);
  int* exp = dev.upload(hexp);
  int* slot = dev.alloc<int>(P);
  long long* fill = dev.alloc<long long>(E);
  long long* dropped = dev.alloc<long long>(1);
  int* pos = dev.alloc<int>(static_cast<long long>(E) * capacity);
  int* status = dev.alloc<int>(2);
  dev.zero(status, 2);
  const size_t wsb = fsmoe_assign_workspace_size(P, E);
  void* work = dev.alloc<char>(static_cast<long long>(wsb));
  throw_on(fsmoe_assign(P, tok, exp, tokens.rows, E, capacity, slot, fill, dropped, pos, status,
                        work, wsb, dev.stream()));
  throw_on(fsmoe_check_status(status, dev.stream()));
  if (tokens.cols > 0 && E * capacity > 0) {
    double* x = dev.upload(tokens.v);
    double* buf = dev.alloc<double>(static_cast<long long>(E) * capacity * tokens.cols);
    throw_on(fsmoe_dispatch(FSMOE_F64, tokens.cols, E, capacity, 1, pos, tok, x, buf,
                            dev.stream()));
    dev.download(r.buffers.v.data(), buf, static_cast<long long>(r.buffers.v.size()));
  }
  dev.download(r.slot_of_pick.data(), slot, P);
  dev.download(r.fill.data(), fill, E);
  dev.download(&r.dropped, dropped, 1);
  return r;
}

Matrix combine_tokens(const Matrix& expert_buffers, const GateOutput& gate,
                      const DispatchResult& layout, int model_dim) {
  if (expert_buffers.cols != model_dim)
    throw ConfigError("combine: buffer width does not match model_dim");
  if (layout.slot_of_pick.size() != gate.picks.size())
    throw ConfigError("combine: layout does not match the gate output");
  const long long P = static_cast<long long>(gate.picks.size());
  const int T = gate.tokens;
  Matrix y(T, model_dim);
  if (T <= 0 || model_dim <= 0) return y;
  std::vector<int> htok(P), hslot(P);
  std::vector<double> hw(P);
  for (long long i = 0; i < P; ++i) {
    htok[i] = gate.picks[i].token;
    hw[i] = gate.picks[i].weight;
    hslot[i] = layout.slot_of_pick[i];
    if (hslot[i] >= expert_buffers.rows)
      throw ConfigError("combine: slot outside the expert buffers");
  }
  // Buffers are addressed as (rows x model_dim) with slot = row (chunks = 1):
  // pass experts = 1, capacity = rows so the row map is the identity.
  DeviceScope dev;
  int* tok = dev.upload(htok);
  int* slot = dev.upload(hslot);
  double* w = dev.upload(hw);
  double* buf = dev.upload(expert_buffers.v);
  int* tptr = dev.alloc<int>(T + 1);
  int* tpick = dev.alloc<int>(P);
  const size_t wsb = fsmoe_token_index_workspace_size(P, T);
  void* work = dev.alloc<char>(static_cast<long long>(wsb));
  throw_on(fsmoe_token_index(P, tok, T, 0, tptr, tpick, work, wsb, dev.stream()));
  double* out = dev.alloc<double>(static_cast<long long>(T) * model_dim);
  const long long rows = expert_buffers.rows > 0 ? expert_buffers.rows : 1;
  throw_on(fsmoe_combine(FSMOE_F64, T, model_dim, 1, rows, 1, tptr, tpick, slot, w, buf, out,
                         dev.stream()));
  dev.download(y.v.data(), out, static_cast<long long>(y.v.size()));
  return y;
}

}  // namespace fsmoe
