// capi_route.cu — extern "C" routing entry points (include/fsmoe_cuda.h).
// Host-side validation reproduces the reference's ConfigError checks and
// messages (workload.cpp:135-159,173-174,237-240,266-271) before any launch.
#include <cuda_runtime.h>

#include <string>

#include "capi_common.h"
#include "kernels.h"
#include "route_common.cuh"

namespace {

using namespace fsmoe;

int dims_error(const char* name, int r, int c) {
  return config_error(std::string("gate: ") + name + " must be " + std::to_string(r) + "x" +
                      std::to_string(c));
}

int validate_gate(const fsmoe_gate_desc* d) {
  if (!d) return config_error("gate: null descriptor");
  const int T = d->tokens, M = d->model_dim, E = d->score_cols, k = d->top_k;
  if (T <= 0 || M <= 0) return config_error("gate: empty token matrix");
  if (E <= 0) return config_error("gate: no experts");
  if (k <= 0) return config_error("gate: top_k must be positive");
  switch (d->kind) {
    case FSMOE_GATE_EXPERT_CHOICE:
      if (k > T) return config_error("gate: expert capacity exceeds token count");
      if (d->score_rows != M) return dims_error("score_weights", M, E);
      return FSMOE_OK;
    case FSMOE_GATE_NOISY_TOPK:
      if (k > E) return config_error("gate: top_k exceeds expert count");
      if (d->score_rows != M) return dims_error("score_weights", M, E);
      if (d->noise_rows != M || d->noise_cols != E) return dims_error("noise_weights", M, E);
      break;
    case FSMOE_GATE_SIGMOID_TOPK:
      if (k > E) return config_error("gate: top_k exceeds expert count");
      if (d->score_rows != M) return dims_error("score_weights", M, E);
      break;
    case FSMOE_GATE_COSINE_TOPK: {
      if (k > E) return config_error("gate: top_k exceeds expert count");
      const int P = d->proj_rows;
      if (d->proj_cols != M) return dims_error("projection", P, M);
      if (d->score_rows != P) return dims_error("score_weights", P, E);
      if (P <= 0) return config_error("gate: projected token has zero norm");
      break;
    }
    default:
      return config_error("gate: unknown gate kind");
  }
  if (E > 256) return config_error("gate: at most 256 experts supported");
  if (d->x_dtype < FSMOE_F64 || d->x_dtype > FSMOE_BF16) return config_error("gate: unknown x dtype");
  return FSMOE_OK;
}

int check_dtype(int dtype) {
  if (dtype < FSMOE_F64 || dtype > FSMOE_BF16) return config_error("unknown dtype");
  return FSMOE_OK;
}

}  // namespace

extern "C" {

size_t fsmoe_gate_workspace_size(const fsmoe_gate_desc* d) {
  return d ? gate_workspace_bytes(*d) : 0;
}

int fsmoe_gate_validate(const fsmoe_gate_desc* d) { return validate_gate(d); }

int fsmoe_gate(const fsmoe_gate_desc* d, const void* x, const double* w_score,
               const double* w_noise, const double* proj, int* pick_token, int* pick_expert,
               double* pick_weight, double* scores_out, double* noise_out, double* spread_out,
               double* proj_out, int* d_status, void* workspace, size_t workspace_bytes,
               void* stream) {
  if (int rc = validate_gate(d)) return rc;
  if (workspace_bytes < gate_workspace_bytes(*d)) return config_error("gate: workspace too small");
  return gate_launch(*d, x, w_score, w_noise, proj, pick_token, pick_expert, pick_weight,
                     scores_out, noise_out, spread_out, proj_out, d_status, workspace,
                     workspace_bytes, as_stream(stream));
}

int fsmoe_check_status(const int* d_status, void* stream) {
  if (!d_status) return FSMOE_OK;
  int h = 0;
  FSMOE_CUDA_TRY(cudaMemcpyAsync(&h, d_status, sizeof(int), cudaMemcpyDeviceToHost,
                                 as_stream(stream)),
                 "fsmoe_check_status");
  FSMOE_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)), "fsmoe_check_status");
  // Reference order: token 0's projection norm is checked before any expert
  // norm; the expert norm fails at token 0 otherwise (workload.cpp:205-222).
  if (h & 2) return config_error("gate: projected token has zero norm");
  if (h & 4) return config_error("gate: expert embedding has zero norm");
  if (h & 1) return config_error("gate: projected token has zero norm");
  if (h & 8) return config_error("dispatch: pick references an unknown token or expert");
  return FSMOE_OK;
}

size_t fsmoe_assign_workspace_size(long long n_picks, int experts) {
  return assign_workspace_bytes(n_picks, experts);
}

int fsmoe_assign(long long n_picks, const int* pick_token, const int* pick_expert, int tokens,
                 int experts, long long capacity, int* slot_of_pick, long long* fill,
                 long long* dropped, int* pick_of_slot, int* d_status, void* workspace,
                 size_t workspace_bytes, void* stream) {
  if (capacity <= 0) return config_error("dispatch: capacity must be positive");
  if (experts <= 0) return config_error("dispatch: no experts");
  if (static_cast<long long>(experts) * capacity > 0x7FFFFFFFLL)
    return config_error("dispatch: experts*capacity exceeds int32 slot range");
  if (workspace_bytes < assign_workspace_bytes(n_picks, experts))
    return config_error("dispatch: workspace too small");
  return assign_launch(n_picks, pick_token, pick_expert, tokens, experts, capacity, slot_of_pick,
                       fill, dropped, pick_of_slot, d_status, workspace, as_stream(stream));
}

size_t fsmoe_token_index_workspace_size(long long n_picks, int tokens) {
  return token_index_workspace_bytes(n_picks, tokens);
}

int fsmoe_token_index(long long n_picks, const int* pick_token, int tokens, int token_major_k,
                      int* tok_ptr, int* tok_pick, void* workspace, size_t workspace_bytes,
                      void* stream) {
  if (tokens < 0) return config_error("token_index: negative token count");
  if (token_major_k > 0 && n_picks != static_cast<long long>(tokens) * token_major_k)
    return config_error("token_index: token-major layout needs tokens*k picks");
  if (token_major_k <= 0 && workspace_bytes < token_index_workspace_bytes(n_picks, tokens))
    return config_error("token_index: workspace too small");
  return token_index_launch(n_picks, pick_token, tokens, token_major_k, tok_ptr, tok_pick,
                            workspace, as_stream(stream));
}

long long fsmoe_slot_row(long long slot, int experts, long long capacity, int chunks) {
  return fsmoe_dev::slot_row(slot, experts, capacity, chunks);
}

int fsmoe_dispatch(int dtype, int model_dim, int experts, long long capacity, int chunks,
                   const int* pick_of_slot, const int* pick_token, const void* x, void* buffers,
                   void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (capacity <= 0) return config_error("dispatch: capacity must be positive");
  if (chunks < 1 || chunks > capacity) return config_error("dispatch: chunks must be in [1, capacity]");
  return dispatch_launch(dtype, model_dim, experts, capacity, chunks, pick_of_slot, pick_token, x,
                         local_rows(buffers), as_stream(stream));
}

static int check_peer_map(const fsmoe_peer_rows* m, int experts, long long capacity) {
  if (!m) return config_error("peer map: null");
  if (m->world < 1 || m->world > FSMOE_MAX_PEERS || m->rank < 0 || m->rank >= m->world)
    return config_error("peer map: world must be in [1, 8] and rank in [0, world)");
  if (m->experts_local * m->world != experts || m->capacity != capacity)
    return config_error("peer map: experts_local * world must equal experts and capacity match");
  for (int p = 0; p < m->world; ++p)
    if (!m->base[p]) return config_error("peer map: missing peer buffer");
  return FSMOE_OK;
}

int fsmoe_dispatch_peer(int dtype, int model_dim, int experts, long long capacity,
                        const int* pick_of_slot, const int* pick_token, const void* x,
                        const fsmoe_peer_rows* dst, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (capacity <= 0) return config_error("dispatch: capacity must be positive");
  if (int rc = check_peer_map(dst, experts, capacity)) return rc;
  return dispatch_launch(dtype, model_dim, experts, capacity, 1, pick_of_slot, pick_token, x,
                         peer_rows_of(dst), as_stream(stream));
}

int fsmoe_dispatch_peer_range(int dtype, int model_dim, int experts, long long capacity,
                              const int* pick_of_slot, const int* pick_token, const void* x,
                              const fsmoe_peer_rows* dst, long long slot_lo, long long slot_hi,
                              int exclude, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (capacity <= 0) return config_error("dispatch: capacity must be positive");
  if (int rc = check_peer_map(dst, experts, capacity)) return rc;
  return dispatch_launch(dtype, model_dim, experts, capacity, 1, pick_of_slot, pick_token, x,
                         peer_rows_of(dst), as_stream(stream),
                         fsmoe_dev::RowRange{slot_lo, slot_hi, exclude});
}

int fsmoe_combine_bwd_peer_range(int dtype, int model_dim, int experts, long long capacity,
                                 long long n_picks, const int* pick_of_slot, const int* pick_token,
                                 const double* pick_weight, const void* dy, const void* buffers,
                                 const fsmoe_peer_rows* d_dst, double* d_weight, long long slot_lo,
                                 long long slot_hi, int exclude, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (int rc = check_peer_map(d_dst, experts, capacity)) return rc;
  return combine_bwd_launch(dtype, model_dim, experts, capacity, 1, n_picks, pick_of_slot,
                            pick_token, pick_weight, dy, buffers, peer_rows_of(d_dst), d_weight,
                            as_stream(stream), fsmoe_dev::RowRange{slot_lo, slot_hi, exclude});
}

int fsmoe_combine_bwd_peer(int dtype, int model_dim, int experts, long long capacity,
                           long long n_picks, const int* pick_of_slot, const int* pick_token,
                           const double* pick_weight, const void* dy, const void* buffers,
                           const fsmoe_peer_rows* d_dst, double* d_weight, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (int rc = check_peer_map(d_dst, experts, capacity)) return rc;
  return combine_bwd_launch(dtype, model_dim, experts, capacity, 1, n_picks, pick_of_slot,
                            pick_token, pick_weight, dy, buffers, peer_rows_of(d_dst), d_weight,
                            as_stream(stream));
}

int fsmoe_combine(int dtype, int tokens, int model_dim, int experts, long long capacity,
                  int chunks, const int* tok_ptr, const int* tok_pick, const int* slot_of_pick,
                  const double* pick_weight, const void* buffers, void* y, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (chunks < 1 || (capacity > 0 && chunks > capacity))
    return config_error("combine: chunks must be in [1, capacity]");
  return combine_launch(dtype, tokens, model_dim, experts, capacity, chunks, tok_ptr, tok_pick,
                        slot_of_pick, pick_weight, buffers, y, as_stream(stream));
}

int fsmoe_combine_bwd(int dtype, int tokens, int model_dim, int experts, long long capacity,
                      int chunks, long long n_picks, const int* pick_of_slot,
                      const int* pick_token, const double* pick_weight, const int* slot_of_pick,
                      const void* dy, const void* buffers, void* d_buffers, double* d_weight,
                      void* stream) {
  (void)tokens;
  (void)slot_of_pick;
  if (int rc = check_dtype(dtype)) return rc;
  return combine_bwd_launch(dtype, model_dim, experts, capacity, chunks, n_picks, pick_of_slot,
                            pick_token, pick_weight, dy, buffers, local_rows(d_buffers), d_weight,
                            as_stream(stream));
}

int fsmoe_dispatch_bwd(int dtype, int tokens, int model_dim, int experts, long long capacity,
                       int chunks, const int* tok_ptr, const int* tok_pick,
                       const int* slot_of_pick, const void* d_buffers, void* dx, int accumulate,
                       void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  return dispatch_bwd_launch(dtype, tokens, model_dim, experts, capacity, chunks, tok_ptr,
                             tok_pick, slot_of_pick, d_buffers, dx, accumulate,
                             as_stream(stream));
}

size_t fsmoe_gate_bwd_workspace_size(const fsmoe_gate_desc* d) {
  return d ? gate_bwd_workspace_bytes(*d) : 0;
}

int fsmoe_gate_bwd(const fsmoe_gate_desc* d, const void* x, const double* w_score,
                   const double* w_noise, const double* proj, const int* pick_token,
                   const int* pick_expert, const double* pick_weight, const double* d_weight,
                   const double* scores, const double* noise, const double* spread,
                   const double* proj_out, void* dx, double* d_w_score, double* d_w_noise,
                   double* d_proj, void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = validate_gate(d)) return rc;
  if (workspace_bytes < gate_bwd_workspace_bytes(*d))
    return config_error("gate_bwd: workspace too small");
  return gate_bwd_launch(*d, x, w_score, w_noise, proj, pick_token, pick_expert, pick_weight,
                         d_weight, scores, noise, spread, proj_out, dx, d_w_score, d_w_noise,
                         d_proj, workspace, as_stream(stream));
}

}  // extern "C"

int fsmoe_zero_rows(int dtype, int model_dim, long long n_rows, const int* src_row, void* dst,
                    void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (model_dim <= 0) return config_error("zero_rows: model_dim must be positive");
  const long long rb = static_cast<long long>(model_dim) * (dtype == FSMOE_F64 ? 8 : dtype == FSMOE_F32 ? 4 : 2);
  return zero_rows_launch(n_rows, rb, src_row, dst, as_stream(stream));
}

int fsmoe_gather_rows(int dtype, int model_dim, long long n_rows, const int* src_row,
                      const void* src, void* dst, const fsmoe_peer_rows* dst_map, void* stream) {
  if (int rc = check_dtype(dtype)) return rc;
  if (model_dim <= 0) return config_error("gather_rows: model_dim must be positive");
  const long long rb = static_cast<long long>(model_dim) * (dtype == FSMOE_F64 ? 8 : dtype == FSMOE_F32 ? 4 : 2);
  if (dst_map) {
    if (dst_map->world < 1 || dst_map->world > FSMOE_MAX_PEERS || dst_map->experts_local < 1 ||
        dst_map->capacity < 1)
      return config_error("gather_rows: bad peer map");
    return gather_rows_launch(n_rows, rb, src_row, src, peer_rows_of(dst_map), as_stream(stream));
  }
  return gather_rows_launch(n_rows, rb, src_row, src, local_rows(dst), as_stream(stream));
}
