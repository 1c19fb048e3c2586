// kernels.h — host launchers of the routing kernels (gate.cu, route.cu,
// gate_bwd.cu), called by the C ABI (capi_route.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "../../include/fsmoe_cuda.h"
#include "route_common.cuh"

namespace fsmoe {

// ABI peer map -> kernel argument; a plain buffer is the one-rank identity.
inline fsmoe_dev::PeerRows peer_rows_of(const fsmoe_peer_rows* m) {
  fsmoe_dev::PeerRows r{};
  r.world = m->world;
  r.rank = m->rank;
  r.el = m->experts_local;
  r.cap = m->capacity;
  for (int i = 0; i < fsmoe_dev::MAX_PEERS; ++i) r.base[i] = static_cast<char*>(m->base[i]);
  return r;
}
inline fsmoe_dev::PeerRows local_rows(void* buf) {
  fsmoe_dev::PeerRows r{};
  r.world = 1;
  r.el = 1;
  r.cap = 1;
  r.base[0] = static_cast<char*>(buf);
  return r;
}

size_t gate_workspace_bytes(const fsmoe_gate_desc& d);
int gate_launch(const fsmoe_gate_desc& d, const void* x, const double* w_score,
                const double* w_noise, const double* proj, int* pick_token, int* pick_expert,
                double* pick_weight, double* scores_out, double* noise_out, double* spread_out,
                double* proj_out, int* d_status, void* ws, size_t ws_bytes, cudaStream_t st);
void cosine_enorm(int P, int E, const double* w, double* en, cudaStream_t st);

// Pruned exact selection for noisy/sigmoid gates (gate_prune.cu).
bool gate_prune_applicable(const fsmoe_gate_desc& d);
size_t gate_prune_workspace_bytes(const fsmoe_gate_desc& d);
int gate_prune_launch(const fsmoe_gate_desc& d, const void* x, const double* w_score,
                      const double* w_noise, int* pick_token, int* pick_expert,
                      double* pick_weight, double* scores_out, double* noise_out,
                      double* spread_out, void* ws, cudaStream_t st);

size_t gate_bwd_workspace_bytes(const fsmoe_gate_desc& d);
int gate_bwd_launch(const fsmoe_gate_desc& d, const void* x, const double* w_score,
                    const double* w_noise, const double* proj, const int* ptok, const int* pexp,
                    const double* pw, const double* dw, const double* scores, const double* noise,
                    const double* spread, const double* proj_out, void* dx, double* dWs,
                    double* dWn, double* dP, void* ws, cudaStream_t st);

size_t assign_workspace_bytes(long long P, int E);
int assign_launch(long long P, const int* ptok, const int* pexp, int T, int E, long long C,
                  int* slot_of_pick, long long* fill, long long* dropped, int* pick_of_slot,
                  int* status, void* ws, cudaStream_t st);

size_t token_index_workspace_bytes(long long P, int T);
int token_index_launch(long long P, const int* ptok, int T, int k, int* tptr, int* tpick,
                       void* ws, cudaStream_t st);

int dispatch_launch(int dtype, int M, int E, long long C, int chunks, const int* pick_of_slot,
                    const int* ptok, const void* x, const fsmoe_dev::PeerRows& buf, cudaStream_t st,
                    const fsmoe_dev::RowRange& rr = fsmoe_dev::all_rows());
int combine_launch(int dtype, int T, int M, int E, long long C, int chunks, const int* tptr,
                   const int* tpick, const int* slot_of_pick, const double* pw, const void* buf,
                   void* y, cudaStream_t st);
int dispatch_bwd_launch(int dtype, int T, int M, int E, long long C, int chunks, const int* tptr,
                        const int* tpick, const int* slot_of_pick, const void* dbuf, void* dx,
                        int accumulate, cudaStream_t st);
int zero_rows_launch(long long n_rows, long long row_bytes, const int* idx, void* dst, cudaStream_t st);
int gather_rows_launch(long long n_rows, long long row_bytes, const int* idx, const void* src,
                       const fsmoe_dev::PeerRows& dst, cudaStream_t st);
int combine_bwd_launch(int dtype, int M, int E, long long C, int chunks, long long P,
                       const int* pick_of_slot, const int* ptok, const double* pw,
                       const void* dy, const void* buf, const fsmoe_dev::PeerRows& dbuf, double* dw,
                       cudaStream_t st, const fsmoe_dev::RowRange& rr = fsmoe_dev::all_rows());

}  // namespace fsmoe
