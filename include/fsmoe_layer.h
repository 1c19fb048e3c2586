/*
 * fsmoe_layer.h — C ABI of libfsmoe.so: the unified MoE layer (C++
 * fsmoe::MoELayer, include/fsmoe/moe_layer.hpp) and the expert-parallel NCCL
 * group, for hosts that bind through an FFI (ctypes here; see INTEGRATION.md
 * for the cgo / JNI shape of the same calls).
 *
 * Status codes as include/fsmoe_cuda.h (0 ok, 2 config, 3 fit quality,
 * 4 invariant, 5 device); message via fsmoe_layer_last_error().
 */
#ifndef FSMOE_LAYER_H
#define FSMOE_LAYER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fsmoe_ep fsmoe_ep;
typedef struct fsmoe_layer fsmoe_layer;

typedef struct fsmoe_layer_config {
  int tokens;          /* local tokens per rank */
  int model_dim;       /* M */
  int ffn_dim;         /* H */
  int experts;         /* E, global */
  int top_k;
  int gate_kind;       /* enum fsmoe_gate_kind */
  int ffn_kind;        /* 0 simple (2 GEMMs, GELU), 1 gated3 (3 GEMMs, SwiGLU) */
  long long capacity;  /* per (rank, expert); 0 -> capacity_tokens(k, capacity_factor, unlimited) */
  int proj_dim;        /* cosine_topk projection rows */
  uint64_t seed;       /* noisy_topk noise seed */
  int precision;       /* 0 bf16 (tcgen05), 1 fp32 check mode */
  int r_fwd, r_bwd;    /* pipeline degrees */
  int device;
  long long dense_grad_elems;   /* optional replicated fp32 gradient, allreduced in slices */
  int n_ar_slices;
  const long long* ar_slices;   /* slice sizes (elements), n_ar_slices entries */
  /* capacity = 0: capacity_tokens (workload.cpp:43-51) of B*L = tokens with
   * this factor (<= 0 means 1.0), or k * tokens when unlimited != 0 */
  double capacity_factor;
  int unlimited;
  /* EP exchange (P > 1): 0 = FSMOE_EP_TRANSPORT or "peer", 1 peer (row stores
   * fused into the producing kernels), 2 ce (FSMoE's chunked pipeline on the
   * copy engines for the dispatch side), 3 nccl (grouped send/recv) */
  int transport;
} fsmoe_layer_config;

typedef struct fsmoe_layer_params {
  double* w_gate;   /* score weights M x E (cosine: proj_dim x E), fp64 */
  double* w_noise;  /* M x E fp64 (noisy_topk) */
  double* proj;     /* proj_dim x M fp64 (cosine_topk) */
  void* w1;         /* [E_local][N1][M], N1 = H or 2H (gated3, 128-unit gate/up interleave) */
  void* w2;         /* [E_local][M][H] */
  double* g_gate;
  double* g_noise;
  double* g_proj;
  float* g_w1;
  float* g_w2;
  float* dense_grad;
} fsmoe_layer_params;

const char* fsmoe_layer_last_error(void);

/* NCCL bootstrap: rank 0 creates the id, the host broadcasts it. */
int fsmoe_ep_unique_id(unsigned char out[128]);
int fsmoe_ep_create(int world, int rank, const unsigned char id[128], int device, int max_ctas,
                    fsmoe_ep** out);
/* Single-GPU multi-rank harness: `world` logical ranks of one group on ONE
 * device, out[0..world-1] (no NCCL, no IPC; peer maps are plain device
 * pointers, collectives host barriers + a summation kernel). Each rank's
 * layer must be created and driven from its own host thread, exactly as one
 * process per GPU would drive it; the peer-memory transport then runs its
 * producer stores and arrival flags unchanged. Destroy each with
 * fsmoe_ep_destroy. */
int fsmoe_ep_create_local(int world, int device, fsmoe_ep** out);
int fsmoe_ep_destroy(fsmoe_ep* ep);
/* In-place sum of n fp32 (f64 = 0) or fp64 (f64 = 1) elements over the
 * group, stream-ordered on `stream` (NCCL allreduce; local group: barrier +
 * in-order summation, same bits on every rank). The tail of the gradient
 * partition plan (grad_partition.hpp) runs through it. */
int fsmoe_ep_allreduce(fsmoe_ep* ep, void* buf, long long n, int f64, void* stream);

/* ep may be NULL (single GPU, all experts local). */
int fsmoe_layer_create(const fsmoe_layer_config* cfg, fsmoe_ep* ep, fsmoe_layer** out);
int fsmoe_layer_destroy(fsmoe_layer* layer);
int fsmoe_layer_bind(fsmoe_layer* layer, const fsmoe_layer_params* params);
long long fsmoe_layer_capacity(const fsmoe_layer* layer);
int fsmoe_layer_forward(fsmoe_layer* layer, const void* x, void* y, void* stream);
int fsmoe_layer_backward(fsmoe_layer* layer, const void* dy, void* dx, void* stream);
/* Measured timeline: enable per-phase CUDA-event tracing (synchronises each
 * call); fsmoe_layer_trace copies the Chrome-trace JSON (fields and labels of
 * the schedule simulator, tid 0 = comm stream, 2 = compute stream) and
 * returns the bytes needed. */
int fsmoe_layer_set_trace(fsmoe_layer* layer, int on);
long long fsmoe_layer_trace(const fsmoe_layer* layer, char* buf, long long cap);
/* Named internal device buffer (pick_token, slot_of_pick, fill, X_send, Z,
 * wait_ns = uint64 nanoseconds the compute stream spent waiting on peers, ...). */
int fsmoe_layer_buffer(const fsmoe_layer* layer, const char* name, void** ptr, long long* bytes);

#ifdef __cplusplus
}
#endif
#endif
