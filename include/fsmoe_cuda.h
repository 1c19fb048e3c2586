/*
 * fsmoe_cuda.h — C ABI of libfsmoe_cuda.so, the B200 (sm_100a) kernels behind
 * the FSMoE MoE-layer hot path.
 *
 * Plain C: device pointers, sizes and an opaque stream (cudaStream_t passed as
 * void*); no torch or C++ types. All calls are stream-ordered and do not
 * synchronise unless stated. Return value: 0 = ok, 2 = config error (the
 * reference's fsmoe::ConfigError / exit_config_error, common.hpp:9-18),
 * 4 = invariant error, 5 = CUDA error. fsmoe_last_error() returns the
 * message of the last failure on the calling thread, using the reference's
 * exception texts where the reference defines them (workload.cpp).
 *
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/proj/src). The reference is a C++ library whose routing
 * functions take host fsmoe::Matrix values; the C++ drop-in (libfsmoe.so,
 * include/fsmoe/workload.hpp) keeps those signatures and calls this ABI.
 */
#ifndef FSMOE_CUDA_H
#define FSMOE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum fsmoe_status {
  FSMOE_OK = 0,
  FSMOE_CONFIG_ERROR = 2,    /* common.hpp:11 exit_config_error */
  FSMOE_INVARIANT_ERROR = 4, /* common.hpp:13 exit_invariant */
  FSMOE_CUDA_ERROR = 5
};

/* GateKind, workload.hpp:75 (same enumerator order). */
enum fsmoe_gate_kind {
  FSMOE_GATE_NOISY_TOPK = 0,
  FSMOE_GATE_SIGMOID_TOPK = 1,
  FSMOE_GATE_COSINE_TOPK = 2,
  FSMOE_GATE_EXPERT_CHOICE = 3
};

enum fsmoe_dtype { FSMOE_F64 = 0, FSMOE_F32 = 1, FSMOE_BF16 = 2 };

const char* fsmoe_last_error(void);
int fsmoe_abi_version(void);
/* Utilities: stream-ordered device-to-device copy; select the CUDA device of
 * the calling thread. */
int fsmoe_copy_device(void* dst, const void* src, size_t bytes, void* stream);
int fsmoe_set_device(int device);
/* Number of kernels launched by this library since load (bench evidence). */
long long fsmoe_launch_count(void);

/* ---------------------------------------------------------------- routing --
 * Replaces fsmoe::run_gate (workload.hpp:110-111, workload.cpp:143-235).
 * Logits are computed in fp64 with the reference's sequential j-order and no
 * FMA; top-k ties go to the lowest index; picks are token-major (token
 * choice) or expert-major (expert_choice), exactly as the reference emits
 * them. n_picks = tokens*top_k (token choice) or experts*top_k (EC).
 */
typedef struct fsmoe_gate_desc {
  int kind;         /* enum fsmoe_gate_kind */
  int top_k;        /* per token, or tokens per expert for expert_choice */
  uint64_t seed;    /* GateConfig::seed (noisy_topk) */
  int tokens;       /* rows of the token matrix */
  int model_dim;    /* cols of the token matrix */
  int x_dtype;      /* enum fsmoe_dtype of x (values are used exactly, upcast to fp64) */
  int score_rows, score_cols; /* GateParams::score_weights shape, cols = experts */
  int noise_rows, noise_cols; /* GateParams::noise_weights shape */
  int proj_rows, proj_cols;   /* GateParams::projection shape */
} fsmoe_gate_desc;

/* Device workspace bytes for fsmoe_gate (0 is valid). */
size_t fsmoe_gate_workspace_size(const fsmoe_gate_desc* d);

/* Host-side validation only (no device access): the reference's ConfigError
 * checks of run_gate (workload.cpp:148-159,173-174,135-139). */
int fsmoe_gate_validate(const fsmoe_gate_desc* d);

/* x: tokens x model_dim (x_dtype). w_score/w_noise/proj: row-major fp64.
 * scores_out (optional, tokens x experts fp64): final per-token scores
 * (post-noise / cosine) used by the gate backward; noise_out / spread_out
 * (optional, noisy only, tokens x experts): the normal draws and x.W_noise.
 * proj_out (optional, cosine only, tokens x proj_rows).
 * d_status (optional, device int[2]): data-dependent errors (cosine zero
 * norms), read with fsmoe_check_status. */
int fsmoe_gate(const fsmoe_gate_desc* d, const void* x, const double* w_score,
               const double* w_noise, const double* proj, int* pick_token,
               int* pick_expert, double* pick_weight, double* scores_out,
               double* noise_out, double* spread_out, double* proj_out,
               int* d_status, void* workspace, size_t workspace_bytes, void* stream);

/* Parity audit of the gate's libm (no reference counterpart): y = f(x) on
 * the device for fn 0 log, 1 exp, 2 log1p, 3 cos, 4 the normal draw
 * sqrt(-2 log x) cos(2 pi x2) (workload.cpp:90-95), 5 softplus
 * log1p(exp(x)) (101); impl 0 = the glibc 2.39 restatement the gate runs
 * (bit-identical to the host libm the reference calls), 1 = CUDA's libm. */
int fsmoe_libm_eval(int fn, int impl, const double* x, const double* x2, double* y, long long n,
                    void* stream);

/* Synchronises `stream`, reads the device status word written by gate /
 * assign and converts it to the reference's ConfigError (return 2 + message). */
int fsmoe_check_status(const int* d_status, void* stream);

/* Capacity assignment: replaces the loop of fsmoe::dispatch_tokens
 * (workload.cpp:248-262). For picks in order, a pick is kept iff fewer than
 * `capacity` earlier picks chose the same expert; slot = expert*capacity +
 * rank. Outputs: slot_of_pick[n_picks] (-1 = dropped), fill[experts],
 * dropped[1], pick_of_slot[experts*capacity] (-1 = padding). */
size_t fsmoe_assign_workspace_size(long long n_picks, int experts);
int fsmoe_assign(long long n_picks, const int* pick_token, const int* pick_expert,
                 int tokens, int experts, long long capacity, int* slot_of_pick,
                 long long* fill, long long* dropped, int* pick_of_slot, int* d_status,
                 void* workspace, size_t workspace_bytes, void* stream);

/* Per-token pick lists in pick order (CSR): tok_ptr[tokens+1], tok_pick[n_picks].
 * token_major_k > 0 declares the reference's token-choice layout (k picks per
 * token, token-major) and skips the sort. */
size_t fsmoe_token_index_workspace_size(long long n_picks, int tokens);
int fsmoe_token_index(long long n_picks, const int* pick_token, int tokens, int token_major_k,
                      int* tok_ptr, int* tok_pick, void* workspace, size_t workspace_bytes,
                      void* stream);

/* Slot -> buffer row. chunks = pipeline degree r: capacity rows split into r
 * ranges [floor(i*C/r), floor((i+1)*C/r)); the buffer is chunk-major
 * (r, experts, len_i, model_dim) so chunk i is one contiguous, expert-major
 * (hence rank-major) block for the AlltoAll. chunks = 1 is the reference's
 * (experts*capacity) x model_dim layout. */
long long fsmoe_slot_row(long long slot, int experts, long long capacity, int chunks);

/* Token dispatch (Order): replaces the copy of dispatch_tokens
 * (workload.cpp:257-259) incl. the zero padding of unused slots. */
int fsmoe_dispatch(int dtype, int model_dim, int experts, long long capacity, int chunks,
                   const int* pick_of_slot, const int* pick_token, const void* x,
                   void* buffers, void* stream);

/* Weighted combine (I-Order): replaces combine_tokens (workload.cpp:266-282).
 * y[t] = sum over t's kept picks, in pick order, of weight * buffers[slot]
 * (fp64: separate multiply and add, bit-identical to the reference). */
int fsmoe_combine(int dtype, int tokens, int model_dim, int experts, long long capacity,
                  int chunks, const int* tok_ptr, const int* tok_pick, const int* slot_of_pick,
                  const double* pick_weight, const void* buffers, void* y, void* stream);

/* ------------------------------------------------------------- backward --
 * The reference has no backward; semantics follow SURVEY.md
 * Appendix D. */

/* d_buffers[slot] = w_p * dy[t_p] (0 for padding); d_weight[p] = <dy[t_p], buffers[slot_p]>
 * (0 for dropped picks). */
int fsmoe_combine_bwd(int dtype, int tokens, int model_dim, int experts, long long capacity,
                      int chunks, long long n_picks, const int* pick_of_slot,
                      const int* pick_token, const double* pick_weight, const int* slot_of_pick,
                      const void* dy, const void* buffers, void* d_buffers, double* d_weight,
                      void* stream);

/* dx[t] (+)= sum over t's kept picks (pick order) of d_buffers[slot]. */
int fsmoe_dispatch_bwd(int dtype, int tokens, int model_dim, int experts, long long capacity,
                       int chunks, const int* tok_ptr, const int* tok_pick,
                       const int* slot_of_pick, const void* d_buffers, void* dx, int accumulate,
                       void* stream);

/* Gate backward: d_weight (per pick) -> d scores -> parameter grads (fp64,
 * accumulated into d_w_*) and dx (fp32/bf16/f64 per x_dtype, accumulated). */
size_t fsmoe_gate_bwd_workspace_size(const fsmoe_gate_desc* d);
int fsmoe_gate_bwd(const fsmoe_gate_desc* d, const void* x, const double* w_score,
                   const double* w_noise, const double* proj, const int* pick_token,
                   const int* pick_expert, const double* pick_weight, const double* d_weight,
                   const double* scores, const double* noise, const double* spread,
                   const double* proj_out, void* dx, double* d_w_score, double* d_w_noise,
                   double* d_proj, void* workspace, size_t workspace_bytes, void* stream);

/* ----------------------------------------------------------- expert FFN --
 * Grouped GEMM (absent in the reference beyond gemm_count, workload.cpp:70).
 * precision 0: bf16 operands on tcgen05 tensor cores (fp32 accumulate in
 * TMEM, TMA-fed); 1: fp32 SIMT check mode. See csrc/gemm.h for the two
 * problem shapes. */
/* ---- peer memory (NVLink / NVSwitch) ------------------------------------
 * The dispatch / combine AlltoAlls of the MoE layer are not separate
 * collectives here: the kernel that produces a [P][E_l][C] block buffer
 * (dispatch, combine backward, the expert GEMM epilogues) stores each row
 * straight into the owning rank's buffer through CUDA-IPC-mapped peer
 * pointers. A row of block b = p*E_l + e_l lands in base[p] at row
 * (rank*E_l + e_l)*C + r%C (the receiver's layout is [P][E_l][C] by source
 * rank). world = 1, rank = 0, base[0] = local buffer is the identity.
 * Replaces the a2a tasks the reference only simulates (schedule_sim.cpp
 * OpKind::a2a_dispatch / a2a_combine). */
#define FSMOE_MAX_PEERS 8
typedef struct fsmoe_peer_rows {
  void* base[FSMOE_MAX_PEERS];
  int world, rank, experts_local;
  long long capacity;
} fsmoe_peer_rows;

/* Arrival flags: uint64 [nslots][world] in every rank's (IPC-shared) memory;
 * signal adds 1 to flag[slot][rank] on every peer (release, system scope)
 * after the stream's previous work, wait spins (acquire) until every
 * flag[slot][src] >= target. Counters only grow: target = uses of the slot. */
typedef struct fsmoe_peer_flags {
  unsigned long long* base[FSMOE_MAX_PEERS];  /* per-rank flag arrays (base[rank] = local) */
  int world, rank, nslots;
  /* optional device counter: every wait adds the nanoseconds (globaltimer) it
   * spent spinning, i.e. the time the stream was stalled on the exchange */
  unsigned long long* wait_ns;
  /* a wait stuck longer than this traps (lost peer); 0 = wait forever */
  unsigned long long timeout_ns;
} fsmoe_peer_flags;

/* Optionally puts a small [P][E_l] row buffer (put_src, rows of put_row_bytes,
 * mapped by put_dst with capacity 1) before raising the flag. */
int fsmoe_peer_signal(const fsmoe_peer_flags* f, int slot, const void* put_src,
                      long long put_row_bytes, const fsmoe_peer_rows* put_dst, void* stream);
int fsmoe_peer_wait(const fsmoe_peer_flags* f, int slot, unsigned long long target, void* stream);
/* dst[i] = src[0][i] + src[1][i] + ... + src[n_src-1][i] (in that order, so
 * every caller of the same sources gets the same bits), dtype F64 or F32,
 * n_src <= FSMOE_MAX_PEERS; dst may alias a source. The allreduce of an
 * expert-parallel group whose ranks share one device (the single-GPU
 * multi-rank harness, fsmoe_ep_create_local in fsmoe_layer.h). */
int fsmoe_sum_buffers(int dtype, int n_src, const void* const* src, long long n, void* dst,
                      void* stream);
/* Copy-engine exchange of one pipeline chunk (no SM work): for every rank p
 * (p == rank only with include_self), rows [lo, hi) of the E_l blocks
 * destined to p in the local canonical send buffer (block b = p*E_l + e_l,
 * `capacity` rows each, dst->capacity) are copied into p's receive map at
 * [rank][e_l][lo, hi). fsmoe_peer_flag_write then sets flag[slot][rank] to
 * `value` on every rank behind the stream's earlier work (stream memory
 * operation with a system-scope fence; `value` = how many times this rank
 * has signalled the slot, matching fsmoe_peer_wait's counting). */
int fsmoe_peer_copy_rows(const void* send, long long row_bytes, const fsmoe_peer_rows* dst, long long lo,
                         long long hi, int include_self, void* stream);
int fsmoe_peer_flag_write(const fsmoe_peer_flags* f, int slot, unsigned long long value, void* stream);
/* fsmoe_dispatch / fsmoe_combine_bwd writing their block buffer through a peer map. */
int fsmoe_dispatch_peer(int dtype, int model_dim, int experts, long long capacity,
                        const int* pick_of_slot, const int* pick_token, const void* x,
                        const fsmoe_peer_rows* dst, void* stream);
int fsmoe_combine_bwd_peer(int dtype, int model_dim, int experts, long long capacity,
                           long long n_picks, const int* pick_of_slot, const int* pick_token,
                           const double* pick_weight, const void* dy, const void* buffers,
                           const fsmoe_peer_rows* d_dst, double* d_weight, void* stream);

/* Row gather through the TMA engine: dst[i] = src[src_row[i]] for i < n_rows
 * (src_row[i] < 0: a zero row); dst through dst_map when non-null (rows land
 * in the owning rank's buffer), else the local buffer dst. With a top-1
 * softmax gate every kept weight is exactly 1.0, so combine_tokens
 * (workload.cpp:266-282) and its backward reduce to such gathers. */
int fsmoe_gather_rows(int dtype, int model_dim, long long n_rows, const int* src_row,
                      const void* src, void* dst, const fsmoe_peer_rows* dst_map, void* stream);

/* dst[i] = 0 for every i < n_rows with src_row[i] < 0 (other rows untouched):
 * the dropped tokens of a top-1 combine whose kept rows the GEMM epilogue
 * scattered (fsmoe_gemm_desc::scatter_rows). Row bytes a multiple of 16. */
int fsmoe_zero_rows(int dtype, int model_dim, long long n_rows, const int* src_row, void* dst,
                    void* stream);

/* The same over the slots [slot_lo, slot_hi) only (exclude = 0) or all but
 * them (exclude = 1): the EP layer moves its own experts' rows first and the
 * peers' rows on a second stream, overlapping the NVLink transfer with the
 * expert GEMMs on the local rows. The range form of combine backward leaves
 * d_weight of dropped picks alone (zero it before the first range call). */
int fsmoe_dispatch_peer_range(int dtype, int model_dim, int experts, long long capacity,
                              const int* pick_of_slot, const int* pick_token, const void* x,
                              const fsmoe_peer_rows* dst, long long slot_lo, long long slot_hi,
                              int exclude, void* stream);
int fsmoe_combine_bwd_peer_range(int dtype, int model_dim, int experts, long long capacity,
                                 long long n_picks, const int* pick_of_slot, const int* pick_token,
                                 const double* pick_weight, const void* dy, const void* buffers,
                                 const fsmoe_peer_rows* d_dst, double* d_weight, long long slot_lo,
                                 long long slot_hi, int exclude, void* stream);

typedef struct fsmoe_gemm_desc {
  int kind;        /* 0 row-grouped (fwd/dgrad), 1 k-grouped (wgrad) */
  int nblk, rows, K, N, Mo, No, n_w;
  int rows_total;  /* rows per block in memory (0 -> rows) */
  int row0;        /* first processed row of each block (pipeline chunk) */
  int b_mn_major;
  const void* A;
  const void* B;
  const long long* valid_rows; /* optional, per block */
  int epi;         /* 0 store bf16, 1 store f32, 2 gelu fwd, 3 swiglu fwd, 4 gelu bwd, 5 swiglu bwd,
                    * 6 add bf16 (row-grouped, tcgen05 only: D = bf16(acc + Zin), Zin may be D).
                    * bf16 gelu: fwd writes D = gelu'(Z) (what the backward
                    * needs, so it does no transcendental work) and D2 = gelu(Z);
                    * bwd writes D = acc * Zin with Zin that saved gelu'(Z). */
  void* D;
  void* D2;
  const void* Zin;
  long long ldd, ldd2, ldz;
  int accumulate;
  int precision;   /* 0 bf16/tcgen05, 1 fp32 check */
  /* row-grouped epi 0/1 only: store output rows through this peer map
   * ([nblk][rows_total] rows, capacity = rows_total) instead of D */
  const fsmoe_peer_rows* d_peers;
  /* row-grouped only: process blocks [blk_lo, blk_hi) (blk_exclude = 0) or
   * all but them (1); blk_hi = 0 means every block */
  int blk_lo, blk_hi, blk_exclude;
  /* > 0: run the persistent grid on at most this many SMs (leaves the rest to
   * a concurrent kernel, e.g. an NVLink row transfer); 0 = all */
  int max_sms;
  /* tile-variant overrides (tests / measurement; 0 = the heuristic):
   * force_ctas 1 | 2 (single CTA / tcgen05 cta_group::2 pair), force_bn 128 |
   * 256 | 512 columns; dbg: measurement-only epilogue ablations */
  int force_ctas, force_bn, dbg;
  /* tile-order override (0 = the heuristic): band_m > 0 walks bands of
   * band_m m-tiles column by column, band_n > 0 bands of band_n n-tiles row
   * by row, band_m < 0 plain m-major order */
  int band_m, band_n;
  /* row-grouped epi 0 (tcgen05) only: instead of D, output row r of
   * [nblk][rows_total] goes to row scatter_rows[r] of scatter_out (row stride
   * scatter_ld elements; < 0: dropped) -- a top-1 combine / its backward
   * fused into the GEMM epilogue */
  const int* scatter_rows;
  void* scatter_out;
  long long scatter_ld;
} fsmoe_gemm_desc;

int fsmoe_grouped_gemm(const fsmoe_gemm_desc* d, void* stream);

/* Elementwise activation kernels used by the fp32 check mode
 * (op: 2 gelu fwd, 3 swiglu fwd, 4 gelu bwd, 5 swiglu bwd; same layouts as
 * the fused tcgen05 epilogues), over rows [row0, row0+rows) of nblk blocks of
 * rows_total rows. */
int fsmoe_activation_f32(int op, int nblk, int rows_total, int row0, int rows, int units,
                         const float* in, const float* z, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
