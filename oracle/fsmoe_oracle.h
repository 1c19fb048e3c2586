/*
 * fsmoe_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's routing numerics (the FSMoE artifact,
 * /root/reference/proj/src/workload.cpp). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library,
 * and only as the checker / CPU baseline. The product path (libfsmoe_cuda.so,
 * libfsmoe.so) never links or calls it.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks this restatement
 * against golden vectors produced by the reference itself compiled from
 * /root/reference (oracle/Makefile -> oracle/_ref/libfsmoe_ref.so,
 * generator oracle/gen_golden.py) and against the reference test-suite KATs
 * (proj/tests/test_workload.cpp, proj/tests/acceptance.cpp:459-610).
 *
 * Error convention mirrors fsmoe::ConfigError (common.hpp:16-18): functions
 * return 0 on success or 2 (exit_config_error) and copy the reference's
 * exception message into `err`.
 */
#ifndef FSMOE_ORACLE_H
#define FSMOE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_NOISY_TOPK = 0, ORC_SIGMOID_TOPK = 1, ORC_COSINE_TOPK = 2, ORC_EXPERT_CHOICE = 3 };

/* libstdc++ std::mt19937_64 restated (used by NormalDraws, workload.cpp:85-99). */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);

/* lo + (hi-lo) * ((next() >> 11) * 2^-53) for n draws (test_util.hpp:92-96). */
void orc_uniform_fill(orc_mt64* g, long long n, double lo, double hi, double* out);

/* Box-Muller normal draw, workload.cpp:90-95. */
double orc_normal_next(orc_mt64* g);

/* E normal draws of NormalDraws(seed + t) (workload.cpp:184-186). */
void orc_noise_row(uint64_t seed, int t, int E, double* out);

/* capacity_tokens, workload.cpp:43-51. Returns -1 and fills err on ConfigError. */
long long orc_capacity_tokens(int batch, int heads, int seq_len, int model_dim,
                              int hidden_scale, double capacity_factor,
                              int unlimited, int experts, int top_k,
                              double t_olp_dense_ms, char* err, int errlen);

/* run_gate, workload.cpp:143-235. Matrices are row-major doubles with the
 * given shapes (the shapes reproduce require_dims errors). Picks are written
 * token-major (token-choice) or expert-major (expert_choice); *n_picks gets
 * the count. Output arrays must hold max(T*k, E*k) entries. */
int orc_run_gate(int kind, int top_k, uint64_t seed,
                 int tokens, int dim, const double* x,
                 int ws_rows, int ws_cols, const double* w_score,
                 int wn_rows, int wn_cols, const double* w_noise,
                 int pj_rows, int pj_cols, const double* proj,
                 int* pick_token, int* pick_expert, double* pick_weight,
                 long long* n_picks, char* err, int errlen);

/* dispatch_tokens, workload.cpp:237-264. buffers must hold experts*capacity*dim
 * doubles (zero-filled here). */
int orc_dispatch(int tokens, int dim, const double* x, int experts,
                 long long n_picks, const int* pick_token, const int* pick_expert,
                 long long capacity, double* buffers, int* slot_of_pick,
                 long long* fill, long long* dropped, char* err, int errlen);

/* combine_tokens, workload.cpp:266-282. y must hold tokens*model_dim. */
int orc_combine(int buf_rows, int buf_cols, const double* buffers, int tokens,
                long long n_picks, const int* pick_token, const double* pick_weight,
                long long n_slots_of_pick, const int* slot_of_pick, int model_dim,
                double* y, char* err, int errlen);

/* FNV-1a 64 over n bytes (test fingerprints). */
uint64_t orc_fnv1a64(const unsigned char* p, long long n);

#ifdef __cplusplus
}
#endif
#endif
