/*
 * fsmoe_oracle.c — TEST INFRASTRUCTURE ONLY (see fsmoe_oracle.h).
 *
 * CPU restatement of the reference routing path, following
 * /root/reference/proj/src/workload.cpp line by line in its arithmetic:
 *   - sequential left-to-right fp64 sums, separate multiply and add (build
 *     with -ffp-contract=off so gcc never fuses them),
 *   - libstdc++ mt19937_64 + Box-Muller noise with glibc log/cos,
 *   - stable top-k (score desc, index asc) re-sorted ascending,
 *   - masked softmax with a running max and an ascending-index sum.
 */
#include "fsmoe_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng -- */

#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = MT_N;
}

static void mt_twist(orc_mt64* g) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t y = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
    g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
  }
  g->idx = 0;
}

uint64_t orc_mt64_next(orc_mt64* g) {
  if (g->idx >= MT_N) mt_twist(g);
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

void orc_uniform_fill(orc_mt64* g, long long n, double lo, double hi, double* out) {
  for (long long i = 0; i < n; ++i) {
    double u = (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53;
    out[i] = lo + (hi - lo) * u;
  }
}

/* workload.cpp:90-95 */
double orc_normal_next(orc_mt64* g) {
  double u1 = ((double)(orc_mt64_next(g) >> 11) + 0.5) * 0x1.0p-53;
  double u2 = ((double)(orc_mt64_next(g) >> 11) + 0.5) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793238462643383279502884 * u2);
}

/* The noise row of token t (workload.cpp:184-186): E draws of
 * NormalDraws(seed + t), in expert order. */
void orc_noise_row(uint64_t seed, int t, int E, double* out) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed + (uint64_t)t);
  for (int e = 0; e < E; ++e) out[e] = orc_normal_next(&g);
}

/* -------------------------------------------------------------- helpers -- */

static int fail(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) snprintf(err, (size_t)errlen, "%s", msg);
  return 2;
}

static int require_dims(int have_r, int have_c, int want_r, int want_c,
                        const char* name, char* err, int errlen) {
  if (have_r == want_r && have_c == want_c) return 0;
  char buf[160];
  snprintf(buf, sizeof buf, "gate: %s must be %dx%d", name, want_r, want_c);
  return fail(err, errlen, buf);
}

/* Ordering used by top_k (workload.cpp:111-121): score descending, then
 * index ascending. A total order for non-NaN scores, so qsort is stable. */
static const double* g_sort_scores;
static int by_score_desc(const void* a, const void* b) {
  int ia = *(const int*)a, ib = *(const int*)b;
  double sa = g_sort_scores[ia], sb = g_sort_scores[ib];
  if (sa != sb) return sa > sb ? -1 : 1;
  return ia < ib ? -1 : (ia > ib);
}
static int by_index(const void* a, const void* b) {
  int ia = *(const int*)a, ib = *(const int*)b;
  return ia < ib ? -1 : (ia > ib);
}

/* keep[] receives the k selected indices in ascending order. scratch holds n ints. */
static void top_k(const double* scores, int n, int k, int* keep, int* scratch) {
  for (int i = 0; i < n; ++i) scratch[i] = i;
  g_sort_scores = scores;
  qsort(scratch, (size_t)n, sizeof(int), by_score_desc);
  memcpy(keep, scratch, sizeof(int) * (size_t)k);
  qsort(keep, (size_t)k, sizeof(int), by_index);
}

/* workload.cpp:123-133 */
static void masked_softmax(const double* scores, const int* keep, int k, double* w) {
  double mx = scores[keep[0]];
  for (int j = 0; j < k; ++j) mx = (mx < scores[keep[j]]) ? scores[keep[j]] : mx;
  double z = 0.0;
  for (int j = 0; j < k; ++j) z += exp(scores[keep[j]] - mx);
  for (int j = 0; j < k; ++j) w[j] = exp(scores[keep[j]] - mx) / z;
}

/* workload.cpp:103-108: out[c] = ((0 + x0*w0c) + x1*w1c) + ... */
static void matvec_row(const double* xrow, int dim, const double* w, int cols, double* out) {
  for (int c = 0; c < cols; ++c) {
    double acc = 0.0;
    for (int j = 0; j < dim; ++j) acc += xrow[j] * w[(size_t)j * cols + c];
    out[c] = acc;
  }
}

/* ------------------------------------------------------------- capacity -- */

long long orc_capacity_tokens(int batch, int heads, int seq_len, int model_dim,
                              int hidden_scale, double capacity_factor,
                              int unlimited, int experts, int top_k_,
                              double t_olp_dense_ms, char* err, int errlen) {
  /* validate(LayerConfig), workload.cpp:10-26 */
  struct { int v; const char* n; } pos[] = {
      {batch, "batch"}, {heads, "heads"}, {seq_len, "seq_len"},
      {model_dim, "model_dim"}, {hidden_scale, "hidden_scale"},
      {experts, "experts"}, {top_k_, "top_k"}};
  for (size_t i = 0; i < sizeof pos / sizeof pos[0]; ++i) {
    if (pos[i].v <= 0) {
      char buf[96];
      snprintf(buf, sizeof buf, "layer: %s must be positive", pos[i].n);
      fail(err, errlen, buf);
      return -1;
    }
  }
  if (!unlimited && capacity_factor <= 0.0) {
    fail(err, errlen, "layer: capacity_factor must be positive");
    return -1;
  }
  if (t_olp_dense_ms < 0.0) {
    fail(err, errlen, "layer: t_olp_dense_ms must be nonnegative");
    return -1;
  }
  double tokens = (double)batch * seq_len;
  if (unlimited) return (long long)((double)top_k_ * tokens);
  double v = top_k_ * capacity_factor * tokens / experts;
  return (long long)ceil(v - 1e-9);
}

/* ----------------------------------------------------------------- gate -- */

int orc_run_gate(int kind, int k, uint64_t seed,
                 int T, int M, const double* x,
                 int ws_rows, int ws_cols, const double* w_score,
                 int wn_rows, int wn_cols, const double* w_noise,
                 int pj_rows, int pj_cols, const double* proj,
                 int* pick_token, int* pick_expert, double* pick_weight,
                 long long* n_picks, char* err, int errlen) {
  const int E = ws_cols;
  *n_picks = 0;
  if (T <= 0 || M <= 0) return fail(err, errlen, "gate: empty token matrix");
  if (E <= 0) return fail(err, errlen, "gate: no experts");
  if (k <= 0) return fail(err, errlen, "gate: top_k must be positive");

  long long np = 0;
  if (kind == ORC_EXPERT_CHOICE) {
    if (k > T) return fail(err, errlen, "gate: expert capacity exceeds token count");
    int rc = require_dims(ws_rows, ws_cols, M, E, "score_weights", err, errlen);
    if (rc) return rc;
    double* scores = (double*)malloc(sizeof(double) * (size_t)T);
    int* keep = (int*)malloc(sizeof(int) * (size_t)k);
    int* scratch = (int*)malloc(sizeof(int) * (size_t)T);
    double* w = (double*)malloc(sizeof(double) * (size_t)k);
    for (int e = 0; e < E; ++e) {
      for (int t = 0; t < T; ++t) {
        double acc = 0.0;
        for (int j = 0; j < M; ++j) acc += x[(size_t)t * M + j] * w_score[(size_t)j * E + e];
        scores[t] = acc;
      }
      top_k(scores, T, k, keep, scratch);
      masked_softmax(scores, keep, k, w);
      for (int j = 0; j < k; ++j, ++np) {
        pick_token[np] = keep[j];
        pick_expert[np] = e;
        pick_weight[np] = w[j];
      }
    }
    free(scores); free(keep); free(scratch); free(w);
    *n_picks = np;
    return 0;
  }

  if (k > E) return fail(err, errlen, "gate: top_k exceeds expert count");

  double* scores = (double*)malloc(sizeof(double) * (size_t)E);
  double* spread = (double*)malloc(sizeof(double) * (size_t)E);
  int* keep = (int*)malloc(sizeof(int) * (size_t)k);
  int* scratch = (int*)malloc(sizeof(int) * (size_t)E);
  double* w = (double*)malloc(sizeof(double) * (size_t)k);
  double* pr = (double*)malloc(sizeof(double) * (size_t)(pj_rows > 0 ? pj_rows : 1));
  int rc = 0;
  for (int t = 0; t < T && rc == 0; ++t) {
    const double* xr = x + (size_t)t * M;
    if (kind == ORC_NOISY_TOPK) {
      if ((rc = require_dims(ws_rows, ws_cols, M, E, "score_weights", err, errlen))) break;
      if ((rc = require_dims(wn_rows, wn_cols, M, E, "noise_weights", err, errlen))) break;
      matvec_row(xr, M, w_score, E, scores);
      matvec_row(xr, M, w_noise, E, spread);
      orc_mt64 g;
      orc_mt64_seed(&g, seed + (uint64_t)t);
      for (int e = 0; e < E; ++e) scores[e] += orc_normal_next(&g) * log1p(exp(spread[e]));
      top_k(scores, E, k, keep, scratch);
      masked_softmax(scores, keep, k, w);
      for (int j = 0; j < k; ++j, ++np) {
        pick_token[np] = t; pick_expert[np] = keep[j]; pick_weight[np] = w[j];
      }
    } else if (kind == ORC_SIGMOID_TOPK) {
      if ((rc = require_dims(ws_rows, ws_cols, M, E, "score_weights", err, errlen))) break;
      matvec_row(xr, M, w_score, E, scores);
      top_k(scores, E, k, keep, scratch);
      for (int j = 0; j < k; ++j, ++np) {
        pick_token[np] = t; pick_expert[np] = keep[j];
        pick_weight[np] = 1.0 / (1.0 + exp(-scores[keep[j]]));
      }
    } else if (kind == ORC_COSINE_TOPK) {
      const int P = pj_rows;
      if ((rc = require_dims(pj_rows, pj_cols, P, M, "projection", err, errlen))) break;
      if ((rc = require_dims(ws_rows, ws_cols, P, E, "score_weights", err, errlen))) break;
      for (int p = 0; p < P; ++p) {
        double acc = 0.0;
        for (int j = 0; j < M; ++j) acc += proj[(size_t)p * M + j] * xr[j];
        pr[p] = acc;
      }
      double pnorm = 0.0;
      for (int p = 0; p < P; ++p) pnorm += pr[p] * pr[p];
      if (pnorm == 0.0) { rc = fail(err, errlen, "gate: projected token has zero norm"); break; }
      for (int e = 0; e < E && rc == 0; ++e) {
        double dot = 0.0, enorm = 0.0;
        for (int p = 0; p < P; ++p) {
          double we = w_score[(size_t)p * E + e];
          dot += pr[p] * we;
          enorm += we * we;
        }
        if (enorm == 0.0) { rc = fail(err, errlen, "gate: expert embedding has zero norm"); break; }
        scores[e] = dot / sqrt(pnorm * enorm);
      }
      if (rc) break;
      top_k(scores, E, k, keep, scratch);
      masked_softmax(scores, keep, k, w);
      for (int j = 0; j < k; ++j, ++np) {
        pick_token[np] = t; pick_expert[np] = keep[j]; pick_weight[np] = w[j];
      }
    } else {
      rc = fail(err, errlen, "gate: unknown gate kind");
    }
  }
  free(scores); free(spread); free(keep); free(scratch); free(w); free(pr);
  if (rc) return rc;
  *n_picks = np;
  return 0;
}

/* ------------------------------------------------------ dispatch/combine -- */

int orc_dispatch(int T, int M, const double* x, int E, long long n_picks,
                 const int* pick_token, const int* pick_expert, long long C,
                 double* buffers, int* slot_of_pick, long long* fill,
                 long long* dropped, char* err, int errlen) {
  if (C <= 0) return fail(err, errlen, "dispatch: capacity must be positive");
  memset(buffers, 0, sizeof(double) * (size_t)E * (size_t)C * (size_t)M);
  for (int e = 0; e < E; ++e) fill[e] = 0;
  *dropped = 0;
  for (long long p = 0; p < n_picks; ++p) slot_of_pick[p] = -1;
  for (long long p = 0; p < n_picks; ++p) {
    int e = pick_expert[p], t = pick_token[p];
    if (e < 0 || e >= E || t < 0 || t >= T)
      return fail(err, errlen, "dispatch: pick references an unknown token or expert");
    if (fill[e] >= C) { ++*dropped; continue; }
    long long slot = (long long)e * C + fill[e];
    memcpy(buffers + (size_t)slot * M, x + (size_t)t * M, sizeof(double) * (size_t)M);
    slot_of_pick[p] = (int)slot;
    ++fill[e];
  }
  return 0;
}

int orc_combine(int buf_rows, int buf_cols, const double* buffers, int T,
                long long n_picks, const int* pick_token, const double* pick_weight,
                long long n_slots_of_pick, const int* slot_of_pick, int M,
                double* y, char* err, int errlen) {
  (void)buf_rows;
  if (buf_cols != M) return fail(err, errlen, "combine: buffer width does not match model_dim");
  if (n_slots_of_pick != n_picks) return fail(err, errlen, "combine: layout does not match the gate output");
  memset(y, 0, sizeof(double) * (size_t)T * (size_t)M);
  for (long long p = 0; p < n_picks; ++p) {
    int s = slot_of_pick[p];
    if (s < 0) continue;
    double w = pick_weight[p];
    double* yr = y + (size_t)pick_token[p] * M;
    const double* br = buffers + (size_t)s * M;
    for (int j = 0; j < M; ++j) yr[j] += w * br[j];
  }
  return 0;
}

/* FNV-1a 64 over n bytes (fingerprint helper for tests). */
uint64_t orc_fnv1a64(const unsigned char* p, long long n) {
  uint64_t h = 0xCBF29CE484222325ULL;
  for (long long i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ULL;
  }
  return h;
}
