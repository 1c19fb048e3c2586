// gate_prune.cu — K1 fast path for the linear-score gates (noisy_topk,
// sigmoid_topk): exact selection without computing every fp64 logit.
//
//  1. approx_scores_kernel: fp32 FMA scores s~ = x . W for all (token,
//     column) (W_g and, for noisy, W_noise), a SIMT tile GEMM.
//  2. prune_select_kernel (one warp per token):
//       * rigorous bound |s~ - s_ref| <= B = c * |x_t|_2 * |W_e|_2 with
//         c = (M+4) 2^-24 (1.01) + (M+2) 2^-53, covering fp32 rounding of x, W
//         and the FMA chain, and the reference's own fp64 sequential rounding
//         (s_ref = matvec_row of workload.cpp:103-108);
//       * noisy: s = raw + n * softplus(spread) with the exact per-token
//         mt19937_64 Box-Muller noise n (workload.cpp:85-99, 183-186);
//         softplus is 1-Lipschitz, so B_s = B_raw + |n| B_spread;
//       * candidates = experts whose upper bound reaches the k-th largest lower
//         bound — provably a superset of the exact top-k;
//       * exact fp64 logits (sequential j, no FMA) only for the candidates,
//         exact top-k among them with ties to the lowest index (111-121),
//         then the masked softmax (123-133) or logistic (198).
//     Outputs are identical to the exhaustive path (tests/test_routing_gpu.py
//     runs both against the reference's golden vectors).
//
// Compiled with --fmad=false (the exact logits must not contract; the
// approximate phase uses explicit fmaf).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "capi_common.h"
#include "kernels.h"
#include "route_common.cuh"

namespace fsmoe {
namespace {

using namespace fsmoe_dev;

constexpr int AP_TOK = 64;   // tokens per block
constexpr int AP_COL = 32;   // columns per block
constexpr int AP_JC = 32;    // reduction chunk

// W32[j][c] = (float)W_a[j][c] (c < Ea) | (float)W_b[j][c - Ea]; wn[c] = |column|_2.
__global__ void w_to_f32_kernel(int M, int Ea, const double* __restrict__ Wa, int Eb,
                                const double* __restrict__ Wb, float* __restrict__ W32,
                                double* __restrict__ wn) {
  const int NC = Ea + Eb;
  const int c = blockIdx.x;
  double ss = 0.0;
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    double v = c < Ea ? Wa[static_cast<long long>(j) * Ea + c] : Wb[static_cast<long long>(j) * Eb + (c - Ea)];
    W32[static_cast<long long>(j) * NC + c] = static_cast<float>(v);
    ss = __fma_rn(v, v, ss);
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int i = 0; i < static_cast<int>(blockDim.x) / 32; ++i) a += red[i];
    wn[c] = sqrt(a) * (1.0 + 1e-12);
  }
}

// out[t][c] = sum_j x[t][j] * W32[j][c]  (fp32 FMA); 64 tokens x 32 cols per
// block, 256 threads, each 2 tokens x 4 columns.
template <int DT>
__global__ void __launch_bounds__(256)
    approx_scores_kernel(const void* __restrict__ x, int T, int M, const float* __restrict__ W32,
                         int NC, float* __restrict__ out) {
  __shared__ float xs[AP_JC][AP_TOK + 1];
  __shared__ __align__(16) float ws[AP_JC][AP_COL];
  const int t0 = blockIdx.x * AP_TOK, c0 = blockIdx.y * AP_COL;
  const int ty = threadIdx.x / 8, tx = threadIdx.x % 8;  // 32 token pairs x 8 column quads
  float acc[2][4] = {};
  for (int j0 = 0; j0 < M; j0 += AP_JC) {
    __syncthreads();
    for (int i = threadIdx.x; i < AP_TOK * AP_JC; i += 256) {
      int tt = i / AP_JC, jj = i % AP_JC;
      int t = t0 + tt, j = j0 + jj;
      xs[jj][tt] = (t < T && j < M) ? static_cast<float>(load_as_double<DT>(x, static_cast<long long>(t) * M + j)) : 0.f;
    }
    for (int i = threadIdx.x; i < AP_JC * AP_COL; i += 256) {
      int jj = i / AP_COL, cc = i % AP_COL;
      int j = j0 + jj, c = c0 + cc;
      ws[jj][cc] = (j < M && c < NC) ? W32[static_cast<long long>(j) * NC + c] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int jj = 0; jj < AP_JC; ++jj) {
      const float a0 = xs[jj][2 * ty], a1 = xs[jj][2 * ty + 1];
      const float4 w = reinterpret_cast<const float4*>(ws[jj])[tx];
      acc[0][0] = fmaf(a0, w.x, acc[0][0]); acc[0][1] = fmaf(a0, w.y, acc[0][1]);
      acc[0][2] = fmaf(a0, w.z, acc[0][2]); acc[0][3] = fmaf(a0, w.w, acc[0][3]);
      acc[1][0] = fmaf(a1, w.x, acc[1][0]); acc[1][1] = fmaf(a1, w.y, acc[1][1]);
      acc[1][2] = fmaf(a1, w.z, acc[1][2]); acc[1][3] = fmaf(a1, w.w, acc[1][3]);
    }
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int t = t0 + 2 * ty + a;
    if (t >= T) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c = c0 + 4 * tx + b;
      if (c < NC) out[static_cast<long long>(t) * NC + c] = acc[a][b];
    }
  }
}

// ---------------------------------------------------------------- noise --

constexpr uint64_t MT_A = 0xB5026F5AA96619E9ULL;
constexpr uint64_t MT_UM = 0xFFFFFFFF80000000ULL;
constexpr uint64_t MT_LM = 0x000000007FFFFFFFULL;

__device__ __forceinline__ uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

// Normal draw of expert e for mt19937_64(seed): outputs 2e and 2e+1
// (requires 2e + 1 < 156: words 2e..2e+2 and 156+2e..157+2e of the seeding).
__device__ double noise_of(uint64_t seed, int e) {
  const int i0 = 2 * e;
  uint64_t w = seed, a = 0, b = 0, c = 0, d = 0, f = 0;
  if (i0 == 0) a = w;
  for (int i = 1; i <= 157 + i0; ++i) {
    w = 6364136223846793005ULL * (w ^ (w >> 62)) + static_cast<uint64_t>(i);
    if (i == i0) a = w;
    if (i == i0 + 1) b = w;
    if (i == i0 + 2) c = w;
    if (i == 156 + i0) d = w;
    if (i == 157 + i0) f = w;
  }
  uint64_t y0 = (a & MT_UM) | (b & MT_LM);
  uint64_t o0 = temper(d ^ (y0 >> 1) ^ ((y0 & 1ULL) ? MT_A : 0ULL));
  uint64_t y1 = (b & MT_UM) | (c & MT_LM);
  uint64_t o1 = temper(f ^ (y1 >> 1) ^ ((y1 & 1ULL) ? MT_A : 0ULL));
  double u1 = __dmul_rn(__dadd_rn(static_cast<double>(o0 >> 11), 0.5), 0x1.0p-53);
  double u2 = __dmul_rn(__dadd_rn(static_cast<double>(o1 >> 11), 0.5), 0x1.0p-53);
  double two_pi = 2.0 * 3.141592653589793238462643383279502884;
  return __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(two_pi, u2)));
}

// Sequential fp64 dot (matvec_row order, separately rounded mul/add).
template <int DT>
__device__ double exact_dot(const void* x, long long xrow, int M, const double* W, int ldw, int c) {
  double acc = 0.0;
#pragma unroll 8
  for (int j = 0; j < M; ++j)
    acc = __dadd_rn(acc, __dmul_rn(load_as_double<DT>(x, xrow + j), W[static_cast<long long>(j) * ldw + c]));
  return acc;
}

constexpr int PS_MAXE = 64;           // experts per token on this path
constexpr int PS_PER = PS_MAXE / 32;  // experts per lane

// KIND 0: noisy_topk, 1: sigmoid_topk. One warp per token.
template <int DT, int KIND>
__global__ void __launch_bounds__(256)
    prune_select_kernel(const void* __restrict__ x, int T, int M, int E, int k, uint64_t seed,
                        const float* __restrict__ approx, const double* __restrict__ wn,
                        double cB, const double* __restrict__ Wg, const double* __restrict__ Wn,
                        int* __restrict__ pick_token, int* __restrict__ pick_expert,
                        double* __restrict__ pick_weight, double* __restrict__ scores_out,
                        double* __restrict__ noise_out, double* __restrict__ spread_out) {
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const long long xrow = static_cast<long long>(t) * M;
  const int NC = KIND == 0 ? 2 * E : E;

  // |x_t|_2 (upper bound)
  double ss = 0.0;
  for (int j = lane; j < M; j += 32) {
    double v = load_as_double<DT>(x, xrow + j);
    ss = __fma_rn(v, v, ss);
  }
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const double xnorm = sqrt(ss) * (1.0 + 1e-12);

  // approximate scores and bounds for this lane's experts
  double sa[PS_PER], bnd[PS_PER], nz[PS_PER], spa[PS_PER];
#pragma unroll
  for (int i = 0; i < PS_PER; ++i) {
    const int e = lane + 32 * i;
    sa[i] = -1e300;
    bnd[i] = 0.0;
    nz[i] = 0.0;
    spa[i] = 0.0;
    if (e >= E) continue;
    const double r = approx[static_cast<long long>(t) * NC + e];
    const double br = cB * xnorm * wn[e];
    if (KIND == 0) {
      nz[i] = noise_of(seed + static_cast<uint64_t>(t), e);
      spa[i] = approx[static_cast<long long>(t) * NC + E + e];
      const double bs = cB * xnorm * wn[E + e];
      const double sp = log1p(exp(spa[i]));
      sa[i] = r + nz[i] * sp;
      bnd[i] = br + fabs(nz[i]) * bs + 1e-12 * (fabs(r) + fabs(nz[i] * sp) + 1e-200);
    } else {
      sa[i] = r;
      bnd[i] = br + 1e-12 * (fabs(r) + 1e-200);
    }
  }

  // k-th largest lower bound (ties irrelevant: only its value is used)
  uint64_t taken = 0;
  double kth = -1e300;
  for (int j = 0; j < k; ++j) {
    double best = -1e300;
    int bi = -1;
#pragma unroll
    for (int i = 0; i < PS_PER; ++i) {
      const int e = lane + 32 * i;
      if (e < E && !((taken >> e) & 1ULL) && (bi < 0 || sa[i] - bnd[i] > best)) {
        best = sa[i] - bnd[i];
        bi = e;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oi >= 0 && (bi < 0 || ob > best || (ob == best && oi < bi))) {
        best = ob;
        bi = oi;
      }
    }
    taken |= 1ULL << bi;
    kth = best;
  }

  // exact logits for candidates
  double sx[PS_PER];
  uint64_t cand = 0;
#pragma unroll
  for (int i = 0; i < PS_PER; ++i) {
    const int e = lane + 32 * i;
    sx[i] = sa[i];
    if (e >= E || sa[i] + bnd[i] < kth) continue;
    cand |= 1ULL << e;
    const double raw = exact_dot<DT>(x, xrow, M, Wg, E, e);
    if (KIND == 0) {
      const double spread = exact_dot<DT>(x, xrow, M, Wn, E, e);
      spa[i] = spread;
      sx[i] = __dadd_rn(raw, __dmul_rn(nz[i], log1p(exp(spread))));
    } else {
      sx[i] = raw;
    }
  }
  for (int o = 16; o > 0; o >>= 1) cand |= __shfl_xor_sync(0xffffffffu, cand, o);

  // exact top-k among candidates: max score, ties to the lowest index
  uint64_t kept = 0;
  for (int j = 0; j < k; ++j) {
    double best = 0.0;
    int bi = -1;
#pragma unroll
    for (int i = 0; i < PS_PER; ++i) {
      const int e = lane + 32 * i;
      if (e < E && ((cand >> e) & 1ULL) && !((kept >> e) & 1ULL) && (bi < 0 || sx[i] > best)) {
        best = sx[i];
        bi = e;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oi >= 0 && (bi < 0 || ob > best || (ob == best && oi < bi))) {
        best = ob;
        bi = oi;
      }
    }
    kept |= 1ULL << bi;
  }

  // saved tensors for the backward (exact where it matters, finite elsewhere)
#pragma unroll
  for (int i = 0; i < PS_PER; ++i) {
    const int e = lane + 32 * i;
    if (e >= E) continue;
    const long long o = static_cast<long long>(t) * E + e;
    if (scores_out) scores_out[o] = sx[i];
    if (KIND == 0) {
      if (noise_out) noise_out[o] = nz[i];
      if (spread_out) spread_out[o] = spa[i];
    }
  }

  // weights over the kept set in ascending expert order (lane 0)
  auto score_of = [&](int e) {
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < PS_PER; ++i) {
      double s = __shfl_sync(0xffffffffu, sx[i], e & 31);
      if ((e >> 5) == i) v = s;
    }
    return v;
  };
  const long long base = static_cast<long long>(t) * k;
  if (KIND == 1) {
    uint64_t m = kept;
    for (int j = 0; j < k; ++j) {
      const int e = __ffsll(static_cast<long long>(m)) - 1;
      m &= m - 1;
      const double s = score_of(e);
      if (lane == 0) {
        pick_token[base + j] = t;
        pick_expert[base + j] = e;
        pick_weight[base + j] = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-s)));
      }
    }
    return;
  }
  double ks[PS_MAXE];
  int ke[PS_MAXE];
  {
    uint64_t m = kept;
    for (int j = 0; j < k; ++j) {
      const int e = __ffsll(static_cast<long long>(m)) - 1;
      m &= m - 1;
      ke[j] = e;
      ks[j] = score_of(e);
    }
  }
  if (lane == 0) {
    double mx = ks[0];
    for (int j = 0; j < k; ++j) mx = (mx < ks[j]) ? ks[j] : mx;
    double z = 0.0;
    for (int j = 0; j < k; ++j) z = __dadd_rn(z, exp(__dsub_rn(ks[j], mx)));
    for (int j = 0; j < k; ++j) {
      pick_token[base + j] = t;
      pick_expert[base + j] = ke[j];
      pick_weight[base + j] = __ddiv_rn(exp(__dsub_rn(ks[j], mx)), z);
    }
  }
}

}  // namespace

size_t gate_prune_workspace_bytes(const fsmoe_gate_desc& d) {
  const size_t T = d.tokens, E = d.score_cols, M = d.model_dim;
  const size_t NC = d.kind == FSMOE_GATE_NOISY_TOPK ? 2 * E : E;
  auto r = [](size_t b) { return (b + 255) & ~size_t(255); };
  return r(4 * M * NC) + r(8 * NC) + r(4 * T * NC);
}

bool gate_prune_applicable(const fsmoe_gate_desc& d) {
  if (d.kind != FSMOE_GATE_NOISY_TOPK && d.kind != FSMOE_GATE_SIGMOID_TOPK) return false;
  if (d.score_cols > PS_MAXE || d.top_k > PS_MAXE) return false;
  return true;
}

int gate_prune_launch(const fsmoe_gate_desc& d, const void* x, const double* w_score,
                      const double* w_noise, int* pick_token, int* pick_expert,
                      double* pick_weight, double* scores_out, double* noise_out,
                      double* spread_out, void* ws, cudaStream_t st) {
  const int T = d.tokens, M = d.model_dim, E = d.score_cols, k = d.top_k;
  const bool noisy = d.kind == FSMOE_GATE_NOISY_TOPK;
  const int NC = noisy ? 2 * E : E;
  char* w = static_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* p = w;
    w += (bytes + 255) & ~size_t(255);
    return p;
  };
  float* W32 = reinterpret_cast<float*>(take(4ull * M * NC));
  double* wn = reinterpret_cast<double*>(take(8ull * NC));
  float* approx = reinterpret_cast<float*>(take(4ull * T * NC));
  w_to_f32_kernel<<<NC, 256, 0, st>>>(M, E, w_score, noisy ? E : 0, w_noise, W32, wn);
  ::fsmoe::count_launch();
  dim3 grid((T + AP_TOK - 1) / AP_TOK, (NC + AP_COL - 1) / AP_COL);
  switch (d.x_dtype) {
    case FSMOE_F64: approx_scores_kernel<0><<<grid, 256, 0, st>>>(x, T, M, W32, NC, approx); break;
    case FSMOE_F32: approx_scores_kernel<1><<<grid, 256, 0, st>>>(x, T, M, W32, NC, approx); break;
    default: approx_scores_kernel<2><<<grid, 256, 0, st>>>(x, T, M, W32, NC, approx); break;
  }
  ::fsmoe::count_launch();
  // |s~ - s_ref| <= cB |x| |w|: fp32 rounding of x, w and the M-term FMA chain
  // (+ slack), plus the reference's own fp64 sequential rounding.
  const double cB = (M + 4.0) * 0x1.0p-24 * 1.01 + (M + 2.0) * 0x1.0p-53;
  const int blocks = (T + 7) / 8;
#define FSMOE_PS(DT, KIND)                                                                        \
  prune_select_kernel<DT, KIND><<<blocks, 256, 0, st>>>(x, T, M, E, k, d.seed, approx, wn, cB,     \
                                                        w_score, w_noise, pick_token, pick_expert, \
                                                        pick_weight, scores_out, noise_out,        \
                                                        spread_out)
  if (noisy) {
    switch (d.x_dtype) {
      case FSMOE_F64: FSMOE_PS(0, 0); break;
      case FSMOE_F32: FSMOE_PS(1, 0); break;
      default: FSMOE_PS(2, 0); break;
    }
  } else {
    switch (d.x_dtype) {
      case FSMOE_F64: FSMOE_PS(0, 1); break;
      case FSMOE_F32: FSMOE_PS(1, 1); break;
      default: FSMOE_PS(2, 1); break;
    }
  }
#undef FSMOE_PS
  ::fsmoe::count_launch();
  return cuda_status(cudaGetLastError(), "fsmoe_gate(prune)");
}

}  // namespace fsmoe
