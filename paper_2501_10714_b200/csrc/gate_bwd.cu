// gate_bwd.cu — backward of the gate (the reference has none, SPEC.md:12;
// semantics of SURVEY.md Appendix D):
//   d_weight -> d scores:  softmax over the kept set (noisy / cosine / EC),
//                          logistic (sigmoid); dropped picks have d_weight 0 but
//                          still couple through the softmax normaliser.
//   d scores -> params:    dW = x^T dS (deterministic split-T reduction, fp64
//                          across splits), dx += dS W^T; noisy adds the
//                          softplus(x W_noise)*n branch; cosine goes through
//                          q = P x and the norms. For bf16 tokens the noisy /
//                          sigmoid contractions run on the tcgen05 GEMM (see
//                          "tensor-core forms" below), else SIMT FMA kernels.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "capi_common.h"
#include "gemm.h"
#include "host_once.h"
#include "kernels.h"
#include "route_common.cuh"

namespace fsmoe {
namespace {

using namespace fsmoe_dev;

// dS for token-choice gates (T x E, dense, zero elsewhere).
// kind 0/2: softmax over the k kept picks; kind 1: sigmoid.
__global__ void dscore_token_kernel(int kind, int T, int E, int k, const int* __restrict__ pexp,
                                    const double* __restrict__ pw, const double* __restrict__ dw,
                                    double* __restrict__ dS) {
  fsmoe_dev::pdl_enter();
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  double* row = dS + static_cast<long long>(t) * E;
  for (int e = 0; e < E; ++e) row[e] = 0.0;
  const long long b = static_cast<long long>(t) * k;
  if (kind == 1) {
    for (int j = 0; j < k; ++j) {
      double w = pw[b + j];
      row[pexp[b + j]] = dw[b + j] * w * (1.0 - w);
    }
    return;
  }
  double sig = 0.0;
  for (int j = 0; j < k; ++j) sig += pw[b + j] * dw[b + j];
  for (int j = 0; j < k; ++j) row[pexp[b + j]] = pw[b + j] * (dw[b + j] - sig);
}

// dS for expert choice, layout E x T (like the forward scores).
__global__ void dscore_ec_kernel(int T, int E, int C, const int* __restrict__ ptok,
                                 const double* __restrict__ pw, const double* __restrict__ dw,
                                 double* __restrict__ dS) {
  __shared__ double red[32];
  const int e = blockIdx.x;
  const long long b = static_cast<long long>(e) * C;
  double part = 0.0;
  for (int j = threadIdx.x; j < C; j += blockDim.x) part += pw[b + j] * dw[b + j];
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  double sig = 0.0;
  for (int i = 0; i < static_cast<int>(blockDim.x) / 32; ++i) sig += red[i];
  double* row = dS + static_cast<long long>(e) * T;
  for (int t = threadIdx.x; t < T; t += blockDim.x) row[t] = 0.0;
  __syncthreads();
  for (int j = threadIdx.x; j < C; j += blockDim.x) row[ptok[b + j]] = pw[b + j] * (dw[b + j] - sig);
}

// noisy: dZ = dS * n * sigmoid(spread)
__global__ void noisy_dz_kernel(long long n, const double* __restrict__ dS,
                                const double* __restrict__ noise, const double* __restrict__ spread,
                                double* __restrict__ dZ) {
  fsmoe_dev::pdl_enter();
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i < n) dZ[i] = dS[i] * noise[i] / (1.0 + exp(-spread[i]));
}

// cosine: dq[t][p] = sum_e dS[t][e] (w_pe/(|q||w_e|) - s_e q_p/|q|^2);
// qn[t] = q/|q|. One thread per (token, p) -- the same operations in the same
// order as a per-token loop, with T x P threads to spread the fp64 divisions.
__global__ void cosine_dq_kernel(int T, int E, int P, const double* __restrict__ q,
                                 const double* __restrict__ w, const double* __restrict__ enorm,
                                 const double* __restrict__ s, const double* __restrict__ dS,
                                 double* __restrict__ dq, double* __restrict__ qn) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(T) * P) return;
  const int t = static_cast<int>(i / P), p = static_cast<int>(i % P);
  const double* qt = q + static_cast<long long>(t) * P;
  double pn = 0.0;
  for (int pp = 0; pp < P; ++pp) pn += qt[pp] * qt[pp];
  const double qnorm = sqrt(pn);
  qn[i] = qt[p] / qnorm;
  double d = 0.0;
  for (int e = 0; e < E; ++e) {
    const double g = dS[static_cast<long long>(t) * E + e];
    if (g == 0.0) continue;
    const double wn = sqrt(enorm[e]);
    const double se = s[static_cast<long long>(t) * E + e];
    d += g * (w[static_cast<long long>(p) * E + e] / (qnorm * wn) - se * qt[p] / pn);
  }
  dq[i] = d;
}

// b[e] = sum_t dS[t][e] * s[t][e]
__global__ void cosine_b_kernel(int T, int E, const double* __restrict__ s,
                                const double* __restrict__ dS, double* __restrict__ b) {
  __shared__ double red[32];
  const int e = blockIdx.x;
  double part = 0.0;
  for (int t = threadIdx.x; t < T; t += blockDim.x)
    part += dS[static_cast<long long>(t) * E + e] * s[static_cast<long long>(t) * E + e];
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int i = 0; i < static_cast<int>(blockDim.x) / 32; ++i) acc += red[i];
    b[e] = acc;
  }
}

// dW[p][e] += A[p][e]/|w_e| - w[p][e] b[e]/|w_e|^2
__global__ void cosine_dw_kernel(int P, int E, const double* __restrict__ A,
                                 const double* __restrict__ w, const double* __restrict__ enorm,
                                 const double* __restrict__ b, double* __restrict__ dW) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P * E) return;
  int e = i % E;
  double wn = sqrt(enorm[e]);
  dW[i] += A[i] / wn - w[i] * b[e] / enorm[e];
}

constexpr int XT_TCH = 256;  // tokens per partial (at most; fewer when that leaves SMs idle)

// Tokens per partial chunk: 256, or fewer (a multiple of 32, at least 32) so
// that chunks x column blocks gives the GPU two blocks per SM (small T, or a
// narrow M such as the cosine projection's P rows).
inline int xt_tch(int T, long long colblocks) {
  const long long want = 2LL * device_sms();
  const long long nch = (want + colblocks - 1) / colblocks;
  long long tch = (T + nch - 1) / nch;
  tch = (tch + 31) / 32 * 32;
  return static_cast<int>(tch < 32 ? 32 : tch > XT_TCH ? XT_TCH : tch);
}
inline long long xt_chunks(int T, long long colblocks) {
  const int tch = xt_tch(T, colblocks);
  return (T + tch - 1) / tch;
}
constexpr int XT_J = 64;
constexpr int XT_C = 16;

// partial[chunk][j][c] = sum_{t in chunk} X(t, j) * G(t, c).
// A = the arithmetic type: fp64 for fp64 tokens; fp32 for bf16 / fp32 tokens
// (exact in fp32) -- the gate gradient has no reference counterpart (the
// reference has no backward), B200's fp64 pipe is a small fraction of its
// fp32 rate, and 256-token fp32 partials summed in fp64 keep the relative
// error near 1e-6, far inside the layer's gradient tolerances.
template <int DT, typename A>
__global__ void __launch_bounds__(XT_J * XT_C)
    xtg_partial_kernel(int T, int M, int NC, const void* __restrict__ X,
                       const double* __restrict__ G, long long gst, long long gsc,
                       double* __restrict__ part, int tch) {
  __shared__ A xs[32][XT_J];
  __shared__ A gs[32][XT_C];
  const int chunk = blockIdx.z;
  const int j0 = blockIdx.x * XT_J, c0 = blockIdx.y * XT_C;
  const int jj = threadIdx.x % XT_J, cc = threadIdx.x / XT_J;
  A acc = A(0);
  const int t_end = min(T, (chunk + 1) * tch);
  for (int t0 = chunk * tch; t0 < t_end; t0 += 32) {
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * XT_J; i += XT_J * XT_C) {
      int tt = i / XT_J, j = i % XT_J;
      int t = t0 + tt;
      xs[tt][j] = (t < t_end && j0 + j < M) ? static_cast<A>(load_as_double<DT>(X, static_cast<long long>(t) * M + j0 + j)) : A(0);
    }
    for (int i = threadIdx.x; i < 32 * XT_C; i += XT_J * XT_C) {
      int tt = i / XT_C, c = i % XT_C;
      int t = t0 + tt;
      gs[tt][c] = (t < t_end && c0 + c < NC) ? static_cast<A>(G[t * gst + (c0 + c) * gsc]) : A(0);
    }
    __syncthreads();
#pragma unroll 8
    for (int tt = 0; tt < 32; ++tt) acc += xs[tt][jj] * gs[tt][cc];
  }
  if (j0 + jj < M && c0 + cc < NC)
    part[(static_cast<long long>(chunk) * M + j0 + jj) * NC + c0 + cc] = static_cast<double>(acc);
}

// out[j*osj + c*osc] (+)= sum_chunk partial[chunk][j][c]  (fixed order)
__global__ void xtg_reduce_kernel(int nchunks, int M, int NC, const double* __restrict__ part,
                                  double* __restrict__ out, long long osj, long long osc,
                                  int accumulate) {
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(M) * NC) return;
  int j = static_cast<int>(i / NC), c = static_cast<int>(i % NC);
  double a = 0.0;
  for (int k = 0; k < nchunks; ++k) a += part[static_cast<long long>(k) * M * NC + i];
  double* o = out + j * osj + c * osc;
  *o = accumulate ? *o + a : a;
}

// dx[t][j] += sum_c G(t,c) * W(j,c)   (arithmetic type A as above)
template <typename T, typename A>
__global__ void __launch_bounds__(256)
    dx_acc_kernel(int Tn, int M, int NC, const double* __restrict__ G, long long gst,
                  long long gsc, const double* __restrict__ W, long long wsj, long long wsc,
                  T* __restrict__ dx) {
  const int j = blockIdx.x * 256 + threadIdx.x;
  const int t0 = blockIdx.y * 32;
  __shared__ A gs[32][64];
  for (int c0 = 0; c0 < NC; c0 += 64) {
    const int nc = min(64, NC - c0);
    A wr[64];
    if (j < M)
      for (int c = 0; c < nc; ++c) wr[c] = static_cast<A>(W[j * wsj + (c0 + c) * wsc]);
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 64; i += 256) {
      int tt = i / 64, c = i % 64;
      gs[tt][c] = (t0 + tt < Tn && c < nc) ? static_cast<A>(G[(t0 + tt) * gst + (c0 + c) * gsc]) : A(0);
    }
    __syncthreads();
    if (j < M) {
      for (int tt = 0; tt < 32 && t0 + tt < Tn; ++tt) {
        A a = A(0);
        for (int c = 0; c < nc; ++c) a += gs[tt][c] * wr[c];
        T* p = dx + static_cast<long long>(t0 + tt) * M + j;
        if constexpr (sizeof(T) == 2) *p = __float2bfloat16(__bfloat162float(*p) + static_cast<float>(a));
        else *p = static_cast<T>(static_cast<double>(*p) + static_cast<double>(a));
      }
    }
  }
}

// Register-tiled replacements (the gate gradient contractions are skinny:
// NC = E or P columns): thread = one model column j, all NC accumulators in
// registers (NCT = NC rounded up), the chunk's G rows broadcast from shared
// memory, x read coalesced along j. Same fixed per-chunk order, so results
// stay deterministic.
template <int DT, typename A, int NCT>
__global__ void __launch_bounds__(256)
    xtg2_kernel(int T, int M, int NC, const void* __restrict__ X, const double* __restrict__ G,
                long long gst, long long gsc, double* __restrict__ part, int tch) {
  __shared__ __align__(16) A gs[32][NCT];
  const int chunk = blockIdx.y;
  const int j = blockIdx.x * 256 + threadIdx.x;
  A acc[NCT];
#pragma unroll
  for (int c = 0; c < NCT; ++c) acc[c] = A(0);
  const int t_end = min(T, (chunk + 1) * tch);
  for (int t0 = chunk * tch; t0 < t_end; t0 += 32) {
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * NCT; i += 256) {
      const int tt = i / NCT, c = i % NCT;
      const int t = t0 + tt;
      gs[tt][c] = (t < t_end && c < NC) ? static_cast<A>(G[t * gst + c * gsc]) : A(0);
    }
    __syncthreads();
    if (j < M) {
      const int nt = min(32, t_end - t0);
      for (int u0 = 0; u0 < nt; u0 += 8) {  // eight tokens' x loads in flight
        A xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          xv[u] = u0 + u < nt ? static_cast<A>(load_as_double<DT>(X, static_cast<long long>(t0 + u0 + u) * M + j))
                              : A(0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (u0 + u >= nt) break;
#pragma unroll
          for (int c = 0; c < NCT; ++c) acc[c] += xv[u] * gs[u0 + u][c];
        }
      }
    }
  }
  if (j < M)
#pragma unroll
    for (int c = 0; c < NCT; ++c)
      if (c < NC) part[(static_cast<long long>(chunk) * M + j) * NC + c] = static_cast<double>(acc[c]);
}

// dx[t][j] += sum_c G1(t,c) W1(j,c) [+ sum_c G2(t,c) W2(j,c)]: one pass over
// dx for both projections of the noisy gate
template <typename T, typename A, int NCT>
__global__ void __launch_bounds__(256)
    dx_acc2_kernel(int Tn, int M, int NC, const double* __restrict__ G1, const double* __restrict__ W1,
                   const double* __restrict__ G2, const double* __restrict__ W2, long long gst,
                   long long gsc, long long wsj, long long wsc, T* __restrict__ dx) {
  __shared__ __align__(16) A gs[2][32][NCT];
  const int j = blockIdx.x * 256 + threadIdx.x;
  const int t0 = blockIdx.y * 32;
  const int npj = G2 ? 2 : 1;
  A w1[NCT], w2[NCT];
#pragma unroll
  for (int c = 0; c < NCT; ++c) {
    w1[c] = (j < M && c < NC) ? static_cast<A>(W1[j * wsj + c * wsc]) : A(0);
    w2[c] = (j < M && c < NC && G2) ? static_cast<A>(W2[j * wsj + c * wsc]) : A(0);
  }
  for (int i = threadIdx.x; i < npj * 32 * NCT; i += 256) {
    const int pj = i / (32 * NCT), tt = (i / NCT) % 32, c = i % NCT;
    const double* G = pj ? G2 : G1;
    gs[pj][tt][c] = (t0 + tt < Tn && c < NC) ? static_cast<A>(G[(t0 + tt) * gst + c * gsc]) : A(0);
  }
  __syncthreads();
  if (j >= M) return;
  const int nt = min(32, Tn - t0);
  for (int u0 = 0; u0 < nt; u0 += 8) {  // eight tokens' dx loads in flight
    T dv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) dv[u] = u0 + u < nt ? dx[static_cast<long long>(t0 + u0 + u) * M + j] : T(0);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (u0 + u >= nt) break;
      const int tt = u0 + u;
      A a = A(0);
#pragma unroll
      for (int c = 0; c < NCT; ++c) a += gs[0][tt][c] * w1[c];
      if (G2)
#pragma unroll
        for (int c = 0; c < NCT; ++c) a += gs[1][tt][c] * w2[c];
      T* p = dx + static_cast<long long>(t0 + tt) * M + j;
      if constexpr (sizeof(T) == 2) *p = __float2bfloat16(__bfloat162float(dv[u]) + static_cast<float>(a));
      else *p = static_cast<T>(static_cast<double>(dv[u]) + static_cast<double>(a));
    }
  }
}

// Paired-column forms of xtg2 / dx_acc2 for fp32-arithmetic tokens (bf16 /
// fp32 x) with M even: a thread owns columns (j, j+1), so x moves as one
// 4- or 8-byte load per token and the chunk's G rows are read back from
// shared memory as float4 broadcasts; the noisy gate's two projections share
// one pass over x (columns [0, NC) from G1, [NC, 2 NC) from G2). Every output
// element is accumulated in the same order as in the single-column kernels.
template <typename XT>
__device__ __forceinline__ float2 load_pair(const XT* p);
template <>
__device__ __forceinline__ float2 load_pair<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
}
template <>
__device__ __forceinline__ float2 load_pair<float>(const float* p) {
  return *reinterpret_cast<const float2*>(p);
}

template <typename XT, int NCT2>
__global__ void __launch_bounds__(256)
    xtg_pair_kernel(int T, int M, int NC, const XT* __restrict__ X, const double* __restrict__ G1,
                    const double* __restrict__ G2, long long gst, long long gsc,
                    double* __restrict__ part, int tch) {
  __shared__ __align__(16) float gs[32][NCT2];
  const int NC2 = G2 ? 2 * NC : NC;
  const int chunk = blockIdx.y;
  const int j = (blockIdx.x * 256 + threadIdx.x) * 2;
  float a0[NCT2], a1[NCT2];
#pragma unroll
  for (int c = 0; c < NCT2; ++c) a0[c] = a1[c] = 0.f;
  const int t_end = min(T, (chunk + 1) * tch);
  for (int t0 = chunk * tch; t0 < t_end; t0 += 32) {
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * NCT2; i += 256) {
      const int tt = i / NCT2, c = i % NCT2;
      const int t = t0 + tt;
      float v = 0.f;
      if (t < t_end && c < NC2)
        v = static_cast<float>(c < NC ? G1[t * gst + c * gsc] : G2[t * gst + (c - NC) * gsc]);
      gs[tt][c] = v;
    }
    __syncthreads();
    if (j < M) {
      const int nt = min(32, t_end - t0);
      // eight tokens' x loads in flight before their FMAs
      for (int u0 = 0; u0 < nt; u0 += 8) {
        float2 xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          xv[u] = u0 + u < nt ? load_pair<XT>(X + static_cast<long long>(t0 + u0 + u) * M + j)
                              : make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (u0 + u >= nt) break;
          const float4* g4 = reinterpret_cast<const float4*>(gs[u0 + u]);
#pragma unroll
          for (int q = 0; q < NCT2 / 4; ++q) {
            const float4 g = g4[q];
            a0[4 * q] += xv[u].x * g.x;
            a0[4 * q + 1] += xv[u].x * g.y;
            a0[4 * q + 2] += xv[u].x * g.z;
            a0[4 * q + 3] += xv[u].x * g.w;
            a1[4 * q] += xv[u].y * g.x;
            a1[4 * q + 1] += xv[u].y * g.y;
            a1[4 * q + 2] += xv[u].y * g.z;
            a1[4 * q + 3] += xv[u].y * g.w;
          }
        }
      }
    }
  }
  if (j < M) {
    double* o = part + (static_cast<long long>(chunk) * M + j) * NC2;
#pragma unroll
    for (int c = 0; c < NCT2; ++c)
      if (c < NC2) {
        o[c] = static_cast<double>(a0[c]);
        o[NC2 + c] = static_cast<double>(a1[c]);
      }
  }
}

// out1 / out2 (+)= sum_chunk part[chunk][j][c] (fixed order) for the two
// column groups of xtg_pair_kernel
__global__ void xtg_reduce_pair_kernel(int nchunks, int M, int NC, int NC2,
                                       const double* __restrict__ part, double* __restrict__ out1,
                                       double* __restrict__ out2, long long osj, long long osc,
                                       int accumulate) {
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(M) * NC2) return;
  const int j = static_cast<int>(i / NC2), c2 = static_cast<int>(i % NC2);
  double a = 0.0;
  for (int k = 0; k < nchunks; ++k) a += part[static_cast<long long>(k) * M * NC2 + i];
  double* o = c2 < NC ? out1 + j * osj + c2 * osc : out2 + j * osj + (c2 - NC) * osc;
  *o = accumulate ? *o + a : a;
}

constexpr int DXP_TOK = 128;  // tokens per block of dx_pair_kernel

template <typename XT, int NCT>
__global__ void __launch_bounds__(256)
    dx_pair_kernel(int Tn, int M, int NC, const double* __restrict__ G1, const double* __restrict__ W1,
                   const double* __restrict__ G2, const double* __restrict__ W2, long long gst,
                   long long gsc, long long wsj, long long wsc, XT* __restrict__ dx) {
  __shared__ __align__(16) float gs[2][DXP_TOK][NCT];
  const int j = (blockIdx.x * 256 + threadIdx.x) * 2;
  const int t0 = blockIdx.y * DXP_TOK;
  const int npj = G2 ? 2 : 1;
  float w1a[NCT], w1b[NCT], w2a[NCT], w2b[NCT];
#pragma unroll
  for (int c = 0; c < NCT; ++c) {
    const bool ok = j < M && c < NC;
    w1a[c] = ok ? static_cast<float>(W1[j * wsj + c * wsc]) : 0.f;
    w1b[c] = ok ? static_cast<float>(W1[(j + 1) * wsj + c * wsc]) : 0.f;
    w2a[c] = ok && G2 ? static_cast<float>(W2[j * wsj + c * wsc]) : 0.f;
    w2b[c] = ok && G2 ? static_cast<float>(W2[(j + 1) * wsj + c * wsc]) : 0.f;
  }
  for (int i = threadIdx.x; i < npj * DXP_TOK * NCT; i += 256) {
    const int pj = i / (DXP_TOK * NCT), tt = (i / NCT) % DXP_TOK, c = i % NCT;
    const double* G = pj ? G2 : G1;
    gs[pj][tt][c] = (t0 + tt < Tn && c < NC) ? static_cast<float>(G[(t0 + tt) * gst + c * gsc]) : 0.f;
  }
  __syncthreads();
  if (j >= M) return;
  const int nt = min(DXP_TOK, Tn - t0);
  for (int u0 = 0; u0 < nt; u0 += 8) {
  // eight tokens' dx loads in flight before their updates
  float2 dv[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const XT* q = dx + static_cast<long long>(t0 + u0 + u) * M + j;
    if (u0 + u < nt) {
      if constexpr (sizeof(XT) == 2) dv[u] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(q));
      else dv[u] = *reinterpret_cast<const float2*>(q);
    } else {
      dv[u] = make_float2(0.f, 0.f);
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    if (u0 + u >= nt) break;
    const int tt = u0 + u;
    float s0 = 0.f, s1 = 0.f;
    const float4* g1 = reinterpret_cast<const float4*>(gs[0][tt]);
#pragma unroll
    for (int q = 0; q < NCT / 4; ++q) {
      const float4 g = g1[q];
      s0 += g.x * w1a[4 * q]; s0 += g.y * w1a[4 * q + 1]; s0 += g.z * w1a[4 * q + 2]; s0 += g.w * w1a[4 * q + 3];
      s1 += g.x * w1b[4 * q]; s1 += g.y * w1b[4 * q + 1]; s1 += g.z * w1b[4 * q + 2]; s1 += g.w * w1b[4 * q + 3];
    }
    if (G2) {
      const float4* g2 = reinterpret_cast<const float4*>(gs[1][tt]);
#pragma unroll
      for (int q = 0; q < NCT / 4; ++q) {
        const float4 g = g2[q];
        s0 += g.x * w2a[4 * q]; s0 += g.y * w2a[4 * q + 1]; s0 += g.z * w2a[4 * q + 2]; s0 += g.w * w2a[4 * q + 3];
        s1 += g.x * w2b[4 * q]; s1 += g.y * w2b[4 * q + 1]; s1 += g.z * w2b[4 * q + 2]; s1 += g.w * w2b[4 * q + 3];
      }
    }
    XT* p = dx + static_cast<long long>(t0 + tt) * M + j;
    const float2 d = dv[u];
    if constexpr (sizeof(XT) == 2) {
      *reinterpret_cast<__nv_bfloat162*>(p) = __halves2bfloat162(__float2bfloat16(d.x + s0), __float2bfloat16(d.y + s1));
    } else {
      *reinterpret_cast<float2*>(p) = make_float2(static_cast<float>(static_cast<double>(d.x) + static_cast<double>(s0)),
                                                  static_cast<float>(static_cast<double>(d.y) + static_cast<double>(s1)));
    }
  }
  }
}

struct Ws {
  char* p;
  double* take(size_t n) {
    double* r = reinterpret_cast<double*>(p);
    p += (n * sizeof(double) + 255) & ~size_t(255);
    return r;
  }
};

template <int NCT>
void xtg2_launch(int xdt, int T, int M, int NC, const void* X, const double* G, long long gst,
                 long long gsc, double* part, cudaStream_t st) {
  const int tch = xt_tch(T, (M + 255) / 256);
  dim3 grid((M + 255) / 256, (T + tch - 1) / tch);
  switch (xdt) {
    case FSMOE_F64: xtg2_kernel<0, double, NCT><<<grid, 256, 0, st>>>(T, M, NC, X, G, gst, gsc, part, tch); break;
    case FSMOE_F32: xtg2_kernel<1, float, NCT><<<grid, 256, 0, st>>>(T, M, NC, X, G, gst, gsc, part, tch); break;
    default: xtg2_kernel<2, float, NCT><<<grid, 256, 0, st>>>(T, M, NC, X, G, gst, gsc, part, tch); break;
  }
  ::fsmoe::count_launch();
}

// x^T [G1 | G2] in one pass (fp32-arithmetic tokens, M even, 2 NC <= 32);
// false when the shape needs the general kernels
bool xtg_pair(int xdt, int T, int M, int NC, const void* X, const double* G1, const double* G2,
              long long gst, long long gsc, double* out1, double* out2, long long osj, long long osc,
              int accumulate, double* part, cudaStream_t st) {
  const int NC2 = G2 ? 2 * NC : NC;
  if (xdt == FSMOE_F64 || M % 2 || NC2 > 32) return false;
  const int tch = xt_tch(T, (M / 2 + 255) / 256);
  const int nchunks = (T + tch - 1) / tch;
  dim3 grid((M / 2 + 255) / 256, nchunks);
  auto go = [&](auto nct) {
    constexpr int N = decltype(nct)::value;
    if (xdt == FSMOE_F32)
      xtg_pair_kernel<float, N><<<grid, 256, 0, st>>>(T, M, NC, static_cast<const float*>(X), G1, G2, gst, gsc, part, tch);
    else
      xtg_pair_kernel<__nv_bfloat16, N><<<grid, 256, 0, st>>>(T, M, NC, static_cast<const __nv_bfloat16*>(X), G1,
                                                                G2, gst, gsc, part, tch);
    ::fsmoe::count_launch();
  };
  if (NC2 <= 8) go(std::integral_constant<int, 8>{});
  else if (NC2 <= 16) go(std::integral_constant<int, 16>{});
  else go(std::integral_constant<int, 32>{});
  const long long n = static_cast<long long>(M) * NC2;
  xtg_reduce_pair_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, st>>>(nchunks, M, NC, NC2, part, out1,
                                                                            G2 ? out2 : out1, osj, osc, accumulate);
  ::fsmoe::count_launch();
  return true;
}

void xtg(int xdt, int T, int M, int NC, const void* X, const double* G, long long gst,
         long long gsc, double* out, long long osj, long long osc, int accumulate, double* part,
         cudaStream_t st) {
  if (NC <= 64) {
    const int nchunks = static_cast<int>(xt_chunks(T, (M + 255) / 256));
    if (NC <= 8) xtg2_launch<8>(xdt, T, M, NC, X, G, gst, gsc, part, st);
    else if (NC <= 16) xtg2_launch<16>(xdt, T, M, NC, X, G, gst, gsc, part, st);
    else if (NC <= 32) xtg2_launch<32>(xdt, T, M, NC, X, G, gst, gsc, part, st);
    else xtg2_launch<64>(xdt, T, M, NC, X, G, gst, gsc, part, st);
    long long n = static_cast<long long>(M) * NC;
    xtg_reduce_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, st>>>(nchunks, M, NC, part, out,
                                                                         osj, osc, accumulate);
    ::fsmoe::count_launch();
    return;
  }
  const long long cb = static_cast<long long>((M + XT_J - 1) / XT_J) * ((NC + XT_C - 1) / XT_C);
  const int tch = xt_tch(T, cb);
  const int nchunks = (T + tch - 1) / tch;
  dim3 grid((M + XT_J - 1) / XT_J, (NC + XT_C - 1) / XT_C, nchunks);
  switch (xdt) {
    case FSMOE_F64: xtg_partial_kernel<0, double><<<grid, XT_J * XT_C, 0, st>>>(T, M, NC, X, G, gst, gsc, part, tch); ::fsmoe::count_launch(); break;
    case FSMOE_F32: xtg_partial_kernel<1, float><<<grid, XT_J * XT_C, 0, st>>>(T, M, NC, X, G, gst, gsc, part, tch); ::fsmoe::count_launch(); break;
    default: xtg_partial_kernel<2, float><<<grid, XT_J * XT_C, 0, st>>>(T, M, NC, X, G, gst, gsc, part, tch); ::fsmoe::count_launch(); break;
  }
  long long n = static_cast<long long>(M) * NC;
  xtg_reduce_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, st>>>(nchunks, M, NC, part, out,
                                                                       osj, osc, accumulate); ::fsmoe::count_launch();
}

template <int NCT>
void dx_acc2_launch(int xdt, int T, int M, int NC, const double* G1, const double* W1,
                    const double* G2, const double* W2, long long gst, long long gsc, long long wsj,
                    long long wsc, void* dx, cudaStream_t st) {
  dim3 grid((M + 255) / 256, (T + 31) / 32);
  switch (xdt) {
    case FSMOE_F64: dx_acc2_kernel<double, double, NCT><<<grid, 256, 0, st>>>(T, M, NC, G1, W1, G2, W2, gst, gsc, wsj, wsc, static_cast<double*>(dx)); break;
    case FSMOE_F32: dx_acc2_kernel<float, float, NCT><<<grid, 256, 0, st>>>(T, M, NC, G1, W1, G2, W2, gst, gsc, wsj, wsc, static_cast<float*>(dx)); break;
    default: dx_acc2_kernel<__nv_bfloat16, float, NCT><<<grid, 256, 0, st>>>(T, M, NC, G1, W1, G2, W2, gst, gsc, wsj, wsc, static_cast<__nv_bfloat16*>(dx)); break;
  }
  ::fsmoe::count_launch();
}

// both projections at once when G2 != null (same strides)
bool dx_acc_pair(int xdt, int T, int M, int NC, const double* G1, const double* W1,
                 const double* G2, const double* W2, long long gst, long long gsc, long long wsj,
                 long long wsc, void* dx, cudaStream_t st) {
  if (NC > 64) return false;
  if (xdt != FSMOE_F64 && M % 2 == 0 && NC <= 16) {
    dim3 grid((M / 2 + 255) / 256, (T + DXP_TOK - 1) / DXP_TOK);
    auto go = [&](auto nct) {
      constexpr int N = decltype(nct)::value;
      if (xdt == FSMOE_F32)
        dx_pair_kernel<float, N><<<grid, 256, 0, st>>>(T, M, NC, G1, W1, G2, W2, gst, gsc, wsj, wsc,
                                                       static_cast<float*>(dx));
      else
        dx_pair_kernel<__nv_bfloat16, N><<<grid, 256, 0, st>>>(T, M, NC, G1, W1, G2, W2, gst, gsc, wsj,
                                                               wsc, static_cast<__nv_bfloat16*>(dx));
      ::fsmoe::count_launch();
    };
    if (NC <= 8) go(std::integral_constant<int, 8>{});
    else go(std::integral_constant<int, 16>{});
    return true;
  }
  if (NC <= 8) dx_acc2_launch<8>(xdt, T, M, NC, G1, W1, G2, W2, gst, gsc, wsj, wsc, dx, st);
  else if (NC <= 16) dx_acc2_launch<16>(xdt, T, M, NC, G1, W1, G2, W2, gst, gsc, wsj, wsc, dx, st);
  else if (NC <= 32) dx_acc2_launch<32>(xdt, T, M, NC, G1, W1, G2, W2, gst, gsc, wsj, wsc, dx, st);
  else dx_acc2_launch<64>(xdt, T, M, NC, G1, W1, G2, W2, gst, gsc, wsj, wsc, dx, st);
  return true;
}

void dx_acc(int xdt, int T, int M, int NC, const double* G, long long gst, long long gsc,
            const double* W, long long wsj, long long wsc, void* dx, cudaStream_t st) {
  if (dx_acc_pair(xdt, T, M, NC, G, W, nullptr, nullptr, gst, gsc, wsj, wsc, dx, st)) return;
  dim3 grid((M + 255) / 256, (T + 31) / 32);
  switch (xdt) {
    case FSMOE_F64: dx_acc_kernel<double, double><<<grid, 256, 0, st>>>(T, M, NC, G, gst, gsc, W, wsj, wsc, static_cast<double*>(dx)); ::fsmoe::count_launch(); break;
    case FSMOE_F32: dx_acc_kernel<float, float><<<grid, 256, 0, st>>>(T, M, NC, G, gst, gsc, W, wsj, wsc, static_cast<float*>(dx)); ::fsmoe::count_launch(); break;
    default: dx_acc_kernel<__nv_bfloat16, float><<<grid, 256, 0, st>>>(T, M, NC, G, gst, gsc, W, wsj, wsc, static_cast<__nv_bfloat16*>(dx)); ::fsmoe::count_launch(); break;
  }
}

// ------------------------------------------------ tensor-core forms --
// For bf16 tokens the two contractions of a noisy / sigmoid gate backward
// run on the tcgen05 grouped GEMM (they were fp32 SIMT FMA bound: 2 T M NC2
// flops each, ~0.2 of HBM at the configs[2] shape):
//   x^T [G1 | G2]: a k-grouped GEMM of x against G split into three bf16
//     terms (hi, mid, lo: ~24 significant bits, fp32 accumulation, exact
//     products) over S token blocks -> fp32 partials, then a fixed-order fp64
//     sum of blocks and terms;
//   dx += [G1 | G2] [W1 | W2]^T: a row-grouped GEMM of K = 3 NC2 (G_hi W_hi +
//     G_hi W_lo + G_lo W_hi, ~16 bits) with the AddBF16 epilogue adding into
//     dx in place (bf16(dx + acc), the rounding of the SIMT form).
constexpr int TC_KMAX = 128;  // 3 * NC2 rounded up to 64 columns

__device__ __forceinline__ double gval(int c, int NC, long long t, const double* G1, const double* G2,
                                       long long gst, long long gsc) {
  return c < NC ? G1[t * gst + c * gsc] : G2[t * gst + (c - NC) * gsc];
}

// Gx[t][No] = [hi | mid | lo | 0] of G's NC2 columns; Gd[t][Kp] = [hi | hi | lo' | 0]
// (lo' = bf16(g - hi), the two-term split)
__global__ void g_split_kernel(int T, int NC, int NC2, int No, int Kp, const double* __restrict__ G1,
                               const double* __restrict__ G2, long long gst, long long gsc,
                               __nv_bfloat16* __restrict__ Gx, __nv_bfloat16* __restrict__ Gd) {
  fsmoe_dev::pdl_enter();
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const int W = No > Kp ? No : Kp;
  if (i >= static_cast<long long>(T) * W) return;
  const long long t = i / W;
  const int col = static_cast<int>(i % W);
  const int c = col % NC2, term = col / NC2;
  double g = 0.0;
  if (term < 3) g = gval(c, NC, t, G1, G2, gst, gsc);
  const __nv_bfloat16 hi = __double2bfloat16(g);
  const double r1 = g - static_cast<double>(__bfloat162float(hi));
  const __nv_bfloat16 mid = __double2bfloat16(r1);
  const __nv_bfloat16 lo = __double2bfloat16(r1 - static_cast<double>(__bfloat162float(mid)));
  const __nv_bfloat16 z = __float2bfloat16(0.f);
  if (col < No) Gx[t * No + col] = term == 0 ? hi : term == 1 ? mid : term == 2 ? lo : z;
  if (col < Kp) Gd[t * Kp + col] = term == 0 || term == 1 ? hi : term == 2 ? mid : z;
}

// Wd[j][Kp] = [W_hi | W_lo | W_hi | 0] over the NC2 columns of [W1 | W2]
__global__ void w_split_kernel(int M, int NC, int NC2, int Kp, const double* __restrict__ W1,
                               const double* __restrict__ W2, long long wsj, long long wsc,
                               __nv_bfloat16* __restrict__ Wd) {
  fsmoe_dev::pdl_enter();
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(M) * Kp) return;
  const long long j = i / Kp;
  const int col = static_cast<int>(i % Kp);
  const int c = col % NC2, term = col / NC2;
  double w = 0.0;
  if (term < 3) w = c < NC ? W1[j * wsj + c * wsc] : W2[j * wsj + (c - NC) * wsc];
  const __nv_bfloat16 hi = __double2bfloat16(w);
  const __nv_bfloat16 lo = __double2bfloat16(w - static_cast<double>(__bfloat162float(hi)));
  Wd[i] = term == 0 || term == 2 ? hi : term == 1 ? lo : __float2bfloat16(0.f);
}

// out1 / out2 [j][c] (+)= sum_s (P[s][j][c] + P[s][j][NC2 + c] + P[s][j][2 NC2 + c]), fixed order
__global__ void xtg_tc_reduce_kernel(int S, int M, int NC, int NC2, int No, const float* __restrict__ P,
                                     double* __restrict__ out1, double* __restrict__ out2, long long osj,
                                     long long osc, int accumulate) {
  fsmoe_dev::pdl_enter();
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(M) * NC2) return;
  const int j = static_cast<int>(i / NC2), c = static_cast<int>(i % NC2);
  double a = 0.0;
  for (int s = 0; s < S; ++s) {
    const float* r = P + (static_cast<long long>(s) * M + j) * No;
    a += static_cast<double>(r[c]);
    a += static_cast<double>(r[NC2 + c]);
    a += static_cast<double>(r[2 * NC2 + c]);
  }
  double* o = c < NC ? out1 + j * osj + c * osc : out2 + j * osj + (c - NC) * osc;
  *o = accumulate ? *o + a : a;
}

struct TcShape {
  int NC2, No, Kp, S;
};
// the tensor-core forms apply: bf16 tokens, 64-aligned model dim, <= 42 columns
bool tc_shape(int xdt, int T, int M, int NC2, TcShape* sh) {
  if (xdt != FSMOE_BF16 || M % 64 || NC2 <= 0 || 3 * NC2 > TC_KMAX || T < 64) return false;
  sh->NC2 = NC2;
  sh->No = sh->Kp = (3 * NC2 + 63) / 64 * 64;
  // token blocks of the x^T G GEMM: about two pair tiles per SM, T divisible
  const int mt = (M + 255) / 256;
  int S = (device_sms() + mt - 1) / mt;
  if (S > 64) S = 64;
  while (S > 1 && (T % S || T / S < 64)) --S;
  sh->S = S;
  return true;
}
size_t tc_ws_elems(int T, int M, int NC2max) {  // in doubles (8-byte units)
  TcShape sh{};
  if (!tc_shape(FSMOE_BF16, T, M, NC2max, &sh)) return 0;
  const size_t b = static_cast<size_t>(T) * sh.No * 2 + static_cast<size_t>(T) * sh.Kp * 2 +
                   static_cast<size_t>(M) * sh.Kp * 2 + static_cast<size_t>(sh.S) * M * sh.No * 4;
  return (b + 7) / 8 + 128;
}

// x^T [G1 | G2] and dx += [G1 | G2] [W1 | W2]^T on the tensor cores.
// Returns -1 when the shape needs the SIMT kernels (nothing was written),
// else a status. tw: workspace of tc_ws_elems.
int gate_bwd_tc(int xdt, int T, int M, int NC, const void* X, const double* G1, const double* G2,
                 long long gst, long long gsc, double* out1, double* out2, long long osj, long long osc,
                 const double* W1, const double* W2, long long wsj, long long wsc, void* dx, double* tw,
                 cudaStream_t st) {
  const int NC2 = G2 ? 2 * NC : NC;
  TcShape sh{};
  if (!tw || !tc_shape(xdt, T, M, NC2, &sh)) return -1;
  char* p = reinterpret_cast<char*>(tw);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  auto* Gx = reinterpret_cast<__nv_bfloat16*>(take(static_cast<size_t>(T) * sh.No * 2));
  auto* Gd = reinterpret_cast<__nv_bfloat16*>(take(static_cast<size_t>(T) * sh.Kp * 2));
  auto* Wd = reinterpret_cast<__nv_bfloat16*>(take(static_cast<size_t>(M) * sh.Kp * 2));
  auto* P = reinterpret_cast<float*>(take(static_cast<size_t>(sh.S) * M * sh.No * 4));
  const long long ng = static_cast<long long>(T) * (sh.No > sh.Kp ? sh.No : sh.Kp);
  pdl_launch(g_split_kernel, static_cast<int>((ng + 255) / 256), 256, 0, st, T, NC, NC2, sh.No, sh.Kp, G1, G2 ? G2 : G1,
                                                                     gst, gsc, Gx, Gd);
  ::fsmoe::count_launch();
  const long long nw = static_cast<long long>(M) * sh.Kp;
  pdl_launch(w_split_kernel, static_cast<int>((nw + 255) / 256), 256, 0, st, M, NC, NC2, sh.Kp, W1, W2 ? W2 : W1, wsj,
                                                                     wsc, Wd);
  ::fsmoe::count_launch();
  // x^T G: S blocks of T/S tokens, each its own output block (n_w = S)
  GemmProblem g{};
  g.kind = GemmKind::KGrouped;
  g.nblk = sh.S;
  g.n_w = sh.S;
  g.rows = g.rows_total = T / sh.S;
  g.Mo = M;
  g.No = sh.No;
  g.A = X;
  g.B = Gx;
  g.epi = Epi::StoreF32;
  g.D = P;
  g.ldd = sh.No;
  g.force_ctas = 2;
  g.force_bn = 128;
  int rc = gemm_sm100_launch(g, st);
  if (rc != cudaSuccess) return cuda_status(static_cast<cudaError_t>(rc), "gate backward x^T G (tcgen05)");
  const long long nr = static_cast<long long>(M) * NC2;
  pdl_launch(xtg_tc_reduce_kernel, static_cast<int>((nr + 255) / 256), 256, 0, st, sh.S, M, NC, NC2, sh.No, P, out1,
                                                                           out2 ? out2 : out1, osj, osc, 1);
  ::fsmoe::count_launch();
  // dx += Gd . Wd^T, in place through the AddBF16 epilogue
  GemmProblem h{};
  h.kind = GemmKind::RowGrouped;
  h.nblk = 1;
  h.n_w = 1;
  h.rows = h.rows_total = T;
  h.K = sh.Kp;
  h.N = M;
  h.A = Gd;
  h.B = Wd;
  h.epi = Epi::AddBF16;
  h.D = dx;
  h.ldd = M;
  h.Zin = dx;
  h.ldz = M;
  rc = gemm_sm100_launch(h, st);
  if (rc != cudaSuccess) return cuda_status(static_cast<cudaError_t>(rc), "gate backward dx (tcgen05)");
  return FSMOE_OK;
}

}  // namespace

// Partial-sum elements the largest x^T G of a gate backward needs: every
// (rows, columns) contraction it may run (rows M or P; columns E, 2E paired,
// or P) with the chunking its kernel would pick.
size_t xt_part_elems(int T, int M, int E, int P) {
  size_t best = 1;
  auto consider = [&](int rows, int nc2) {
    if (rows <= 0 || nc2 <= 0) return;
    const long long cbs[3] = {(rows / 2 + 255) / 256, (rows + 255) / 256,
                              static_cast<long long>((rows + XT_J - 1) / XT_J) * ((nc2 + XT_C - 1) / XT_C)};
    for (long long cb : cbs) {
      const size_t n = static_cast<size_t>(xt_chunks(T, cb < 1 ? 1 : cb)) * rows * nc2;
      if (n > best) best = n;
    }
  };
  consider(M, 2 * E);
  consider(M, P);
  consider(P, E);
  return best;
}

size_t gate_bwd_workspace_bytes(const fsmoe_gate_desc& d) {
  const size_t T = d.tokens, E = d.score_cols, M = d.model_dim, P = d.proj_rows > 0 ? d.proj_rows : 0;
  auto r = [](size_t n) { return (n * 8 + 255) & ~size_t(255); };
  const size_t tcw = d.x_dtype == FSMOE_BF16 ? tc_ws_elems(static_cast<int>(T), static_cast<int>(M),
                                                            static_cast<int>(2 * E)) : 0;
  return r(T * E) * 2 + r(T * P) * 2 + r(xt_part_elems(static_cast<int>(T), static_cast<int>(M),
                                                        static_cast<int>(E), static_cast<int>(P))) +
         r(P * E) + r(E) * 2 + r(tcw) + 1024;
}

int gate_bwd_launch(const fsmoe_gate_desc& d, const void* x, const double* w_score,
                    const double* w_noise, const double* proj, const int* ptok, const int* pexp,
                    const double* pw, const double* dw, const double* scores, const double* noise,
                    const double* spread, const double* proj_out, void* dx, double* dWs,
                    double* dWn, double* dP, void* ws, cudaStream_t st) {
  const int T = d.tokens, M = d.model_dim, E = d.score_cols, k = d.top_k;
  // A softmax over a single survivor is the constant 1 (workload.cpp:123-133
  // with one kept index): dS = w*(dw - w*dw) = 0 exactly, so every gate
  // gradient contribution vanishes (Switch-style top-1).
  const bool softmax_gate = d.kind == FSMOE_GATE_NOISY_TOPK || d.kind == FSMOE_GATE_COSINE_TOPK ||
                            d.kind == FSMOE_GATE_EXPERT_CHOICE;
  if (softmax_gate && k == 1) return FSMOE_OK;
  Ws w{static_cast<char*>(ws)};
  double* dS = w.take(static_cast<size_t>(T) * E);
  const int P = d.proj_rows > 0 ? d.proj_rows : 0;
  double* part = w.take(xt_part_elems(T, M, E, P));
  const size_t tcw = d.x_dtype == FSMOE_BF16 ? tc_ws_elems(T, M, 2 * E) : 0;
  double* tw = tcw ? w.take(tcw) : nullptr;
  switch (d.kind) {
    case FSMOE_GATE_NOISY_TOPK: {
      pdl_launch(dscore_token_kernel, (T + per_token_block(T) - 1) / per_token_block(T), per_token_block(T), 0, st, 0, T, E, k, pexp, pw, dw, dS); ::fsmoe::count_launch();
      double* dZ = w.take(static_cast<size_t>(T) * E);
      long long n = static_cast<long long>(T) * E;
      pdl_launch(noisy_dz_kernel, static_cast<int>((n + 255) / 256), 256, 0, st, n, dS, noise, spread, dZ); ::fsmoe::count_launch();
      const int tc = gate_bwd_tc(d.x_dtype, T, M, E, x, dS, dZ, E, 1, dWs, dWn, E, 1, w_score, w_noise, E, 1,
                                 dx, tw, st);
      if (tc >= 0) {
        if (tc != FSMOE_OK) return tc;
        break;
      }
      if (!xtg_pair(d.x_dtype, T, M, E, x, dS, dZ, E, 1, dWs, dWn, E, 1, 1, part, st)) {
        xtg(d.x_dtype, T, M, E, x, dS, E, 1, dWs, E, 1, 1, part, st);
        xtg(d.x_dtype, T, M, E, x, dZ, E, 1, dWn, E, 1, 1, part, st);
      }
      if (!dx_acc_pair(d.x_dtype, T, M, E, dS, w_score, dZ, w_noise, E, 1, E, 1, dx, st)) {
        dx_acc(d.x_dtype, T, M, E, dS, E, 1, w_score, E, 1, dx, st);
        dx_acc(d.x_dtype, T, M, E, dZ, E, 1, w_noise, E, 1, dx, st);
      }
      break;
    }
    case FSMOE_GATE_SIGMOID_TOPK: {
      pdl_launch(dscore_token_kernel, (T + per_token_block(T) - 1) / per_token_block(T), per_token_block(T), 0, st, 1, T, E, k, pexp, pw, dw, dS); ::fsmoe::count_launch();
      const int tc = gate_bwd_tc(d.x_dtype, T, M, E, x, dS, nullptr, E, 1, dWs, nullptr, E, 1, w_score, nullptr,
                                 E, 1, dx, tw, st);
      if (tc >= 0) {
        if (tc != FSMOE_OK) return tc;
        break;
      }
      if (!xtg_pair(d.x_dtype, T, M, E, x, dS, nullptr, E, 1, dWs, nullptr, E, 1, 1, part, st))
        xtg(d.x_dtype, T, M, E, x, dS, E, 1, dWs, E, 1, 1, part, st);
      dx_acc(d.x_dtype, T, M, E, dS, E, 1, w_score, E, 1, dx, st);
      break;
    }
    case FSMOE_GATE_EXPERT_CHOICE: {
      dscore_ec_kernel<<<E, 256, 0, st>>>(T, E, k, ptok, pw, dw, dS); ::fsmoe::count_launch();  // E x T
      xtg(d.x_dtype, T, M, E, x, dS, 1, T, dWs, E, 1, 1, part, st);
      dx_acc(d.x_dtype, T, M, E, dS, 1, T, w_score, E, 1, dx, st);
      break;
    }
    case FSMOE_GATE_COSINE_TOPK: {
      pdl_launch(dscore_token_kernel, (T + per_token_block(T) - 1) / per_token_block(T), per_token_block(T), 0, st, 0, T, E, k, pexp, pw, dw, dS); ::fsmoe::count_launch();
      double* dq = w.take(static_cast<size_t>(T) * P);
      double* qn = w.take(static_cast<size_t>(T) * P);
      double* en = w.take(E);
      double* bb = w.take(E);
      double* A = w.take(static_cast<size_t>(P) * E);
      // enorm recomputed (cheap) with the forward's arithmetic
      cosine_enorm(P, E, w_score, en, st);
      cosine_dq_kernel<<<static_cast<int>((static_cast<long long>(T) * P + 255) / 256), 256, 0, st>>>(
          T, E, P, proj_out, w_score, en, scores, dS, dq, qn); ::fsmoe::count_launch();
      cosine_b_kernel<<<E, 256, 0, st>>>(T, E, scores, dS, bb); ::fsmoe::count_launch();
      xtg(FSMOE_F64, T, P, E, qn, dS, E, 1, A, E, 1, 0, part, st);
      cosine_dw_kernel<<<(P * E + 255) / 256, 256, 0, st>>>(P, E, A, w_score, en, bb, dWs); ::fsmoe::count_launch();
      // dProj[p][j] += sum_t dq[t][p] x[t][j]
      xtg(d.x_dtype, T, M, P, x, dq, P, 1, dP, 1, M, 1, part, st);
      // dx += dq . Proj  (W(j,p) = Proj[p*M + j])
      dx_acc(d.x_dtype, T, M, P, dq, P, 1, proj, 1, M, dx, st);
      break;
    }
    default:
      return config_error("gate: unknown gate kind");
  }
  return cuda_status(cudaGetLastError(), "fsmoe_gate_bwd");
}

}  // namespace fsmoe
