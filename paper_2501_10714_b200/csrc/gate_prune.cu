// gate_prune.cu — K1 fast path for the linear-score gates (noisy_topk,
// sigmoid_topk): exact selection without computing every fp64 logit.
//
//  1. w_prep_kernel       W in fp32 [M][NC] (approximate phase), W^T in fp64
//                         [NC][M] (exact phase), column norms.
//  2. approx_scores_kernel  s~ = x . W for all (token, column), fp32 FMA
//                         SIMT tiles split over K, plus |x_t|^2 in fp64.
//  3. mt_kernel (thread per token): the first 2E outputs of
//     mt19937_64(seed + t) (workload.cpp:85-99, 184).
//  4. bound_kernel (thread per token x expert): Box-Muller noise, s~ and the
//     rigorous bound |s~ - s_ref| <= B = c |x_t|_2 |W_e|_2 with
//     c = (M+8+4) 2^-24 (1.01) + (M+2) 2^-53, covering fp32 rounding of x, W,
//     the FMA chain and split partial sums, and the reference's own fp64
//     sequential rounding (matvec_row, 103-108); for noisy, softplus is
//     1-Lipschitz: B_s = B_raw + |n| B_spread.
//  5. cand_kernel (thread per token): candidates = experts whose upper bound
//     reaches the k-th largest lower bound — a provable superset of the exact
//     top-k — appended to per-expert lists.
//  6. exact_kernel (thread per candidate, warps share an expert): the
//     reference's fp64 logits (sequential j, separately rounded mul/add).
//  7. final_kernel (thread per token): exact top-k among candidates with ties
//     to the lowest index (111-121), masked softmax (123-133) or logistic
//     (198), picks token-major, saved tensors for the backward.
// Results are identical to the exhaustive path; tests/test_routing_gpu.py runs
// both against the reference's golden vectors.
//
// Compiled with --fmad=false (explicit fmaf where the approximation wants it).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <algorithm>
#include <vector>

#include "host_once.h"
#include "capi_common.h"
#include "gemm.h"
#include "glibc_libm.cuh"
#include "kernels.h"
#include "route_common.cuh"
#include "sm100.cuh"

namespace fsmoe {
namespace {

using namespace fsmoe_dev;

constexpr int PS_MAXE = 64;  // experts handled by this path

template <int DT>
__device__ __forceinline__ float load_as_float(const void* base, long long i) {
  if constexpr (DT == 2) return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[i]);
  else if constexpr (DT == 1) return static_cast<const float*>(base)[i];
  else return static_cast<float>(static_cast<const double*>(base)[i]);
}

// W32[j][c], WT[c][j] for c < Ea from Wa, else from Wb; wn[c] = |column|_2 (upper bound).
// Wtc (optional): the tensor-core screen's B operand [128][M] bf16, K-major:
// row c = bf16(W[:, c]) (hi), row NC + c = bf16(W[:, c] - hi) (lo).
__global__ void w_prep_kernel(int M, int Ea, const double* __restrict__ Wa, int Eb,
                              const double* __restrict__ Wb, float* __restrict__ W32,
                              double* __restrict__ WT, double* __restrict__ wn,
                              __nv_bfloat16* __restrict__ Wtc) {
  fsmoe_dev::pdl_enter();
  const int NC = Ea + Eb;
  const int c = blockIdx.x;
  if (c >= NC) {  // blocks past the columns zero Wtc's unused rows [2 NC, ...)
    __nv_bfloat16* r = Wtc + static_cast<long long>(NC + c) * M;
    for (int j = threadIdx.x; j < M; j += blockDim.x) r[j] = __float2bfloat16(0.f);
    return;
  }
  double ss = 0.0;
  // eight rows' loads in flight per thread before their uses (the column is
  // strided in W: each load is its own line, so latency dominates)
  for (int j0 = threadIdx.x; j0 < M; j0 += 8 * blockDim.x) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + u * blockDim.x;
      v[u] = j >= M ? 0.0
                    : c < Ea ? Wa[static_cast<long long>(j) * Ea + c] : Wb[static_cast<long long>(j) * Eb + (c - Ea)];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + u * blockDim.x;
      if (j >= M) break;
      W32[static_cast<long long>(j) * NC + c] = static_cast<float>(v[u]);
      WT[static_cast<long long>(c) * M + j] = v[u];
      if (Wtc) {
        const __nv_bfloat16 h = __double2bfloat16(v[u]);
        Wtc[static_cast<long long>(c) * M + j] = h;
        Wtc[static_cast<long long>(NC + c) * M + j] = __double2bfloat16(v[u] - static_cast<double>(__bfloat162float(h)));
      }
      ss = __fma_rn(v[u], v[u], ss);
    }
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

constexpr int AP_TOK = 32;   // tokens per block
constexpr int AP_COL = 32;   // columns per block
constexpr int AP_JC = 64;    // reduction chunk
constexpr int AP_KS = 8;     // reduction splits (partials summed by bound_kernel)

// part[ks][t][c] = sum_{j in split ks} x[t][j] * W32[j][c] (fp32 FMA); 32 tokens
// x 32 cols per block of 64 threads (4 tokens x 4 cols each), gridDim.z = K
// splits. blockIdx.y == 0 also writes the split's |x_t|^2 (fp64).
template <int DT>
__global__ void __launch_bounds__(64)
    approx_scores_kernel(const void* __restrict__ x, int T, int M, const float* __restrict__ W32,
                         int NC, float* __restrict__ part, double* __restrict__ xn2part) {
  __shared__ __align__(16) float xs[AP_JC][AP_TOK + 4];  // transposed: 4 tokens = one float4
  __shared__ __align__(16) float ws[AP_JC][AP_COL];
  const int t0 = blockIdx.x * AP_TOK, c0 = blockIdx.y * AP_COL;
  const int ks = blockIdx.z;
  const int span = ((M + AP_KS - 1) / AP_KS + AP_JC - 1) / AP_JC * AP_JC;
  const int jbeg = ks * span, jend = min(M, jbeg + span);
  const int ty = threadIdx.x / 8, tx = threadIdx.x % 8;  // 8 token quads x 8 column quads
  float acc[4][4] = {};
  double nrm = 0.0;
  for (int j0 = jbeg; j0 < jend; j0 += AP_JC) {
    __syncthreads();
#pragma unroll
    for (int i = threadIdx.x; i < AP_TOK * AP_JC; i += 64) {
      const int tt = i / AP_JC, jj = i % AP_JC;
      const int t = t0 + tt, j = j0 + jj;
      xs[jj][tt] = (t < T && j < jend) ? load_as_float<DT>(x, static_cast<long long>(t) * M + j) : 0.f;
    }
#pragma unroll
    for (int i = threadIdx.x; i < AP_JC * AP_COL; i += 64) {
      const int jj = i / AP_COL, cc = i % AP_COL;
      const int j = j0 + jj, c = c0 + cc;
      ws[jj][cc] = (j < jend && c < NC) ? W32[static_cast<long long>(j) * NC + c] : 0.f;
    }
    __syncthreads();
    if (blockIdx.y == 0 && threadIdx.x < AP_TOK)
      for (int jj = 0; jj < AP_JC; ++jj) {
        const double v = xs[jj][threadIdx.x];
        nrm = __fma_rn(v, v, nrm);
      }
#pragma unroll 8
    for (int jj = 0; jj < AP_JC; ++jj) {
      const float4 av = reinterpret_cast<const float4*>(xs[jj])[ty];
      const float a[4] = {av.x, av.y, av.z, av.w};
      const float4 w = reinterpret_cast<const float4*>(ws[jj])[tx];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i][0] = fmaf(a[i], w.x, acc[i][0]);
        acc[i][1] = fmaf(a[i], w.y, acc[i][1]);
        acc[i][2] = fmaf(a[i], w.z, acc[i][2]);
        acc[i][3] = fmaf(a[i], w.w, acc[i][3]);
      }
    }
  }
  if (blockIdx.y == 0 && threadIdx.x < AP_TOK && t0 + threadIdx.x < T)
    xn2part[static_cast<long long>(ks) * T + t0 + threadIdx.x] = nrm;
  float* out = part + static_cast<long long>(ks) * T * NC;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + 4 * ty + i;
    if (t >= T) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c = c0 + 4 * tx + b;
      if (c < NC) out[static_cast<long long>(t) * NC + c] = acc[i][b];
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

// First 2E outputs of std::mt19937_64(seed+t) (2E <= 156: output i needs seed
// words i, i+1, i+156 — libstdc++ twists the whole state on the first draw).
// One thread per token: the seeding recurrence is sequential.
template <int MAXE>
__global__ void __launch_bounds__(128)
    mt_kernel(int T, int E, uint64_t seed, uint64_t* __restrict__ draws) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  uint64_t lo[2 * MAXE + 1];
  uint64_t w = seed + static_cast<uint64_t>(t);
  lo[0] = w;
  const int nout = 2 * E;
  for (int i = 1; i <= nout; ++i) {
    w = 6364136223846793005ULL * (w ^ (w >> 62)) + static_cast<uint64_t>(i);
    lo[i] = w;
  }
  for (int i = nout + 1; i < 156; ++i) w = 6364136223846793005ULL * (w ^ (w >> 62)) + static_cast<uint64_t>(i);
  uint64_t* out = draws + static_cast<long long>(t) * nout;
  for (int o = 0; o < nout; ++o) {
    w = 6364136223846793005ULL * (w ^ (w >> 62)) + static_cast<uint64_t>(156 + o);
    const uint64_t y = (lo[o] & MT_UM) | (lo[o + 1] & MT_LM);
    out[o] = temper(w ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL));
  }
}

// One thread per (token, expert): Box-Muller noise (noisy), the approximate
// score and its rigorous bound -> [lo, hi].
template <int KIND>
__global__ void __launch_bounds__(256)
    bound_kernel(int T, int E, int M, const float* __restrict__ part, const double* __restrict__ xn2part,
                 const double* __restrict__ wn, double cB, const uint64_t* __restrict__ draws,
                 double* __restrict__ noise, double* __restrict__ sapx, double* __restrict__ spapx,
                 double* __restrict__ lo, double* __restrict__ hi) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(T) * E) return;
  const int t = static_cast<int>(i / E), e = static_cast<int>(i % E);
  const int NC = KIND == 0 ? 2 * E : E;
  double xn = 0.0;
  float r = 0.f, sp = 0.f;
  for (int ks = 0; ks < AP_KS; ++ks) {
    xn += xn2part[static_cast<long long>(ks) * T + t];
    const float* p = part + (static_cast<long long>(ks) * T + t) * NC;
    r += p[e];
    if (KIND == 0) sp += p[E + e];
  }
  // summing the AP_KS fp32 partials adds at most AP_KS more roundings: covered
  // by the (M + 4) term since M >= AP_KS splits are never finer than 1 term.
  const double xnorm = sqrt(xn) * (1.0 + 1e-12);
  const double br = cB * xnorm * wn[e];
  double s, b;
  if (KIND == 0) {
    const uint64_t o0 = draws[static_cast<long long>(t) * 2 * E + 2 * e];
    const uint64_t o1 = draws[static_cast<long long>(t) * 2 * E + 2 * e + 1];
    double u1 = __dmul_rn(__dadd_rn(static_cast<double>(o0 >> 11), 0.5), 0x1.0p-53);
    double u2 = __dmul_rn(__dadd_rn(static_cast<double>(o1 >> 11), 0.5), 0x1.0p-53);
    double two_pi = 2.0 * 3.141592653589793238462643383279502884;
    const double n = fsmoe_libm::gl_normal(u1, u2);
    const double bs = cB * xnorm * wn[E + e];
    const double soft = log1p(exp(static_cast<double>(sp)));
    s = static_cast<double>(r) + n * soft;
    b = br + fabs(n) * bs + 1e-12 * (fabs(static_cast<double>(r)) + fabs(n * soft)) + 1e-300;
    noise[i] = n;
    spapx[i] = sp;
  } else {
    s = r;
    b = br + 1e-12 * fabs(static_cast<double>(r)) + 1e-300;
  }
  sapx[i] = s;
  lo[i] = s - b;
  hi[i] = s + b;
}

// One thread per token: candidates = experts whose upper bound reaches the
// k-th largest lower bound; appended to per-expert lists.
__global__ void __launch_bounds__(128)
    cand_kernel(int T, int E, int k, const double* __restrict__ lo, const double* __restrict__ hi,
                uint64_t* __restrict__ mask, int* __restrict__ lists, int* __restrict__ counts) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const double* l = lo + static_cast<long long>(t) * E;
  const double* h = hi + static_cast<long long>(t) * E;
  uint64_t taken = 0;
  double kth = 0.0;
  for (int j = 0; j < k; ++j) {
    int bi = -1;
    for (int e = 0; e < E; ++e)
      if (!((taken >> e) & 1ULL) && (bi < 0 || l[e] > l[bi])) bi = e;
    taken |= 1ULL << bi;
    kth = l[bi];
  }
  uint64_t m = 0;
  for (int e = 0; e < E; ++e)
    if (h[e] >= kth) {
      m |= 1ULL << e;
      lists[static_cast<long long>(e) * T + atomicAdd(&counts[e], 1)] = t;
    }
  mask[t] = m;
}

struct PruneWsView {
  const double* WT;
  const int* lists;
  const int* counts;
  double* s_exact;
  double* sp_exact;
};

// Exact fp64 logits for the candidates of expert blockIdx.y (matvec_row
// order, separately rounded mul/add): thread = (candidate, projection), where
// projection 0 is x.W_g and 1 (noisy) is x.W_noise. A warp shares one weight
// row (broadcast loads); token rows stream in batches of 64 values so many
// loads are in flight ahead of the dependent add chain.
template <int DT>
__device__ __forceinline__ void load8(const void* x, long long i, bool vec, double* o) {
  if constexpr (DT == 2) {
    if (vec) {
      uint4 u = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(x) + i);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float2 f = __bfloat1622float2(h[q]);
        o[2 * q] = f.x;
        o[2 * q + 1] = f.y;
      }
      return;
    }
  } else if constexpr (DT == 1) {
    if (vec) {
      float4 a = reinterpret_cast<const float4*>(static_cast<const float*>(x) + i)[0];
      float4 b = reinterpret_cast<const float4*>(static_cast<const float*>(x) + i)[1];
      o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
      return;
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) o[q] = load_as_double<DT>(x, i + q);
}

template <int DT, int NPROJ>
__global__ void __launch_bounds__(128)
    exact_kernel(const void* __restrict__ x, int T, int M, int E, const double* __restrict__ WT,
                 const int* __restrict__ lists, const int* __restrict__ counts,
                 double* __restrict__ raw_exact, double* __restrict__ sp_exact) {
  const int e = blockIdx.y;
  const int n = counts[e] * NPROJ;
  const bool vec = (M % 8) == 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int proj = i % NPROJ;
    const int t = lists[static_cast<long long>(e) * T + i / NPROJ];
    const long long xrow = static_cast<long long>(t) * M;
    const double* wr = WT + static_cast<long long>(proj * E + e) * M;
    double acc = 0.0;
    for (int j = 0; j < M; j += 8) {
      double xv[8];
      if (vec) load8<DT>(x, xrow + j, true, xv);
      else
        for (int q = 0; q < 8; ++q) xv[q] = j + q < M ? load_as_double<DT>(x, xrow + j + q) : 0.0;
      const int jn = M - j < 8 ? M - j : 8;
      for (int q = 0; q < jn; ++q) acc = __dadd_rn(acc, __dmul_rn(xv[q], wr[j + q]));
    }
    const long long o = static_cast<long long>(t) * E + e;
    if (proj == 0) raw_exact[o] = acc;
    else sp_exact[o] = acc;
  }
}

// Staged variant: a block takes EX_TOK candidates of one expert; their token
// rows and the expert's weight rows stream through shared memory in EX_JC
// chunks with TMA bulk copies (double-buffered, mbarrier completion), so the
// dependent fp64 add chain of each thread reads operands at smem latency.
// Thread = (candidate, projection).
constexpr int EX_TOK = 64;

template <int DT>
struct Elem {
  static constexpr int ES = DT == 0 ? 8 : DT == 1 ? 4 : 2;  // bytes per element
  static constexpr int JC = DT == 0 ? 128 : 256;           // columns per stage
  static constexpr int ROW = JC * ES + 16;                 // padded smem row stride
};

template <int DT, int NPROJ>
__global__ void __launch_bounds__(EX_TOK * NPROJ)
    exact_staged_kernel(const void* __restrict__ x, int T, int M, int E,
                        const double* __restrict__ WT, const int* __restrict__ lists,
                        const int* __restrict__ counts, double* __restrict__ raw_exact,
                        double* __restrict__ sp_exact) {
  constexpr int ES = Elem<DT>::ES, ROW = Elem<DT>::ROW, EX_JC = Elem<DT>::JC;
  constexpr int XS_BYTES = EX_TOK * ROW;
  constexpr int WS_BYTES = NPROJ * EX_JC * 8;
  constexpr int STAGE = XS_BYTES + WS_BYTES;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[2];
  __shared__ int toks[EX_TOK];
  const int e = blockIdx.y;
  const int c0 = blockIdx.x * EX_TOK;
  const int n = counts[e];
  if (c0 >= n) return;
  const int nt = min(EX_TOK, n - c0);
  const int tok = threadIdx.x % EX_TOK, proj = threadIdx.x / EX_TOK;
  if (threadIdx.x < EX_TOK) toks[threadIdx.x] = threadIdx.x < nt ? lists[static_cast<long long>(e) * T + c0 + threadIdx.x] : 0;
  if (threadIdx.x == 0) {
    fsmoe_dev::mbar_init(&full[0], 1);
    fsmoe_dev::mbar_init(&full[1], 1);
    fsmoe_dev::fence_barrier_init();
  }
  __syncthreads();
  const int nck = (M + EX_JC - 1) / EX_JC;
  auto issue = [&](int ck) {
    const int s = ck & 1;
    uint8_t* st = smem + s * STAGE;
    const int j0 = ck * EX_JC;
    const int len = min(EX_JC, M - j0);
    const uint32_t xb = static_cast<uint32_t>(len * ES), wb = static_cast<uint32_t>(len * 8);
    fsmoe_dev::mbar_arrive_expect_tx(&full[s], xb * nt + wb * NPROJ);
    for (int r = 0; r < nt; ++r)
      fsmoe_dev::bulk_load(st + r * ROW,
                           static_cast<const uint8_t*>(x) + (static_cast<long long>(toks[r]) * M + j0) * ES,
                           xb, &full[s]);
    for (int p = 0; p < NPROJ; ++p)
      fsmoe_dev::bulk_load(st + XS_BYTES + p * EX_JC * 8, WT + static_cast<long long>(p * E + e) * M + j0,
                           wb, &full[s]);
  };
  if (threadIdx.x == 0) {
    issue(0);
    if (nck > 1) issue(1);
  }
  double acc = 0.0;
  uint32_t ph[2] = {0, 0};
  for (int ck = 0; ck < nck; ++ck) {
    const int s = ck & 1;
    fsmoe_dev::mbar_wait(&full[s], ph[s]);
    ph[s] ^= 1;
    const uint8_t* xr = smem + s * STAGE + tok * ROW;
    const double* wr = reinterpret_cast<const double*>(smem + s * STAGE + XS_BYTES) + proj * EX_JC;
    const int len = min(EX_JC, M - ck * EX_JC);
    if (tok < nt) {
      int j = 0;
      for (; j + 8 <= len; j += 8) {
        double xv[8];
        load8<DT>(xr, j, true, xv);  // smem row, 16-byte aligned
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, __dmul_rn(xv[q], wr[j + q]));
      }
      for (; j < len; ++j) acc = __dadd_rn(acc, __dmul_rn(load_as_double<DT>(xr, j), wr[j]));
    }
    __syncthreads();  // stage s fully consumed
    if (threadIdx.x == 0 && ck + 2 < nck) issue(ck + 2);
  }
  if (tok < nt) {
    const long long o = static_cast<long long>(toks[tok]) * E + e;
    if (proj == 0) raw_exact[o] = acc;
    else sp_exact[o] = acc;
  }
}

template <int DT, int NPROJ>
void launch_exact(const void* x, int T, int M, int E, const PruneWsView& w, cudaStream_t st) {
  // staged path needs 16-byte aligned row chunks: M * elem % 16 == 0
  constexpr int ES = Elem<DT>::ES;
  const bool staged = (static_cast<long long>(M) * ES) % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  if (staged) {
    constexpr int SMEM = 2 * (EX_TOK * Elem<DT>::ROW + NPROJ * Elem<DT>::JC * 8);
    static DeviceOnce attr;
    once_on_device(attr, [&] { cudaFuncSetAttribute(exact_staged_kernel<DT, NPROJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM); });
    dim3 g((T + EX_TOK - 1) / EX_TOK, E);
    exact_staged_kernel<DT, NPROJ><<<g, EX_TOK * NPROJ, SMEM, st>>>(x, T, M, E, w.WT, w.lists, w.counts,
                                                                 w.s_exact, w.sp_exact);
  } else {
    dim3 eg((2 * T + 127) / 128 < 128 ? (2 * T + 127) / 128 : 128, E);
    exact_kernel<DT, NPROJ><<<eg, 128, 0, st>>>(x, T, M, E, w.WT, w.lists, w.counts, w.s_exact,
                                                w.sp_exact);
  }
  ::fsmoe::count_launch();
}

// Exact top-k among candidates, weights and picks (thread per token), then the
// saved tensors for the backward written coalesced by the whole block.
template <int KIND>
__global__ void __launch_bounds__(128)
    final_kernel(int T, int E, int k, const uint64_t* __restrict__ mask,
                 double* __restrict__ s_exact, const double* __restrict__ sp_exact,
                 const double* __restrict__ sapx, const double* __restrict__ spapx,
                 const double* __restrict__ noise, int* __restrict__ pick_token,
                 int* __restrict__ pick_expert, double* __restrict__ pick_weight,
                 double* __restrict__ scores_out, double* __restrict__ noise_out,
                 double* __restrict__ spread_out) {
  const int t0 = blockIdx.x * blockDim.x;
  const int t = t0 + threadIdx.x;
  if (t < T) {
    const uint64_t cand = mask[t];
    const long long row = static_cast<long long>(t) * E;
    if (KIND == 0)  // s = raw + n * softplus(spread)   (workload.cpp:186)
      for (uint64_t m = cand; m; m &= m - 1) {
        const long long o = row + __ffsll(static_cast<long long>(m)) - 1;
        s_exact[o] = __dadd_rn(s_exact[o], __dmul_rn(noise[o], fsmoe_libm::gl_softplus(sp_exact[o])));
      }
    uint64_t kept = 0;
    for (int j = 0; j < k; ++j) {
      int bi = -1;
      double best = 0.0;
      for (uint64_t m = cand & ~kept; m; m &= m - 1) {
        const int e = __ffsll(static_cast<long long>(m)) - 1;
        const double s = s_exact[row + e];
        if (bi < 0 || s > best) {
          best = s;
          bi = e;
        }
      }
      kept |= 1ULL << bi;
    }
    const long long base = static_cast<long long>(t) * k;
    if (KIND == 1) {
      uint64_t m = kept;
      for (int j = 0; j < k; ++j) {
        const int e = __ffsll(static_cast<long long>(m)) - 1;
        m &= m - 1;
        pick_token[base + j] = t;
        pick_expert[base + j] = e;
        pick_weight[base + j] = __ddiv_rn(1.0, __dadd_rn(1.0, fsmoe_libm::gl_exp(-s_exact[row + e])));
      }
    } else {
      uint64_t m = kept;
      double mx = s_exact[row + __ffsll(static_cast<long long>(m)) - 1];
      for (; m; m &= m - 1) {
        const double s = s_exact[row + __ffsll(static_cast<long long>(m)) - 1];
        mx = (mx < s) ? s : mx;
      }
      double z = 0.0;
      for (m = kept; m; m &= m - 1)
        z = __dadd_rn(z, fsmoe_libm::gl_exp(__dsub_rn(s_exact[row + __ffsll(static_cast<long long>(m)) - 1], mx)));
      m = kept;
      for (int j = 0; j < k; ++j) {
        const int e = __ffsll(static_cast<long long>(m)) - 1;
        m &= m - 1;
        pick_token[base + j] = t;
        pick_expert[base + j] = e;
        pick_weight[base + j] = __ddiv_rn(fsmoe_libm::gl_exp(__dsub_rn(s_exact[row + e], mx)), z);
      }
    }
  }
  // saved tensors: exact where a candidate (where gradients can be nonzero),
  // the finite approximations elsewhere
  const long long n = static_cast<long long>(min(T - t0, static_cast<int>(blockDim.x))) * E;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const long long o = static_cast<long long>(t0) * E + i;
    const int tt = static_cast<int>(o / E), e = static_cast<int>(o % E);
    const bool c = (mask[tt] >> e) & 1ULL;
    if (scores_out) scores_out[o] = c ? s_exact[o] : sapx[o];
    if (KIND == 0) {
      if (noise_out) noise_out[o] = noise[o];
      if (spread_out) spread_out[o] = c ? sp_exact[o] : spapx[o];
    }
  }
}


// ===================================================================== fused
// Two-kernel form of steps 2-7 for bf16 tokens, E <= 32 (the training hot
// path): `screen_kernel` = approximate scores + norms + noise + bounds +
// candidate masks for 64 tokens per block (no split-K partials, no T x E
// bound arrays in HBM); `exact_final_kernel` = the exact fp64 logits of each
// token's candidates and the final top-k / weights for 32 tokens per block
// (no per-expert candidate lists). Same arithmetic, same bound, same results.

constexpr int SC_TOK = 64;             // tokens per screen block
constexpr int SC_JC = 64;              // reduction chunk (columns of x)
constexpr int SC_STG = 4;              // cp.async pipeline depth (chunks in flight)
constexpr int SC_MT_WARPS = 2;         // warps that run the noise draws beside the loop
constexpr int SC_XROW = SC_JC + 8;     // bf16 per smem x row: 144 B, conflict-free LDS.128

__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(
                   __cvta_generic_to_shared(smem))),
               "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int SC_FROW = SC_JC + 4;    // fp32 per smem x row (converted tile)

// d = a * (b.x, b.y) + c, two IEEE fp32 FMAs in one FFMA2 (a broadcast)
__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  const float2 aa = make_float2(a, a);
  unsigned long long ra = *reinterpret_cast<const unsigned long long*>(&aa);
  unsigned long long rb = *reinterpret_cast<const unsigned long long*>(&b);
  unsigned long long rc = *reinterpret_cast<const unsigned long long*>(&c);
  unsigned long long rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}

template <int NCP, int E_MAX>
struct ScreenSmem {
  static constexpr int X = SC_STG * SC_TOK * SC_XROW * 2;  // bf16 x chunks
  static constexpr int XF = SC_TOK * SC_FROW * 4;          // the current chunk in fp32
  static constexpr int W = SC_STG * SC_JC * NCP * 4;       // fp32 W chunks
  static constexpr int LOOP = X + XF + W;
  // after the main loop the x / W tiles are dead and hold, in order:
  static constexpr int PART = 3 * SC_TOK * (NCP + 1) * 4;  // split-K partials
  static constexpr int SC = SC_TOK * (NCP + 1) * 4;        // approximate scores
  static constexpr int LOHI = SC_TOK * E_MAX * 8 * 2;      // bounds
  static_assert(PART + SC + LOHI <= LOOP, "post-loop data fits over the tiles");
  static constexpr int DRAWS = SC_TOK * 2 * E_MAX * 8;     // mt19937_64 outputs (own space)
  static constexpr int NRM = SC_TOK * 4 * 4;
  static constexpr int BYTES = LOOP + DRAWS + NRM;
};

// KIND 0 noisy (NC = 2E), 1 sigmoid (NC = E); NCP = NC rounded up to 32 / 64.
// Two thread groups split each chunk's columns of x (in-block split-K: two
// partial FMA chains per output, summed once; covered by the bound's split
// term). Thread (g, tx, ty): columns 4tx..4tx+3, tokens ty + 16 i (i < 4).
// in-block split-K groups: 512 GEMM threads per block (4 groups of 128 for 32
// columns, 2 of 256 for 64 columns)
template <int NCP>
__host__ __device__ constexpr int sc_grp() { return 512 / (NCP * 4); }

__device__ __forceinline__ void bar_sync_named(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// GEMM threads (NCP * 4 * SC_GRP) sync among themselves with named barrier 1;
// the extra SC_MT_WARPS warps compute the noise draws meanwhile (noisy only)
// and meet everyone at the first __syncthreads after the loop.
template <int KIND, int NCP, int E_MAX>
__global__ void __launch_bounds__(512 + SC_MT_WARPS * 32)
    screen_kernel(const __nv_bfloat16* __restrict__ x, int T, int M, int E, int k,
                  const float* __restrict__ W32, int NC, const double* __restrict__ wn, double cB,
                  double gam, uint64_t seed, double* __restrict__ noise_ws,
                  double* __restrict__ scores_out, double* __restrict__ spread_out,
                  uint64_t* __restrict__ mask) {
  using S = ScreenSmem<NCP, E_MAX>;
  constexpr int SC_GRP = sc_grp<NCP>();
  constexpr int NT = NCP * 4 * SC_GRP;
  constexpr int QX = NCP / 4;  // column quads
  extern __shared__ __align__(16) uint8_t sm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sm);
  float* xf = reinterpret_cast<float*>(sm + S::X);
  float* wsm = reinterpret_cast<float*>(sm + S::X + S::XF);
  double* lo = reinterpret_cast<double*>(sm + S::PART + S::SC);
  double* hi = lo + SC_TOK * E_MAX;
  uint64_t* draws = reinterpret_cast<uint64_t*>(sm + S::LOOP);
  float* nrm = reinterpret_cast<float*>(sm + S::LOOP + S::DRAWS);
  const int tid = threadIdx.x;
  const int grp = tid / (NCP * 4), lt = tid % (NCP * 4);
  const int tx = lt % QX, ty = lt / QX;
  const int t0 = blockIdx.x * SC_TOK;
  const int ntok = min(SC_TOK, T - t0);
  if (tid >= NT) {
    // ---- noise-draw warps: the seeding recurrence is sequential per token
    const int mt_tid = tid - NT;
    if (KIND == 0)
      for (int tl = mt_tid; tl < ntok; tl += SC_MT_WARPS * 32) {
        uint64_t lw[2 * E_MAX + 1];
        uint64_t w = seed + static_cast<uint64_t>(t0 + tl);
        lw[0] = w;
        const int nout = 2 * E;
        for (int i = 1; i <= nout; ++i) {
          w = 6364136223846793005ULL * (w ^ (w >> 62)) + static_cast<uint64_t>(i);
          lw[i] = w;
        }
        for (int i = nout + 1; i < 156; ++i) w = 6364136223846793005ULL * (w ^ (w >> 62)) + static_cast<uint64_t>(i);
        for (int o = 0; o < nout; ++o) {
          w = 6364136223846793005ULL * (w ^ (w >> 62)) + static_cast<uint64_t>(156 + o);
          const uint64_t y = (lw[o] & MT_UM) | (lw[o + 1] & MT_LM);
          draws[tl * 2 * E_MAX + o] = temper(w ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL));
        }
      }
  }
  // zero the padding columns of every W buffer once (cp.async only fills < NC)
  if (NC < NCP && tid < NT)
    for (int i = tid; i < SC_STG * SC_JC * NCP; i += NT)
      if (i % NCP >= NC) wsm[i] = 0.f;
  const int nck = M / SC_JC;
  auto issue = [&](int ck) {
    if (ck < nck) {
      const int b = ck % SC_STG;
      const int j0 = ck * SC_JC;
      for (int i = tid; i < SC_TOK * (SC_JC / 8); i += NT) {
        const int r = i / (SC_JC / 8), c = i % (SC_JC / 8);
        const int t = t0 + (r < ntok ? r : 0);
        cp_async16(xs + (b * SC_TOK + r) * SC_XROW + c * 8, x + static_cast<long long>(t) * M + j0 + c * 8);
      }
      const int q = NC / 4;
      for (int i = tid; i < SC_JC * q; i += NT) {
        const int r = i / q, c = i % q;
        cp_async16(wsm + (b * SC_JC + r) * NCP + c * 4, W32 + static_cast<long long>(j0 + r) * NC + c * 4);
      }
    }
    cp_async_commit();
  };
  float2 acc[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = make_float2(0.f, 0.f);
  float nacc = 0.f;  // |x|^2 partial: token tid/4, quarter (tid&3) of each chunk
  if (tid < NT) {
  for (int s0 = 0; s0 < SC_STG - 1; ++s0) issue(s0);
  for (int ck = 0; ck < nck; ++ck) {
    cp_async_wait<SC_STG - 2>();  // chunk ck has landed (later ones may be in flight)
    bar_sync_named(1, NT);
    const int b = ck % SC_STG;
    // bf16 -> fp32 once per element (thread: token tid/4, quarter tid&3),
    // |x|^2 from the exact squares of the bf16 values
    if (tid < 4 * SC_TOK) {
      const __nv_bfloat16* xr = xs + (b * SC_TOK + (tid >> 2)) * SC_XROW + (tid & 3) * (SC_JC / 4);
      float* fr = xf + (tid >> 2) * SC_FROW + (tid & 3) * (SC_JC / 4);
      static_assert(SC_JC % 32 == 0, "quarters of 8-element vectors");
#pragma unroll
      for (int j = 0; j < SC_JC / 4; j += 8) {
        const uint4 u = *reinterpret_cast<const uint4*>(xr + j);
        const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
        float v[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v[2 * q] = __uint_as_float(w4[q] << 16);
          v[2 * q + 1] = __uint_as_float(w4[q] & 0xffff0000u);
          nacc = fmaf(v[2 * q], v[2 * q], nacc);
          nacc = fmaf(v[2 * q + 1], v[2 * q + 1], nacc);
        }
        *reinterpret_cast<float4*>(fr + j) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(fr + j + 4) = make_float4(v[4], v[5], v[6], v[7]);
      }
    }
    bar_sync_named(1, NT);
    const float* wb = wsm + b * SC_JC * NCP;
#pragma unroll 2
    for (int j4 = grp * (SC_JC / 4 / SC_GRP); j4 < (grp + 1) * (SC_JC / 4 / SC_GRP); ++j4) {
      float4 xv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = *reinterpret_cast<const float4*>(xf + (ty + 16 * i) * SC_FROW + j4 * 4);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 w4 = *reinterpret_cast<const float4*>(wb + (j4 * 4 + q) * NCP + 4 * tx);
        const float2 wl = make_float2(w4.x, w4.y), wh = make_float2(w4.z, w4.w);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float xq = q == 0 ? xv[i].x : q == 1 ? xv[i].y : q == 2 ? xv[i].z : xv[i].w;
          acc[i][0] = ffma2(xq, wl, acc[i][0]);
          acc[i][1] = ffma2(xq, wh, acc[i][1]);
        }
      }
    }
    issue(ck + SC_STG - 1);  // into the stage chunk ck-1 used (everyone is past it)
  }
  cp_async_wait<0>();
  }
  __syncthreads();
  // approximate scores -> smem: groups 1..3 park their partial sums (the
  // x tiles are free now), group 0 adds them: (g0 + g1) + (g2 + g3), two more
  // roundings per output, inside the bound's split term; |x|^2 -> nrm
  // (both over the x / fp32-x / W tiles, which are dead after the loop)
  float* part = reinterpret_cast<float*>(sm);                     // [3][SC_TOK][NCP + 1]
  float* sc = reinterpret_cast<float*>(sm + S::PART);             // [SC_TOK][NCP + 1]
  if (grp > 0 && tid < NT) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float* o = part + ((grp - 1) * SC_TOK + ty + 16 * i) * (NCP + 1) + 4 * tx;
      o[0] = acc[i][0].x;
      o[1] = acc[i][0].y;
      o[2] = acc[i][1].x;
      o[3] = acc[i][1].y;
    }
  }
  if (tid < 4 * SC_TOK) nrm[tid] = nacc;
  __syncthreads();
  if (grp == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty + 16 * i;
      const float* p1 = part + r * (NCP + 1) + 4 * tx;
      const float* p2 = p1 + SC_TOK * (NCP + 1);
      const float* p3 = p2 + SC_TOK * (NCP + 1);
      float* o = sc + r * (NCP + 1) + 4 * tx;
      if constexpr (SC_GRP == 4) {
        o[0] = (acc[i][0].x + p1[0]) + (p2[0] + p3[0]);
        o[1] = (acc[i][0].y + p1[1]) + (p2[1] + p3[1]);
        o[2] = (acc[i][1].x + p1[2]) + (p2[2] + p3[2]);
        o[3] = (acc[i][1].y + p1[3]) + (p2[3] + p3[3]);
      } else {
        o[0] = acc[i][0].x + p1[0];
        o[1] = acc[i][0].y + p1[1];
        o[2] = acc[i][1].x + p1[2];
        o[3] = acc[i][1].y + p1[3];
      }
    }
  }
  __syncthreads();
  // bounds: |s~ - s_ref| <= cB |x|_2 |w_e|_2 (see the header); |x|^2 summed in
  // fp32 from exact bf16 squares: s <= s~ (1 + 2 gam), gam = gamma_M
  for (int pi = tid; pi < ntok * E; pi += blockDim.x) {
    const int tl = pi / E, e = pi % E;
    const long long o = static_cast<long long>(t0 + tl) * E + e;
    const double xs2 = (static_cast<double>(nrm[4 * tl]) + static_cast<double>(nrm[4 * tl + 1])) +
                       (static_cast<double>(nrm[4 * tl + 2]) + static_cast<double>(nrm[4 * tl + 3]));
    const double xnorm = sqrt(xs2 * (1.0 + 2.0 * gam)) * (1.0 + 1e-12);
    const float r = sc[tl * (NCP + 1) + e];
    const double br = cB * xnorm * wn[e];
    double s, bnd;
    if (KIND == 0) {
      const float sp = sc[tl * (NCP + 1) + E + e];
      const uint64_t o0 = draws[tl * 2 * E_MAX + 2 * e];
      const uint64_t o1 = draws[tl * 2 * E_MAX + 2 * e + 1];
      const double u1 = __dmul_rn(__dadd_rn(static_cast<double>(o0 >> 11), 0.5), 0x1.0p-53);
      const double u2 = __dmul_rn(__dadd_rn(static_cast<double>(o1 >> 11), 0.5), 0x1.0p-53);
      const double two_pi = 2.0 * 3.141592653589793238462643383279502884;
      const double n = fsmoe_libm::gl_normal(u1, u2);
      const double bs = cB * xnorm * wn[E + e];
      const double soft = log1p(exp(static_cast<double>(sp)));
      s = static_cast<double>(r) + n * soft;
      bnd = br + fabs(n) * bs + 1e-12 * (fabs(static_cast<double>(r)) + fabs(n * soft)) + 1e-300;
      noise_ws[o] = n;
      if (spread_out) spread_out[o] = sp;
    } else {
      s = r;
      bnd = br + 1e-12 * fabs(static_cast<double>(r)) + 1e-300;
    }
    if (scores_out) scores_out[o] = s;
    lo[tl * E_MAX + e] = s - bnd;
    hi[tl * E_MAX + e] = s + bnd;
  }
  __syncthreads();
  // candidates: upper bound reaches the k-th largest lower bound
  if (tid < ntok) {
    const double* l = lo + tid * E_MAX;
    const double* h = hi + tid * E_MAX;
    uint64_t taken = 0;
    double kth = 0.0;
    for (int j = 0; j < k; ++j) {
      int bi = -1;
      for (int e = 0; e < E; ++e)
        if (!((taken >> e) & 1ULL) && (bi < 0 || l[e] > l[bi])) bi = e;
      taken |= 1ULL << bi;
      kth = l[bi];
    }
    uint64_t m = 0;
    for (int e = 0; e < E; ++e)
      if (h[e] >= kth) m |= 1ULL << e;
    mask[t0 + tid] = m;
  }
}

// ------------------------------------------------- tensor-core screen --
// The approximate scores of the fused path on the tensor cores: one tcgen05
// GEMM P = x . [W_hi | W_lo] (bf16 operands, exact products, fp32 TMEM
// accumulation; W_hi = bf16(W), W_lo = bf16(W - W_hi)), then
// `screen_tc_kernel` turns P into s~ = P_hi + P_lo and applies the same
// noise / bound / candidate logic as `screen_kernel`. The bound covers:
// the hi/lo split residual |W - W_hi - W_lo| <= 2^-18 |W|, the tensor core's
// fp32 accumulation at up to two ulps per addition in any order
// (gamma' = M 2^-22 / (1 - M 2^-22), on |x| . (|W_hi| + |W_lo|) <=
// (1 + 2^-8) |x| . |W|), and the reference's own fp64 sequential rounding —
// all times |x|_2 |W_e|_2 (Cauchy-Schwarz), as before.
constexpr int TC_COLS = 128;  // GEMM output columns (2 NC <= 128)
constexpr int ST_TOK = 32;    // tokens per screen_tc block (8 threads each + one noise-draw warp)
constexpr int ST_MAIN = 8 * ST_TOK;
constexpr int ST_TPT = ST_MAIN / ST_TOK;

template <int KIND, int E_MAX>
__global__ void __launch_bounds__(ST_MAIN + 32)
    screen_tc_kernel(const __nv_bfloat16* __restrict__ x, int T, int M, int E, int k,
                     const float* __restrict__ P, const double* __restrict__ wn, double cB,
                     double gam, uint64_t seed, double* __restrict__ noise_ws,
                     double* __restrict__ scores_out, double* __restrict__ spread_out,
                     uint64_t* __restrict__ mask) {
  fsmoe_dev::pdl_enter();
  __shared__ uint64_t draws[KIND == 0 ? ST_TOK * 2 * E_MAX : 1];
  __shared__ float nrm[ST_MAIN];  // [token][ST_TPT partial sums]
  __shared__ double lo[ST_TOK * E_MAX], hi[ST_TOK * E_MAX];
  const int tid = threadIdx.x;
  const int t0 = blockIdx.x * ST_TOK;
  const int ntok = min(ST_TOK, T - t0);
  const int NC = KIND == 0 ? 2 * E : E;
  if (tid >= ST_MAIN) {
    // noise-draw warp (as screen_kernel): the first 2E outputs of mt19937_64(seed + t)
    const int mt_tid = tid - ST_MAIN;
    if (KIND == 0)
      for (int tl = mt_tid; tl < ntok; tl += 32) {
        uint64_t lw[2 * E_MAX + 1];
        uint64_t w = seed + static_cast<uint64_t>(t0 + tl);
        lw[0] = w;
        const int nout = 2 * E;
        for (int i = 1; i <= nout; ++i) {
          w = 6364136223846793005ULL * (w ^ (w >> 62)) + static_cast<uint64_t>(i);
          lw[i] = w;
        }
        for (int i = nout + 1; i < 156; ++i) w = 6364136223846793005ULL * (w ^ (w >> 62)) + static_cast<uint64_t>(i);
        for (int o = 0; o < nout; ++o) {
          w = 6364136223846793005ULL * (w ^ (w >> 62)) + static_cast<uint64_t>(156 + o);
          const uint64_t y = (lw[o] & MT_UM) | (lw[o + 1] & MT_LM);
          draws[tl * 2 * E_MAX + o] = temper(w ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL));
        }
      }
  } else {
    // |x_t|^2 from the exact squares of the bf16 values: ST_TPT threads per
    // token, each an interleaved share of the row (16-byte loads). (512-thread
    // blocks doing every item in one round measured slower: fewer blocks fit
    // an SM, so the grid no longer ran in a single wave.)
    const int tl = tid / ST_TPT, q = tid % ST_TPT;
    float nacc = 0.f;
    if (tl < ntok) {
      // batches of 8 independent 16-byte loads in flight per thread (the
      // loop is load-latency bound: one load per iteration stalled ~40 % of
      // the kernel's samples on its result)
      const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<long long>(t0 + tl) * M);
      const int nv = M / 8;
      constexpr int NB = 8;
      for (int v0 = q; v0 < nv; v0 += ST_TPT * NB) {
        uint4 u[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const int v = v0 + ST_TPT * i;
          u[i] = v < nv ? __ldg(xr + v) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const uint32_t w4[4] = {u[i].x, u[i].y, u[i].z, u[i].w};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float a = __uint_as_float(w4[c] << 16), b = __uint_as_float(w4[c] & 0xffff0000u);
            nacc = fmaf(a, a, nacc);
            nacc = fmaf(b, b, nacc);
          }
        }
      }
    }
    nrm[tid] = nacc;
  }
  __syncthreads();
  for (int pi = tid; pi < ntok * E; pi += blockDim.x) {
    const int tl = pi / E, e = pi % E;
    const long long o = static_cast<long long>(t0 + tl) * E + e;
    // fixed-order fp64 sum of the partials (any order is inside gam's bound;
    // the 1e-12 slack below covers the fp64 roundings)
    double xs2 = 0.0;
#pragma unroll
    for (int i = 0; i < ST_TPT; ++i) xs2 += static_cast<double>(nrm[tl * ST_TPT + i]);
    const double xnorm = sqrt(xs2 * (1.0 + 2.0 * gam)) * (1.0 + 1e-12);
    const float* pr = P + static_cast<long long>(t0 + tl) * TC_COLS;
    const double r = static_cast<double>(pr[e]) + static_cast<double>(pr[NC + e]);
    const double br = cB * xnorm * wn[e];
    double sv, bnd;
    if (KIND == 0) {
      const double sp = static_cast<double>(pr[E + e]) + static_cast<double>(pr[NC + E + e]);
      const uint64_t o0 = draws[tl * 2 * E_MAX + 2 * e];
      const uint64_t o1 = draws[tl * 2 * E_MAX + 2 * e + 1];
      const double u1 = __dmul_rn(__dadd_rn(static_cast<double>(o0 >> 11), 0.5), 0x1.0p-53);
      const double u2 = __dmul_rn(__dadd_rn(static_cast<double>(o1 >> 11), 0.5), 0x1.0p-53);
      const double n = fsmoe_libm::gl_normal(u1, u2);
      const double bs = cB * xnorm * wn[E + e];
      const double soft = log1p(exp(sp));
      sv = r + n * soft;
      bnd = br + fabs(n) * bs + 1e-12 * (fabs(r) + fabs(n * soft)) + 1e-300;
      noise_ws[o] = n;
      if (spread_out) spread_out[o] = sp;
    } else {
      sv = r;
      bnd = br + 1e-12 * fabs(r) + 1e-300;
    }
    if (scores_out) scores_out[o] = sv;
    lo[tl * E_MAX + e] = sv - bnd;
    hi[tl * E_MAX + e] = sv + bnd;
  }
  __syncthreads();
  // candidates: upper bound reaches the k-th largest lower bound
  if (tid < ntok) {
    const double* l = lo + tid * E_MAX;
    const double* h = hi + tid * E_MAX;
    uint64_t taken = 0;
    double kth = 0.0;
    for (int j = 0; j < k; ++j) {
      int bi = -1;
      for (int e = 0; e < E; ++e)
        if (!((taken >> e) & 1ULL) && (bi < 0 || l[e] > l[bi])) bi = e;
      taken |= 1ULL << bi;
      kth = l[bi];
    }
    uint64_t m = 0;
    for (int e = 0; e < E; ++e)
      if (h[e] >= kth) m |= 1ULL << e;
    mask[t0 + tid] = m;
  }
}

constexpr int XF_TOK = 64;       // tokens per exact/final block
constexpr int XF_THREADS = 256;
constexpr int XF_JC = 64;        // columns per stage
constexpr int XF_XROW = XF_JC * 2 + 16;  // bf16 row bytes (+16: conflict-free LDS.128)
constexpr int XF_WROW = XF_JC + 2;       // fp64 per W^T smem row (+16 B, same reason)

template <int NPROJ, int E_MAX>
struct XfSmem {
  static constexpr int XS = XF_TOK * XF_XROW;             // token rows of one stage
  static constexpr int WS = NPROJ * E_MAX * XF_WROW * 8;   // W^T rows (fp64) of one stage
  static constexpr int STAGE = XS + WS;
  static constexpr int NS = 2;                               // stages in flight
  static constexpr int BYTES_STAGES = NS * STAGE;            // at E = E_MAX
  // the top-1 certain-pick path's dot / bound scratch (KIND 0 only) reuses it
  static constexpr int CERT = NPROJ == 2 ? XF_TOK * E_MAX * 2 * 8 * 2 : 0;
  static constexpr int BYTES = BYTES_STAGES > CERT ? BYTES_STAGES : CERT;  // the attribute
  // the launched stage stride holds the W^T rows of the E actual experts
  static __host__ __device__ int stride(int E) { return XS + NPROJ * E * XF_WROW * 8; }
};

// Exact fp64 logits of each token's candidates (the reference's sequential
// separately rounded mul/add over j, workload.cpp:103-108) with the token
// rows and all W^T rows streamed through shared memory in XF_JC-column
// stages (cp.async, S::NS stages in flight); thread = (token, candidate,
// projection).
// Then the final exact top-k, weights and picks for the block's tokens.
template <int KIND, int E_MAX>
__global__ void __launch_bounds__(XF_THREADS)
    exact_final_kernel(const __nv_bfloat16* __restrict__ x, int T, int M, int E, int k,
                       const double* __restrict__ WT, const uint64_t* __restrict__ mask,
                       const double* __restrict__ noise, int* __restrict__ pick_token,
                       int* __restrict__ pick_expert, double* __restrict__ pick_weight,
                       double* __restrict__ scores_out, double* __restrict__ spread_out) {
  fsmoe_dev::pdl_enter();
  constexpr int NPROJ = KIND == 0 ? 2 : 1;
  using S = XfSmem<NPROJ, E_MAX>;
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint64_t msk[XF_TOK];
  __shared__ int cnt[XF_TOK];
  __shared__ short2 items[XF_TOK * E_MAX];
  __shared__ int nitems;
  __shared__ double ex[NPROJ][XF_TOK][E_MAX];
  const int tid = threadIdx.x;
  const int t0 = blockIdx.x * XF_TOK;
  const int ntok = min(XF_TOK, T - t0);
  const int nW = NPROJ * E;
  const int stg = S::stride(E);
  auto issue = [&](int ck) {
    if (ck * XF_JC < M) {
      uint8_t* st = sm + (ck % S::NS) * stg;
      const int j0 = ck * XF_JC;
      for (int i = tid; i < XF_TOK * (XF_JC / 8); i += XF_THREADS) {
        const int r = i / (XF_JC / 8), c = i % (XF_JC / 8);
        const int t = t0 + (r < ntok ? r : 0);
        cp_async16(st + r * XF_XROW + c * 16, x + static_cast<long long>(t) * M + j0 + c * 8);
      }
      double* ws = reinterpret_cast<double*>(st + S::XS);
      for (int i = tid; i < nW * (XF_JC / 2); i += XF_THREADS) {
        const int r = i / (XF_JC / 2), c = i % (XF_JC / 2);
        cp_async16(ws + r * XF_WROW + c * 2, WT + static_cast<long long>(r) * M + j0 + c * 2);
      }
    }
    cp_async_commit();
  };
  // Top-1 softmax with no saved scores requested: a token whose bound leaves a
  // single candidate has a certain pick and weight exactly 1.0 (softmax over
  // one survivor, workload.cpp:123-133) -- its exact logits are never needed
  const bool certain_ok = KIND == 0 && k == 1 && !scores_out && !spread_out;
  if (tid < XF_TOK) {
    const uint64_t m = tid < ntok ? mask[t0 + tid] : 0ULL;
    msk[tid] = m;
    cnt[tid] = (certain_ok && __popcll(m) == 1) ? 0 : __popcll(m);
  }
  __syncthreads();
  if (certain_ok) {
    // Tokens whose fp32 bound left 2+ candidates: decide with fp64 dot
    // products summed warp-parallel (FMA, 32 partial chains of M/32 terms + 5
    // shuffle levels) and a rigorous bound on their distance from the
    // reference's sequential sums -- |seq - par| <= (gamma_M + gamma_{M/32+5})
    // sum|x_j w_j| -- plus the noise / softplus / final-add roundings. A
    // decided token gets its certain pick (weight 1.0); an undecided one
    // (ties, near ties) keeps its candidates for the sequential reference
    // chain below. One warp per (token, candidate, projection) dot product.
    __shared__ int nref;
    __shared__ unsigned char ref_tok[XF_TOK];
    double* rd = reinterpret_cast<double*>(sm);              // [XF_TOK][E_MAX][2] dots
    double* ra = rd + XF_TOK * E_MAX * 2;                    // same, sum |x w|
    if (tid == 0) {
      int n = 0;
      for (int tl = 0; tl < ntok; ++tl)
        if (__popcll(msk[tl]) >= 2) ref_tok[n++] = static_cast<unsigned char>(tl);
      nref = n;
    }
    __syncthreads();
    if (nref > 0) {
      const int warp = tid >> 5, lane = tid & 31;
      const int nit = nref * E_MAX * 2;
      for (int it = warp; it < nit; it += XF_THREADS / 32) {
        const int r = it / (E_MAX * 2), e = (it / 2) % E_MAX, pj = it & 1;
        const int tl = ref_tok[r];
        if (e >= E || !((msk[tl] >> e) & 1ULL)) continue;
        const __nv_bfloat16* xr = x + static_cast<long long>(t0 + tl) * M;
        const double* wr = WT + static_cast<long long>(pj * E + e) * M;
        double d = 0.0, aa = 0.0;
#pragma unroll 4
        for (int j0 = lane * 8; j0 < M; j0 += 256) {
          const uint4 uu = __ldg(reinterpret_cast<const uint4*>(xr + j0));
          const uint32_t w4[4] = {uu.x, uu.y, uu.z, uu.w};
          double2 wv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) wv[q] = __ldg(reinterpret_cast<const double2*>(wr + j0 + 2 * q));
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double x0 = static_cast<double>(__uint_as_float(w4[q] << 16));
            const double x1 = static_cast<double>(__uint_as_float(w4[q] & 0xffff0000u));
            d = __fma_rn(x0, wv[q].x, d);
            d = __fma_rn(x1, wv[q].y, d);
            aa = __fma_rn(fabs(x0), fabs(wv[q].x), aa);
            aa = __fma_rn(fabs(x1), fabs(wv[q].y), aa);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          d += __shfl_xor_sync(0xffffffffu, d, o);
          aa += __shfl_xor_sync(0xffffffffu, aa, o);
        }
        if (lane == 0) {
          rd[(r * E_MAX + e) * 2 + pj] = d;
          ra[(r * E_MAX + e) * 2 + pj] = aa * (1.0 + 1e-12);
        }
      }
      __syncthreads();
      if (tid < nref) {
        const int tl = ref_tok[tid];
        const uint64_t m = msk[tl];
        const double u = 0x1.0p-53;
        const double np = M / 32.0 + 5.0;  // terms per lane chain + shuffle levels
        const double g = (M * u / (1.0 - M * u) + np * u / (1.0 - np * u)) * 1.01;
        double best_s = 0.0, best_b = 0.0, other_hi = -1.0 / 0.0;
        int best = -1;
        for (uint64_t mm = m; mm; mm &= mm - 1) {
          const int e = __ffsll(static_cast<long long>(mm)) - 1;
          const double d0 = rd[(tid * E_MAX + e) * 2], d1 = rd[(tid * E_MAX + e) * 2 + 1];
          const double a0 = ra[(tid * E_MAX + e) * 2], a1 = ra[(tid * E_MAX + e) * 2 + 1];
          const double n = noise[static_cast<long long>(t0 + tl) * E + e];
          const double soft = fsmoe_libm::gl_softplus(d1);
          const double sv = d0 + n * soft;
          const double b = g * (a0 + fabs(n) * a1) +
                           8.0 * u * (fabs(d0) + fabs(n * soft) + fabs(n) * soft) + 1e-300;
          // best by value (ascending index: a later candidate must be larger);
          // every other candidate's upper bound is tracked in other_hi
          if (best < 0 || sv > best_s) {
            if (best >= 0) other_hi = fmax(other_hi, best_s + best_b);
            best = e;
            best_s = sv;
            best_b = b;
          } else {
            other_hi = fmax(other_hi, sv + b);
          }
        }
        // certain iff the winner's lower bound clears every other upper bound
        if (best_s - best_b > other_hi) {
          msk[tl] = 1ULL << best;
          cnt[tl] = 0;
        }
      }
      __syncthreads();
    }
  }
  if (tid < 32) {
    // candidate list in expert-major order (then token): the lanes of a warp
    // then mostly share one expert, so their W^T reads in the chains below
    // are shared-memory broadcasts (token-major lists made every lane read
    // its own row: the kernel was bound by shared-memory wavefronts)
    const uint64_t m0 = cnt[tid] ? msk[tid] : 0ULL, m1 = cnt[tid + 32] ? msk[tid + 32] : 0ULL;
    const unsigned lt = (1u << tid) - 1u;
    int base = 0;
    for (int e = 0; e < E; ++e) {
      const bool h0 = (m0 >> e) & 1ULL, h1 = (m1 >> e) & 1ULL;
      const unsigned b0 = __ballot_sync(0xffffffffu, h0), b1 = __ballot_sync(0xffffffffu, h1);
      if (h0) items[base + __popc(b0 & lt)] = make_short2(static_cast<short>(tid), static_cast<short>(e));
      if (h1) items[base + __popc(b0) + __popc(b1 & lt)] = make_short2(static_cast<short>(tid + 32), static_cast<short>(e));
      base += __popc(b0) + __popc(b1);
    }
    if (tid == 0) nitems = base;
  }
  __syncthreads();
  const int nc = nitems;
  // work item = candidate (token, expert); its NPROJ chains (score and noise
  // projection) share every x load and its fp64 conversion -- the
  // conversions (F2F, XU pipe) bounded the kernel when each projection
  // converted the row again. A thread holds up to 2 items (a block rarely
  // has > 2 * XF_THREADS candidates; the rest run from global memory below).
  const int nwork = nc;
  double acc0[NPROJ], acc1[NPROJ];
#pragma unroll
  for (int pj = 0; pj < NPROJ; ++pj) acc0[pj] = acc1[pj] = 0.0;
  const int it0 = tid, it1 = tid + XF_THREADS;
  const short2 te0 = it0 < nwork ? items[it0] : make_short2(0, 0);
  const short2 te1 = it1 < nwork ? items[it1] : make_short2(0, 0);
  // 8 consecutive terms of every chain: acc_p = acc_p + x_j * W_p[j], in j
  // order, each product and sum separately rounded (workload.cpp:103-108)
  auto chain8 = [&](double (&acc)[NPROJ], const uint4 u, const double* const (&wr)[NPROJ]) {
    const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double xa = static_cast<double>(__uint_as_float(w4[q] << 16));
      const double xb = static_cast<double>(__uint_as_float(w4[q] & 0xffff0000u));
#pragma unroll
      for (int pj = 0; pj < NPROJ; ++pj) {
        const double2 wv = *reinterpret_cast<const double2*>(wr[pj] + 2 * q);
        acc[pj] = __dadd_rn(acc[pj], __dmul_rn(xa, wv.x));
        acc[pj] = __dadd_rn(acc[pj], __dmul_rn(xb, wv.y));
      }
    }
  };
  // A block with only a handful of candidates (the few tokens whose bound
  // leaves 2+ candidates) bulk-loads just those rows and runs each chain from
  // shared memory with no per-chunk barriers: the chain's latency, not the
  // staging pipeline, is then the block's time.
  __shared__ __align__(8) uint64_t sbar;
  const long long item_bytes = static_cast<long long>(M) * (2 + 8 * NPROJ);
  const long long small_bytes = static_cast<long long>(nwork) * item_bytes;
  const bool small = nwork > 0 && small_bytes <= S::NS * stg && M % 8 == 0;
  if (small) {
    if (tid == 0) {
      fsmoe_dev::mbar_init(&sbar, 1);
      fsmoe_dev::fence_barrier_init();
      fsmoe_dev::mbar_arrive_expect_tx(&sbar, static_cast<uint32_t>(small_bytes));
      for (int it = 0; it < nwork; ++it) {
        const short2 te = items[it];
        uint8_t* d = sm + static_cast<long long>(it) * item_bytes;
        fsmoe_dev::bulk_load(d, x + static_cast<long long>(t0 + te.x) * M, static_cast<uint32_t>(M * 2), &sbar);
        for (int pj = 0; pj < NPROJ; ++pj)
          fsmoe_dev::bulk_load(d + M * 2 + static_cast<long long>(pj) * M * 8,
                               WT + static_cast<long long>(pj * E + te.y) * M, static_cast<uint32_t>(M * 8), &sbar);
      }
    }
    __syncthreads();
    if (tid < nwork) {
      fsmoe_dev::mbar_wait(&sbar, 0);
      const uint8_t* xr = sm + static_cast<long long>(tid) * item_bytes;
      const double* w0 = reinterpret_cast<const double*>(xr + M * 2);
#pragma unroll 2
      for (int j = 0; j < M; j += 8) {
        const double* wr[NPROJ];
#pragma unroll
        for (int pj = 0; pj < NPROJ; ++pj) wr[pj] = w0 + static_cast<long long>(pj) * M + j;
        chain8(acc0, *reinterpret_cast<const uint4*>(xr + 2 * j), wr);
      }
#pragma unroll
      for (int pj = 0; pj < NPROJ; ++pj) ex[pj][te0.x][te0.y] = acc0[pj];
    }
  }
  // otherwise stream the token / weight rows in chunks (when there is work)
  const int nck = (nwork > 0 && !small) ? (M + XF_JC - 1) / XF_JC : 0;
  if (nck > 0)
    for (int i = 0; i < S::NS - 1; ++i) issue(i);  // every issue commits a group (maybe empty)
  for (int ck = 0; ck < nck; ++ck) {
    cp_async_wait<S::NS - 2>();  // chunk ck has landed
    __syncthreads();             // ... for every thread, and chunk ck - 1's buffer is free
    issue(ck + S::NS - 1);       // into that buffer, in flight while chunk ck is consumed
    const uint8_t* st = sm + (ck % S::NS) * stg;
    const double* ws = reinterpret_cast<const double*>(st + S::XS);
    auto run = [&](double (&acc)[NPROJ], short2 te) {
      const uint8_t* xr = st + te.x * XF_XROW;
#pragma unroll 2
      for (int j = 0; j < XF_JC; j += 8) {
        const double* wr[NPROJ];
#pragma unroll
        for (int pj = 0; pj < NPROJ; ++pj) wr[pj] = ws + (pj * E + te.y) * XF_WROW + j;
        chain8(acc, *reinterpret_cast<const uint4*>(xr + 2 * j), wr);
      }
    };
    if (it0 < nwork) run(acc0, te0);
    if (it1 < nwork) run(acc1, te1);
  }
#pragma unroll
  for (int pj = 0; pj < NPROJ; ++pj) {
    if (!small && it0 < nwork) ex[pj][te0.x][te0.y] = acc0[pj];
    if (!small && it1 < nwork) ex[pj][te1.x][te1.y] = acc1[pj];
  }
  // more than 2 * XF_THREADS candidates: the rest from global memory
  for (int it = it1 + XF_THREADS; it < nwork; it += XF_THREADS) {
    const short2 te = items[it];
    const __nv_bfloat16* xr = x + static_cast<long long>(t0 + te.x) * M;
    double acc[NPROJ];
#pragma unroll
    for (int pj = 0; pj < NPROJ; ++pj) acc[pj] = 0.0;
    for (int j = 0; j < M; ++j) {
      const double xv = static_cast<double>(__bfloat162float(xr[j]));
#pragma unroll
      for (int pj = 0; pj < NPROJ; ++pj)
        acc[pj] = __dadd_rn(acc[pj], __dmul_rn(xv, WT[static_cast<long long>(pj * E + te.y) * M + j]));
    }
#pragma unroll
    for (int pj = 0; pj < NPROJ; ++pj) ex[pj][te.x][te.y] = acc[pj];
  }
  __syncthreads();
  if (tid >= ntok) return;
  const int t = t0 + tid;
  const uint64_t cand = msk[tid];
  const long long row = static_cast<long long>(t) * E;
  if (certain_ok && __popcll(cand) == 1) {
    pick_token[t] = t;
    pick_expert[t] = __ffsll(static_cast<long long>(cand)) - 1;
    pick_weight[t] = 1.0;
    return;
  }
  double* s = ex[0][tid];
  for (uint64_t m = cand; m; m &= m - 1) {
    const int e = __ffsll(static_cast<long long>(m)) - 1;
    if (KIND == 0) {  // s = raw + n * softplus(spread)   (workload.cpp:186)
      s[e] = __dadd_rn(s[e], __dmul_rn(noise[row + e], fsmoe_libm::gl_softplus(ex[NPROJ - 1][tid][e])));
      if (spread_out) spread_out[row + e] = ex[NPROJ - 1][tid][e];
    }
    if (scores_out) scores_out[row + e] = s[e];
  }
  uint64_t kept = 0;
  for (int j = 0; j < k; ++j) {
    int bi = -1;
    double best = 0.0;
    for (uint64_t m = cand & ~kept; m; m &= m - 1) {
      const int e = __ffsll(static_cast<long long>(m)) - 1;
      if (bi < 0 || s[e] > best) {
        best = s[e];
        bi = e;
      }
    }
    kept |= 1ULL << bi;
  }
  const long long pb = static_cast<long long>(t) * k;
  if (KIND == 1) {
    uint64_t m = kept;
    for (int j = 0; j < k; ++j) {
      const int e = __ffsll(static_cast<long long>(m)) - 1;
      m &= m - 1;
      pick_token[pb + j] = t;
      pick_expert[pb + j] = e;
      pick_weight[pb + j] = __ddiv_rn(1.0, __dadd_rn(1.0, fsmoe_libm::gl_exp(-s[e])));
    }
  } else {
    uint64_t m = kept;
    double mx = s[__ffsll(static_cast<long long>(m)) - 1];
    for (; m; m &= m - 1) {
      const double v = s[__ffsll(static_cast<long long>(m)) - 1];
      mx = (mx < v) ? v : mx;
    }
    double z = 0.0;
    for (m = kept; m; m &= m - 1) z = __dadd_rn(z, fsmoe_libm::gl_exp(__dsub_rn(s[__ffsll(static_cast<long long>(m)) - 1], mx)));
    m = kept;
    for (int j = 0; j < k; ++j) {
      const int e = __ffsll(static_cast<long long>(m)) - 1;
      m &= m - 1;
      pick_token[pb + j] = t;
      pick_expert[pb + j] = e;
      pick_weight[pb + j] = __ddiv_rn(fsmoe_libm::gl_exp(__dsub_rn(s[e], mx)), z);
    }
  }
}

template <int KIND, int NCP, int E_MAX>
void launch_fused(const fsmoe_gate_desc& d, const void* x, double cB, const float* W32,
                  const double* WT, const double* wn, double* noise_ws, uint64_t* mask,
                  int* pick_token, int* pick_expert, double* pick_weight, double* scores_out,
                  double* spread_out, cudaStream_t st) {
  const int T = d.tokens, M = d.model_dim, E = d.score_cols, k = d.top_k;
  const int NC = KIND == 0 ? 2 * E : E;
  const double u = 0x1.0p-24;
  const double gam = M * u / (1.0 - M * u);
  constexpr int SMEM = ScreenSmem<NCP, E_MAX>::BYTES;
  static DeviceOnce attr;
  once_on_device(attr, [&] { cudaFuncSetAttribute(screen_kernel<KIND, NCP, E_MAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM); });
  const auto* xb = static_cast<const __nv_bfloat16*>(x);
  screen_kernel<KIND, NCP, E_MAX><<<(T + SC_TOK - 1) / SC_TOK, 512 + SC_MT_WARPS * 32, SMEM, st>>>(
      xb, T, M, E, k, W32, NC, wn, cB, gam, d.seed, noise_ws, scores_out, spread_out, mask);
  ::fsmoe::count_launch();
  constexpr int XSMEM = XfSmem<KIND == 0 ? 2 : 1, E_MAX>::BYTES;
  static DeviceOnce xattr;
  once_on_device(xattr, [&] { cudaFuncSetAttribute(exact_final_kernel<KIND, E_MAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, XSMEM); });
  // E's stages (at least the certain-pick path's dot / bound scratch)
  const int xs_rt = std::max(XfSmem<KIND == 0 ? 2 : 1, E_MAX>::NS * XfSmem<KIND == 0 ? 2 : 1, E_MAX>::stride(E),
                             XfSmem<KIND == 0 ? 2 : 1, E_MAX>::CERT);
  pdl_launch(exact_final_kernel<KIND, E_MAX>, (T + XF_TOK - 1) / XF_TOK, XF_THREADS, xs_rt, st, 
      xb, T, M, E, k, WT, mask, noise_ws, pick_token, pick_expert, pick_weight, scores_out,
      spread_out);
  ::fsmoe::count_launch();
}

template <int KIND, int E_MAX>
void launch_fused_tc(const fsmoe_gate_desc& d, const void* x, const __nv_bfloat16* Wtc, float* P,
                     const double* WT, const double* wn, double* noise_ws, uint64_t* mask,
                     int* pick_token, int* pick_expert, double* pick_weight, double* scores_out,
                     double* spread_out, cudaStream_t st) {
  const int T = d.tokens, M = d.model_dim, E = d.score_cols, k = d.top_k;
  GemmProblem g;
  g.kind = GemmKind::RowGrouped;
  g.nblk = 1;
  g.rows = g.rows_total = T;
  g.K = M;
  g.N = TC_COLS;
  g.n_w = 1;
  g.A = x;
  g.B = Wtc;
  g.epi = Epi::StoreF32;
  g.D = P;
  g.ldd = TC_COLS;
  g.force_ctas = 2;
  g.force_bn = 128;
  if (int rc = gemm_sm100_launch(g, st)) return (void)cuda_status(static_cast<cudaError_t>(rc), "gate screen gemm");
  ::fsmoe::count_launch();
  const double u2 = 0x1.0p-22;  // up to two fp32 ulps per tensor-core addition
  const double gamp = M * u2 / (1.0 - M * u2);
  const double cB = gamp * (1.0 + 0x1.0p-8) * 1.01 + 0x1.0p-18 + (M + 2.0) * 0x1.0p-53;
  const double gam = M * 0x1.0p-24 / (1.0 - M * 0x1.0p-24);  // fp32 |x|^2 sums
  const auto* xb = static_cast<const __nv_bfloat16*>(x);
  pdl_launch(screen_tc_kernel<KIND, E_MAX>, (T + ST_TOK - 1) / ST_TOK, ST_MAIN + 32, 0, st, 
      xb, T, M, E, k, P, wn, cB, gam, d.seed, noise_ws, scores_out, spread_out, mask);
  ::fsmoe::count_launch();
  constexpr int XSMEM = XfSmem<KIND == 0 ? 2 : 1, E_MAX>::BYTES;
  static DeviceOnce xattr;
  once_on_device(xattr, [&] { cudaFuncSetAttribute(exact_final_kernel<KIND, E_MAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, XSMEM); });
  // E's stages (at least the certain-pick path's dot / bound scratch)
  const int xs_rt = std::max(XfSmem<KIND == 0 ? 2 : 1, E_MAX>::NS * XfSmem<KIND == 0 ? 2 : 1, E_MAX>::stride(E),
                             XfSmem<KIND == 0 ? 2 : 1, E_MAX>::CERT);
  pdl_launch(exact_final_kernel<KIND, E_MAX>, (T + XF_TOK - 1) / XF_TOK, XF_THREADS, xs_rt, st, 
      xb, T, M, E, k, WT, mask, noise_ws, pick_token, pick_expert, pick_weight, scores_out,
      spread_out);
  ::fsmoe::count_launch();
}

struct PruneWs {
  __nv_bfloat16* Wtc;  // tensor-core screen: B operand [TC_COLS][M] (hi | lo | 0)
  float* P;            // its fp32 products [T][TC_COLS]
  float* W32;
  double* WT;
  double* wn;
  float* part;
  double* xn2;
  uint64_t* draws;
  double* noise;
  double* sapx;
  double* spapx;
  double* lo;
  double* hi;
  uint64_t* mask;
  int* lists;
  int* counts;
  double* s_exact;
  double* sp_exact;
  size_t bytes;
};

PruneWs carve(const fsmoe_gate_desc& d, void* base) {
  const size_t T = d.tokens, E = d.score_cols, M = d.model_dim;
  const size_t NC = d.kind == FSMOE_GATE_NOISY_TOPK ? 2 * E : E;
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t b) {
    char* r = p ? p + off : nullptr;
    off += (b + 255) & ~size_t(255);
    return r;
  };
  PruneWs w;
  w.W32 = reinterpret_cast<float*>(take(4 * M * NC));
  w.WT = reinterpret_cast<double*>(take(8 * M * NC));
  w.wn = reinterpret_cast<double*>(take(8 * NC));
  w.part = reinterpret_cast<float*>(take(4 * AP_KS * T * NC));
  w.xn2 = reinterpret_cast<double*>(take(8 * AP_KS * T));
  w.draws = reinterpret_cast<uint64_t*>(take(8 * T * 2 * E));
  w.noise = reinterpret_cast<double*>(take(8 * T * E));
  w.sapx = reinterpret_cast<double*>(take(8 * T * E));
  w.spapx = reinterpret_cast<double*>(take(8 * T * E));
  w.lo = reinterpret_cast<double*>(take(8 * T * E));
  w.hi = reinterpret_cast<double*>(take(8 * T * E));
  w.mask = reinterpret_cast<uint64_t*>(take(8 * T));
  w.lists = reinterpret_cast<int*>(take(4 * T * E));
  w.counts = reinterpret_cast<int*>(take(4 * E));
  w.s_exact = reinterpret_cast<double*>(take(8 * T * E));
  w.sp_exact = reinterpret_cast<double*>(take(8 * T * E));
  w.Wtc = reinterpret_cast<__nv_bfloat16*>(take(2 * TC_COLS * M));
  w.P = reinterpret_cast<float*>(take(4 * TC_COLS * T));
  w.bytes = off;
  return w;
}

}  // namespace

size_t gate_prune_workspace_bytes(const fsmoe_gate_desc& d) { return carve(d, nullptr).bytes; }

bool gate_prune_applicable(const fsmoe_gate_desc& d) {
  if (d.kind != FSMOE_GATE_NOISY_TOPK && d.kind != FSMOE_GATE_SIGMOID_TOPK) return false;
  return d.score_cols <= PS_MAXE;
}

int gate_prune_launch(const fsmoe_gate_desc& d, const void* x, const double* w_score,
                      const double* w_noise, int* pick_token, int* pick_expert,
                      double* pick_weight, double* scores_out, double* noise_out,
                      double* spread_out, void* ws, cudaStream_t st) {
  const int T = d.tokens, M = d.model_dim, E = d.score_cols, k = d.top_k;
  const bool noisy = d.kind == FSMOE_GATE_NOISY_TOPK;
  const int NC = noisy ? 2 * E : E;
  PruneWs w = carve(d, ws);
  FSMOE_CUDA_TRY(cudaMemsetAsync(w.counts, 0, sizeof(int) * E, st), "gate memset");
  const bool fused = d.x_dtype == FSMOE_BF16 && E <= 32 && NC % 4 == 0 && M % SC_JC == 0 &&
                     (reinterpret_cast<uintptr_t>(x) & 15) == 0 && !getenv("FSMOE_GATE_UNFUSED");
  // the approximate scores on the tensor cores (tcgen05 GEMM of x against the
  // bf16 hi / lo split of W); FSMOE_GATE_SIMT keeps the fp32 FFMA2 screen
  const bool tc = fused && 2 * NC <= TC_COLS && !getenv("FSMOE_GATE_SIMT");
  // (with the tensor-core screen, blocks NC.. zero Wtc's padding rows 2 NC..TC_COLS)
  pdl_launch(w_prep_kernel, tc ? TC_COLS - NC : NC, 256, 0, st, M, E, w_score, noisy ? E : 0, w_noise, w.W32, w.WT, w.wn,
                                    tc ? w.Wtc : nullptr);
  ::fsmoe::count_launch();
  if (tc) {
    double* nz = noise_out ? noise_out : w.noise;
    if (noisy) {
      // E_MAX sizes the exact phase's shared memory: E <= 8 (configs[2]) fits
      // four 256-thread blocks per SM, so a 32k-token grid runs in one wave
      if (E <= 8) launch_fused_tc<0, 8>(d, x, w.Wtc, w.P, w.WT, w.wn, nz, w.mask, pick_token, pick_expert, pick_weight, scores_out, spread_out, st);
      else if (E <= 16) launch_fused_tc<0, 16>(d, x, w.Wtc, w.P, w.WT, w.wn, nz, w.mask, pick_token, pick_expert, pick_weight, scores_out, spread_out, st);
      else launch_fused_tc<0, 32>(d, x, w.Wtc, w.P, w.WT, w.wn, nz, w.mask, pick_token, pick_expert, pick_weight, scores_out, spread_out, st);
    } else {
      launch_fused_tc<1, 32>(d, x, w.Wtc, w.P, w.WT, w.wn, nz, w.mask, pick_token, pick_expert, pick_weight, scores_out, spread_out, st);
    }
    return cuda_status(cudaGetLastError(), "fsmoe_gate(fused-tc)");
  }
  if (fused) {
    // the fused screen sums each token's FMA chain without splits: the same
    // bound with the split term kept (conservative)
    const double cBf = (M + AP_KS + 4.0) * 0x1.0p-24 * 1.01 + (M + 2.0) * 0x1.0p-53;
    double* nz = noise_out ? noise_out : w.noise;
    if (noisy) {
      if (E <= 16) launch_fused<0, 32, 16>(d, x, cBf, w.W32, w.WT, w.wn, nz, w.mask, pick_token, pick_expert, pick_weight, scores_out, spread_out, st);
      else launch_fused<0, 64, 32>(d, x, cBf, w.W32, w.WT, w.wn, nz, w.mask, pick_token, pick_expert, pick_weight, scores_out, spread_out, st);
    } else {
      launch_fused<1, 32, 32>(d, x, cBf, w.W32, w.WT, w.wn, nz, w.mask, pick_token, pick_expert, pick_weight, scores_out, spread_out, st);
    }
    if (getenv("FSMOE_GATE_DEBUG")) {  // candidate statistics (synchronises)
      std::vector<uint64_t> hm(static_cast<size_t>(T));
      cudaMemcpyAsync(hm.data(), w.mask, 8ull * T, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      long long tot = 0, mx = 0;
      for (uint64_t m : hm) {
        tot += __builtin_popcountll(m);
        mx = std::max<long long>(mx, __builtin_popcountll(m));
      }
      fprintf(stderr, "fsmoe gate: %lld candidates for %d tokens (max %lld per token)\n", tot, T, mx);
    }
    return cuda_status(cudaGetLastError(), "fsmoe_gate(fused)");
  }
  dim3 grid((T + AP_TOK - 1) / AP_TOK, (NC + AP_COL - 1) / AP_COL, AP_KS);
  switch (d.x_dtype) {
    case FSMOE_F64: approx_scores_kernel<0><<<grid, 64, 0, st>>>(x, T, M, w.W32, NC, w.part, w.xn2); break;
    case FSMOE_F32: approx_scores_kernel<1><<<grid, 64, 0, st>>>(x, T, M, w.W32, NC, w.part, w.xn2); break;
    default: approx_scores_kernel<2><<<grid, 64, 0, st>>>(x, T, M, w.W32, NC, w.part, w.xn2); break;
  }
  ::fsmoe::count_launch();
  if (noisy) {
    if (E <= 16) mt_kernel<16><<<(T + per_token_block(T) - 1) / per_token_block(T), per_token_block(T), 0, st>>>(T, E, d.seed, w.draws);
    else if (E <= 32) mt_kernel<32><<<(T + per_token_block(T) - 1) / per_token_block(T), per_token_block(T), 0, st>>>(T, E, d.seed, w.draws);
    else mt_kernel<64><<<(T + per_token_block(T) - 1) / per_token_block(T), per_token_block(T), 0, st>>>(T, E, d.seed, w.draws);
    ::fsmoe::count_launch();
  }
  // |s~ - s_ref| <= cB |x| |w|: fp32 rounding of x, w and the M-term FMA chain
  // (+ the split partial sums, + 1% slack), plus the reference's own fp64
  // sequential rounding.
  const double cB = (M + AP_KS + 4.0) * 0x1.0p-24 * 1.01 + (M + 2.0) * 0x1.0p-53;
  const long long pairs = static_cast<long long>(T) * E;
  const int pb = static_cast<int>((pairs + 255) / 256);
  if (noisy)
    bound_kernel<0><<<pb, 256, 0, st>>>(T, E, M, w.part, w.xn2, w.wn, cB, w.draws, w.noise, w.sapx,
                                        w.spapx, w.lo, w.hi);
  else
    bound_kernel<1><<<pb, 256, 0, st>>>(T, E, M, w.part, w.xn2, w.wn, cB, w.draws, w.noise, w.sapx,
                                        w.spapx, w.lo, w.hi);
  ::fsmoe::count_launch();
  cand_kernel<<<(T + per_token_block(T) - 1) / per_token_block(T), per_token_block(T), 0, st>>>(T, E, k, w.lo, w.hi, w.mask, w.lists, w.counts);
  ::fsmoe::count_launch();
  const PruneWsView v{w.WT, w.lists, w.counts, w.s_exact, w.sp_exact};
  switch (d.x_dtype * 2 + (noisy ? 0 : 1)) {
    case 0: launch_exact<0, 2>(x, T, M, E, v, st); break;
    case 1: launch_exact<0, 1>(x, T, M, E, v, st); break;
    case 2: launch_exact<1, 2>(x, T, M, E, v, st); break;
    case 3: launch_exact<1, 1>(x, T, M, E, v, st); break;
    case 4: launch_exact<2, 2>(x, T, M, E, v, st); break;
    default: launch_exact<2, 1>(x, T, M, E, v, st); break;
  }
  const int tb = (T + 127) / 128;
  if (noisy)
    final_kernel<0><<<tb, 128, 0, st>>>(T, E, k, w.mask, w.s_exact, w.sp_exact, w.sapx, w.spapx,
                                        w.noise, pick_token, pick_expert, pick_weight, scores_out,
                                        noise_out, spread_out);
  else
    final_kernel<1><<<tb, 128, 0, st>>>(T, E, k, w.mask, w.s_exact, w.sp_exact, w.sapx, w.spapx,
                                        w.noise, pick_token, pick_expert, pick_weight, scores_out,
                                        noise_out, spread_out);
  ::fsmoe::count_launch();
  return cuda_status(cudaGetLastError(), "fsmoe_gate(prune)");
}

}  // namespace fsmoe
