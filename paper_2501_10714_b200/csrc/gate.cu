// gate.cu — K1: the routing functions of fsmoe::run_gate
// (/root/reference/proj/src/workload.cpp:143-235) on the GPU, bit-exact in
// their selection:
//
//   rowdot_kernel      fp64 logits  s[t][c] = ((0 + x0*w0c) + x1*w1c) + ...
//                      (sequential j, separately rounded mul/add — the
//                      reference's matvec_row, workload.cpp:103-108). One
//                      thread owns one token and 16 output columns; the
//                      weight chunk is staged in shared memory.
//   token_select_kernel  noisy_topk / sigmoid_topk / cosine_topk per token:
//                      mt19937_64(seed+t) Box-Muller noise (85-99) added as
//                      n*log1p(exp(spread)) (101, 183-186), top-k with ties to
//                      the lowest index (111-121), masked softmax (123-133)
//                      or logistic (198), cosine scores (201-229).
//   ec_select_kernel   expert_choice (156-171): per expert an exact top-C
//                      over all tokens by radix select on order-preserving
//                      keys, ties to the lowest token, then the masked
//                      softmax over the C survivors in ascending token order.
//
// Compiled with --fmad=false: no multiply-add is ever contracted.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "capi_common.h"
#include "host_once.h"
#include "glibc_libm.cuh"
#include "kernels.h"
#include "route_common.cuh"

namespace fsmoe {
namespace {

using namespace fsmoe_dev;

constexpr int RD_THREADS = 128;  // tokens per block (one per thread)
constexpr int RD_CG = 8;         // output columns per thread (fewer when that leaves SMs idle)

struct RowdotJob {
  const double* W;  // W(j, c) = W[j*wsj + c*wsc]
  long long wsj, wsc;
  int NC;
  double* out;      // out[t*ost + c*osc]
  long long ost, osc;
};

// Token chunk staging type: bf16/fp32 values are exact in fp32, fp64 stays fp64.
template <int DT> struct Stage { using T = float; static constexpr int JC = 64; };
template <> struct Stage<0> { using T = double; static constexpr int JC = 32; };

// out[t][c] = sum_j x[t][j] * W(j, c), sequential j, separately rounded
// mul/add (matvec_row, workload.cpp:103-108). One thread = one token x 8
// columns; blockIdx.y walks the column groups of job a, then of job b, so the
// noisy gate's two projections (x W_g, x W_noise) are one launch. The token
// chunk is staged transposed in smem (conflict-free reads), the weight chunk
// as broadcast rows.
template <int DT, int CG>
__global__ void __launch_bounds__(RD_THREADS)
    rowdot_kernel(const void* __restrict__ x, int T, int M, RowdotJob ja, RowdotJob jb,
                  int groups_a) {
  using ST = typename Stage<DT>::T;
  constexpr int JC = Stage<DT>::JC;
  __shared__ ST xs[JC][RD_THREADS + 1];  // +1: conflict-free transposed stores
  __shared__ __align__(16) double ws[JC][CG];
  const bool second = static_cast<int>(blockIdx.y) >= groups_a;
  const RowdotJob& J = second ? jb : ja;
  const int c0 = (second ? blockIdx.y - groups_a : blockIdx.y) * CG;
  const int t0 = blockIdx.x * RD_THREADS;
  const int t = t0 + threadIdx.x;
  double acc[CG];
#pragma unroll
  for (int c = 0; c < CG; ++c) acc[c] = 0.0;
  for (int j0 = 0; j0 < M; j0 += JC) {
    const int jn = (M - j0) < JC ? (M - j0) : JC;
    __syncthreads();
    for (int i = threadIdx.x; i < JC * CG; i += RD_THREADS) {
      int jj = i / CG, cc = i % CG;
      int c = c0 + cc;
      ws[jj][cc] = (jj < jn && c < J.NC) ? J.W[(j0 + jj) * J.wsj + c * J.wsc] : 0.0;
    }
    // coalesced: consecutive threads read consecutive columns of one token row
    for (int i = threadIdx.x; i < RD_THREADS * JC; i += RD_THREADS) {
      const int tt = i / JC, jj = i % JC;
      if (jj < jn && t0 + tt < T)
        xs[jj][tt] = static_cast<ST>(load_as_double<DT>(x, static_cast<long long>(t0 + tt) * M + j0 + jj));
    }
    __syncthreads();
    if (t < T) {
#pragma unroll 4
      for (int jj = 0; jj < jn; ++jj) {
        const double xv = static_cast<double>(xs[jj][threadIdx.x]);
        if constexpr (CG >= 2) {
          const double2* w2 = reinterpret_cast<const double2*>(ws[jj]);
#pragma unroll
          for (int c = 0; c < CG / 2; ++c) {
            const double2 w = w2[c];
            acc[2 * c] = mul_add_rn(acc[2 * c], xv, w.x);
            acc[2 * c + 1] = mul_add_rn(acc[2 * c + 1], xv, w.y);
          }
        } else {
          acc[0] = mul_add_rn(acc[0], xv, ws[jj][0]);
        }
      }
    }
  }
  if (t < T) {
#pragma unroll
    for (int c = 0; c < CG; ++c)
      if (c0 + c < J.NC) J.out[t * J.ost + (c0 + c) * J.osc] = acc[c];
  }
}

// rowdot_kernel for bf16 tokens with M % 8 == 0 and 16-byte rows: the next
// chunk's token rows (uint4 loads) and weight values are loaded into
// registers while the current chunk is summed, so the global-load latency
// that stalls the staged copy (ncu: long scoreboard) overlaps the fp64
// chains. Same per-thread operation order as rowdot_kernel.
template <int CG>
__global__ void __launch_bounds__(RD_THREADS)
    rowdot_pf_kernel(const __nv_bfloat16* __restrict__ x, int T, int M, RowdotJob ja, RowdotJob jb,
                     int groups_a) {
  constexpr int JC = 64;
  constexpr int XV = RD_THREADS * JC / 8 / RD_THREADS;      // uint4 per thread per chunk (8)
  constexpr int WV = (JC * CG + RD_THREADS - 1) / RD_THREADS;  // weights per thread per chunk
  __shared__ float xs[JC][RD_THREADS + 1];
  __shared__ __align__(16) double ws[JC][CG];
  const bool second = static_cast<int>(blockIdx.y) >= groups_a;
  const RowdotJob& J = second ? jb : ja;
  const int c0 = (second ? blockIdx.y - groups_a : blockIdx.y) * CG;
  const int t0 = blockIdx.x * RD_THREADS;
  const int t = t0 + threadIdx.x;
  uint4 xr[XV];
  double wr[WV];
  auto prefetch = [&](int j0) {
#pragma unroll
    for (int u = 0; u < XV; ++u) {
      const int idx = threadIdx.x + u * RD_THREADS;
      const int tt = idx / (JC / 8), q = idx % (JC / 8);
      const int j = j0 + q * 8;
      xr[u] = (t0 + tt < T && j < M)
                  ? __ldg(reinterpret_cast<const uint4*>(x + static_cast<long long>(t0 + tt) * M + j))
                  : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < WV; ++u) {
      const int i = threadIdx.x + u * RD_THREADS;
      const int jj = i / CG, c = c0 + i % CG;
      wr[u] = (i < JC * CG && j0 + jj < M && c < J.NC) ? J.W[(j0 + jj) * J.wsj + c * J.wsc] : 0.0;
    }
  };
  double acc[CG];
#pragma unroll
  for (int c = 0; c < CG; ++c) acc[c] = 0.0;
  prefetch(0);
  for (int j0 = 0; j0 < M; j0 += JC) {
    const int jn = (M - j0) < JC ? (M - j0) : JC;
    __syncthreads();  // the previous chunk's reads of xs / ws are done
#pragma unroll
    for (int u = 0; u < XV; ++u) {
      const int idx = threadIdx.x + u * RD_THREADS;
      const int tt = idx / (JC / 8), q = idx % (JC / 8);
      const uint32_t w4[4] = {xr[u].x, xr[u].y, xr[u].z, xr[u].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        xs[q * 8 + 2 * e][tt] = __uint_as_float(w4[e] << 16);
        xs[q * 8 + 2 * e + 1][tt] = __uint_as_float(w4[e] & 0xffff0000u);
      }
    }
#pragma unroll
    for (int u = 0; u < WV; ++u) {
      const int i = threadIdx.x + u * RD_THREADS;
      if (i < JC * CG) ws[i / CG][i % CG] = wr[u];
    }
    __syncthreads();
    if (j0 + JC < M) prefetch(j0 + JC);
    if (t < T) {
#pragma unroll 4
      for (int jj = 0; jj < jn; ++jj) {
        const double xv = static_cast<double>(xs[jj][threadIdx.x]);
        if constexpr (CG >= 2) {
          const double2* w2 = reinterpret_cast<const double2*>(ws[jj]);
#pragma unroll
          for (int c = 0; c < CG / 2; ++c) {
            const double2 w = w2[c];
            acc[2 * c] = mul_add_rn(acc[2 * c], xv, w.x);
            acc[2 * c + 1] = mul_add_rn(acc[2 * c + 1], xv, w.y);
          }
        } else {
          acc[0] = mul_add_rn(acc[0], xv, ws[jj][0]);
        }
      }
    }
  }
  if (t < T) {
#pragma unroll
    for (int c = 0; c < CG; ++c)
      if (c0 + c < J.NC) J.out[t * J.ost + (c0 + c) * J.osc] = acc[c];
  }
}

// ---------------------------------------------------------------- noise --

constexpr uint64_t MT_A = 0xB5026F5AA96619E9ULL;
constexpr uint64_t MT_UM = 0xFFFFFFFF80000000ULL;
constexpr uint64_t MT_LM = 0x000000007FFFFFFFULL;

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

__device__ __forceinline__ uint64_t mt_seed_step(uint64_t prev, uint64_t i) {
  return 6364136223846793005ULL * (prev ^ (prev >> 62)) + i;
}

// First n outputs of std::mt19937_64(seed) (libstdc++ twists all 312 words on
// the first draw; output i < 156 only needs seed words i, i+1, i+156).
template <int MAXN>
__device__ void mt64_outputs(uint64_t seed, int n, uint64_t* outv) {
  if constexpr (MAXN <= 156) {
    uint64_t lo[MAXN + 1];
    uint64_t w = seed;
    lo[0] = w;
    for (int i = 1; i < 156 + n; ++i) {
      w = mt_seed_step(w, static_cast<uint64_t>(i));
      if (i <= n) lo[i] = w;
      if (i >= 156) {
        int o = i - 156;
        uint64_t y = (lo[o] & MT_UM) | (lo[o + 1] & MT_LM);
        uint64_t z = w ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
        outv[o] = mt_temper(z);
      }
    }
  } else {
    uint64_t mt[312];
    mt[0] = seed;
    for (int i = 1; i < 312; ++i) mt[i] = mt_seed_step(mt[i - 1], static_cast<uint64_t>(i));
    int idx = 312;
    for (int o = 0; o < n; ++o) {
      if (idx >= 312) {
        for (int i = 0; i < 312; ++i) {
          uint64_t y = (mt[i] & MT_UM) | (mt[(i + 1) % 312] & MT_LM);
          mt[i] = mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
        }
        idx = 0;
      }
      outv[o] = mt_temper(mt[idx++]);
    }
  }
}

// NormalDraws::next (workload.cpp:90-95).
__device__ __forceinline__ double box_muller(uint64_t a, uint64_t b) {
  double u1 = __dmul_rn(__dadd_rn(static_cast<double>(a >> 11), 0.5), 0x1.0p-53);
  double u2 = __dmul_rn(__dadd_rn(static_cast<double>(b >> 11), 0.5), 0x1.0p-53);
  double two_pi = 2.0 * 3.141592653589793238462643383279502884;
  return fsmoe_libm::gl_normal(u1, u2);
}

// ------------------------------------------------------- token selection --

template <int KIND, int MAX_E>
__global__ void __launch_bounds__(128)
    token_select_kernel(int T, int E, int k, uint64_t seed, const double* __restrict__ raw,
                        const double* __restrict__ spread, int P,
                        const double* __restrict__ w_score, const double* __restrict__ enorm,
                        int* __restrict__ pick_token, int* __restrict__ pick_expert,
                        double* __restrict__ pick_weight, double* __restrict__ scores_out,
                        double* __restrict__ noise_out, int* __restrict__ status) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  double s[MAX_E];
  if (KIND == 0) {  // noisy_topk
    uint64_t draws[2 * MAX_E];
    mt64_outputs<2 * MAX_E>(seed + static_cast<uint64_t>(t), 2 * E, draws);
    for (int e = 0; e < E; ++e) {
      double n = box_muller(draws[2 * e], draws[2 * e + 1]);
      double sp = fsmoe_libm::gl_softplus(spread[static_cast<long long>(t) * E + e]);
      s[e] = __dadd_rn(raw[static_cast<long long>(t) * E + e], __dmul_rn(n, sp));
      if (noise_out) noise_out[static_cast<long long>(t) * E + e] = n;
    }
  } else if (KIND == 1) {  // sigmoid_topk
    for (int e = 0; e < E; ++e) s[e] = raw[static_cast<long long>(t) * E + e];
  } else {  // cosine_topk: raw = projected token (T x P)
    const double* q = raw + static_cast<long long>(t) * P;
    double pnorm = 0.0;
    for (int p = 0; p < P; ++p) pnorm = mul_add_rn(pnorm, q[p], q[p]);
    if (pnorm == 0.0) {
      if (status) atomicOr(status, t == 0 ? 3 : 1);
      return;
    }
    for (int e = 0; e < E; ++e) {
      double dot = 0.0;
      for (int p = 0; p < P; ++p) dot = mul_add_rn(dot, q[p], w_score[static_cast<long long>(p) * E + e]);
      double en = enorm[e];
      if (en == 0.0) {
        if (status) atomicOr(status, 4);
        return;
      }
      s[e] = __ddiv_rn(dot, __dsqrt_rn(__dmul_rn(pnorm, en)));
    }
  }
  if (scores_out)
    for (int e = 0; e < E; ++e) scores_out[static_cast<long long>(t) * E + e] = s[e];

  // top-k: repeatedly take the max with ties to the lowest index, then
  // report the kept set in ascending index order.
  uint32_t sel[(MAX_E + 31) / 32];
  for (int i = 0; i < (MAX_E + 31) / 32; ++i) sel[i] = 0;
  for (int j = 0; j < k; ++j) {
    int best = -1;
    for (int e = 0; e < E; ++e) {
      if (sel[e >> 5] & (1u << (e & 31))) continue;
      if (best < 0 || s[e] > s[best]) best = e;
    }
    sel[best >> 5] |= 1u << (best & 31);
  }
  int keep[MAX_E];
  int nk = 0;
  for (int e = 0; e < E; ++e)
    if (sel[e >> 5] & (1u << (e & 31))) keep[nk++] = e;

  const long long base = static_cast<long long>(t) * k;
  if (KIND == 1) {
    for (int j = 0; j < k; ++j) {
      pick_token[base + j] = t;
      pick_expert[base + j] = keep[j];
      pick_weight[base + j] = __ddiv_rn(1.0, __dadd_rn(1.0, fsmoe_libm::gl_exp(-s[keep[j]])));
    }
    return;
  }
  double mx = s[keep[0]];
  for (int j = 0; j < k; ++j) mx = (mx < s[keep[j]]) ? s[keep[j]] : mx;
  double z = 0.0;
  for (int j = 0; j < k; ++j) z = __dadd_rn(z, fsmoe_libm::gl_exp(__dsub_rn(s[keep[j]], mx)));
  for (int j = 0; j < k; ++j) {
    pick_token[base + j] = t;
    pick_expert[base + j] = keep[j];
    pick_weight[base + j] = __ddiv_rn(fsmoe_libm::gl_exp(__dsub_rn(s[keep[j]], mx)), z);
  }
}

template <int KIND>
void launch_select(cudaStream_t st, int T, int E, int k, uint64_t seed, const double* raw,
                   const double* spread, int P, const double* w_score, const double* enorm,
                   int* pt, int* pe, double* pw, double* scores_out, double* noise_out,
                   int* status) {
  const int tpb = per_token_block(T);
  const int blocks = (T + tpb - 1) / tpb;
  if (E <= 16)
    token_select_kernel<KIND, 16><<<blocks, tpb, 0, st>>>(T, E, k, seed, raw, spread, P, w_score,
                                                          enorm, pt, pe, pw, scores_out, noise_out, status);
  else if (E <= 64)
    token_select_kernel<KIND, 64><<<blocks, tpb, 0, st>>>(T, E, k, seed, raw, spread, P, w_score,
                                                          enorm, pt, pe, pw, scores_out, noise_out, status);
  else
    token_select_kernel<KIND, 256><<<blocks, tpb, 0, st>>>(T, E, k, seed, raw, spread, P, w_score,
                                                           enorm, pt, pe, pw, scores_out, noise_out, status);
  ::fsmoe::count_launch();
}

// enorm[e] = sum_p W[p][e]^2 (same order as the reference's per-token loop).
__global__ void expert_norm_kernel(int P, int E, const double* __restrict__ w, double* __restrict__ en) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double a = 0.0;
  for (int p = 0; p < P; ++p) {
    double v = w[static_cast<long long>(p) * E + e];
    a = mul_add_rn(a, v, v);
  }
  en[e] = a;
}

// ------------------------------------------------------- expert choice --

constexpr int EC_THREADS = 1024;

__device__ __forceinline__ int block_excl_scan(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < (EC_THREADS / 32) ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_tot[lane] = w;  // inclusive
  }
  __syncthreads();
  int before = wid > 0 ? warp_tot[wid - 1] : 0;
  total = warp_tot[EC_THREADS / 32 - 1];
  __syncthreads();
  return before + x - v;
}

// scores: experts x tokens (row e contiguous). One block per expert.
__global__ void __launch_bounds__(EC_THREADS)
    ec_select_kernel(int T, int E, int C, const double* __restrict__ scores,
                     int* __restrict__ pick_token, int* __restrict__ pick_expert,
                     double* __restrict__ pick_weight) {
  __shared__ int hist[256];
  __shared__ int warp_tot[32];
  __shared__ int s_digit, s_need;
  __shared__ double s_red[32];
  __shared__ double s_z;
  const int e = blockIdx.x;
  const double* se = scores + static_cast<long long>(e) * T;

  // ---- radix select: key of the C-th largest score
  uint64_t prefix = 0, mask = 0;
  int need = C;  // how many still to take among keys matching `prefix`
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += EC_THREADS) hist[i] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < T; t += EC_THREADS) {
      uint64_t key = order_key(se[t]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xFF], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0, d = 255;
      for (; d > 0; --d) {
        if (acc + hist[d] >= need) break;
        acc += hist[d];
      }
      s_digit = d;
      s_need = need - acc;
    }
    __syncthreads();
    prefix |= static_cast<uint64_t>(s_digit) << shift;
    mask |= 0xFFULL << shift;
    need = s_need;
    __syncthreads();
  }
  const uint64_t thr = prefix;  // keys > thr all kept; `need` of the == thr ones (lowest tokens)

  // ---- ordered compaction in ascending token order
  int base_sel = 0, base_tie = 0;
  double local_max = -__longlong_as_double(0x7FF0000000000000LL);  // -inf
  for (int t0 = 0; t0 < T; t0 += EC_THREADS) {
    int t = t0 + threadIdx.x;
    uint64_t key = t < T ? order_key(se[t]) : 0;
    int tie = (t < T && key == thr) ? 1 : 0;
    int tot_tie;
    int tie_rank = base_tie + block_excl_scan(tie, warp_tot, tot_tie);
    int flag = (t < T) && (key > thr || (tie && tie_rank < need)) ? 1 : 0;
    int tot_sel;
    int pos = base_sel + block_excl_scan(flag, warp_tot, tot_sel);
    if (flag) {
      long long pi = static_cast<long long>(e) * C + pos;
      pick_token[pi] = t;
      pick_expert[pi] = e;
      pick_weight[pi] = se[t];  // score for now
      local_max = se[t] > local_max ? se[t] : local_max;
    }
    base_tie += tot_tie;
    base_sel += tot_sel;
  }
  // ---- masked softmax over the C kept scores (workload.cpp:123-133)
  for (int o = 16; o > 0; o >>= 1) {
    double y = __shfl_xor_sync(0xffffffffu, local_max, o);
    local_max = y > local_max ? y : local_max;
  }
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = local_max;
  __syncthreads();
  double mx = s_red[0];
  for (int i = 1; i < EC_THREADS / 32; ++i) mx = s_red[i] > mx ? s_red[i] : mx;
  double* wts = pick_weight + static_cast<long long>(e) * C;
  __syncthreads();
  for (int j = threadIdx.x; j < C; j += EC_THREADS) wts[j] = fsmoe_libm::gl_exp(__dsub_rn(wts[j], mx));
  __threadfence_block();
  __syncthreads();
  if (threadIdx.x == 0) {
    double z = 0.0;
    for (int j = 0; j < C; ++j) z = __dadd_rn(z, wts[j]);
    s_z = z;
  }
  __syncthreads();
  const double z = s_z;
  for (int j = threadIdx.x; j < C; j += EC_THREADS) wts[j] = __ddiv_rn(wts[j], z);
}

}  // namespace

// ---------------------------------------------------------------- host ----

void cosine_enorm(int P, int E, const double* w, double* en, cudaStream_t st) {
  expert_norm_kernel<<<(E + 127) / 128, 128, 0, st>>>(P, E, w, en); ::fsmoe::count_launch();
}

int gate_launch(const fsmoe_gate_desc& d, const void* x, const double* w_score,
                const double* w_noise, const double* proj, int* pick_token, int* pick_expert,
                double* pick_weight, double* scores_out, double* noise_out, double* spread_out,
                double* proj_out, int* d_status, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int T = d.tokens, M = d.model_dim, E = d.score_cols, k = d.top_k;
  // workspace carve-up (see fsmoe_gate_workspace_size)
  char* w = static_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* p = w;
    w += (bytes + 255) & ~size_t(255);
    return reinterpret_cast<double*>(p);
  };
  // columns per thread: 8 independent fp64 chains per thread, unless that
  // leaves the grid too small to fill the GPU (few tokens or columns: the
  // expert-choice logits, E = 8) -- then fewer chains and more threads
  auto rowdot2 = [&](RowdotJob a, RowdotJob b) {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long tb = (T + RD_THREADS - 1) / RD_THREADS;
    auto blocks = [&](int cg) {
      return tb * ((a.NC + cg - 1) / cg + (b.W ? (b.NC + cg - 1) / cg : 0));
    };
    int cg = RD_CG;
    while (cg > 1 && blocks(cg) < 2LL * sms) cg /= 2;
    auto go = [&](auto cgc) {
      constexpr int CG = decltype(cgc)::value;
      const int ga = (a.NC + CG - 1) / CG, gb = b.W ? (b.NC + CG - 1) / CG : 0;
      dim3 grid(static_cast<unsigned>(tb), ga + gb);
      switch (d.x_dtype) {
        case FSMOE_F64: rowdot_kernel<0, CG><<<grid, RD_THREADS, 0, st>>>(x, T, M, a, b, ga); break;
        case FSMOE_F32: rowdot_kernel<1, CG><<<grid, RD_THREADS, 0, st>>>(x, T, M, a, b, ga); break;
        default:
          if (M % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0)
            rowdot_pf_kernel<CG><<<grid, RD_THREADS, 0, st>>>(static_cast<const __nv_bfloat16*>(x), T, M, a, b, ga);
          else
            rowdot_kernel<2, CG><<<grid, RD_THREADS, 0, st>>>(x, T, M, a, b, ga);
          break;
      }
    };
    if (cg == 8) go(std::integral_constant<int, 8>{});
    else if (cg == 4) go(std::integral_constant<int, 4>{});
    else if (cg == 2) go(std::integral_constant<int, 2>{});
    else go(std::integral_constant<int, 1>{});
    ::fsmoe::count_launch();
  };
  auto rowdot = [&](const double* W, long long wsj, long long wsc, int NC, double* out,
                    long long ost, long long osc) {
    rowdot2(RowdotJob{W, wsj, wsc, NC, out, ost, osc}, RowdotJob{nullptr, 0, 0, 0, nullptr, 0, 0});
  };
  (void)ws_bytes;
  const bool exhaustive = getenv("FSMOE_GATE_EXHAUSTIVE") != nullptr;
  if (!exhaustive && gate_prune_applicable(d))
    return gate_prune_launch(d, x, w_score, w_noise, pick_token, pick_expert, pick_weight,
                             scores_out, noise_out, spread_out, ws, st);
  switch (d.kind) {
    case FSMOE_GATE_NOISY_TOPK: {
      double* raw = take(sizeof(double) * T * E);
      double* spread = spread_out ? spread_out : take(sizeof(double) * T * E);
      rowdot2(RowdotJob{w_score, E, 1, E, raw, E, 1}, RowdotJob{w_noise, E, 1, E, spread, E, 1});
      launch_select<0>(st, T, E, k, d.seed, raw, spread, 0, nullptr, nullptr, pick_token,
                       pick_expert, pick_weight, scores_out, noise_out, d_status);
      break;
    }
    case FSMOE_GATE_SIGMOID_TOPK: {
      double* raw = scores_out ? scores_out : take(sizeof(double) * T * E);
      rowdot(w_score, E, 1, E, raw, E, 1);
      launch_select<1>(st, T, E, k, d.seed, raw, nullptr, 0, nullptr, nullptr, pick_token,
                       pick_expert, pick_weight, nullptr, nullptr, d_status);
      break;
    }
    case FSMOE_GATE_COSINE_TOPK: {
      const int P = d.proj_rows;
      double* q = proj_out ? proj_out : take(sizeof(double) * T * P);
      double* en = take(sizeof(double) * E);
      // proj[p] = sum_j P[p][j] * x[j]  -> W(j, p) = P[p*M + j]
      rowdot(proj, 1, M, P, q, P, 1);
      expert_norm_kernel<<<(E + 127) / 128, 128, 0, st>>>(P, E, w_score, en); ::fsmoe::count_launch();
      launch_select<2>(st, T, E, k, d.seed, q, nullptr, P, w_score, en, pick_token, pick_expert,
                       pick_weight, scores_out, nullptr, d_status);
      break;
    }
    case FSMOE_GATE_EXPERT_CHOICE: {
      double* sc = scores_out ? scores_out : take(sizeof(double) * T * E);  // E x T
      rowdot(w_score, E, 1, E, sc, 1, T);
      ec_select_kernel<<<E, EC_THREADS, 0, st>>>(T, E, k, sc, pick_token, pick_expert,
                                                 pick_weight); ::fsmoe::count_launch();
      break;
    }
    default:
      return config_error("gate: unknown gate kind");
  }
  return cuda_status(cudaGetLastError(), "fsmoe_gate");
}

size_t gate_workspace_bytes(const fsmoe_gate_desc& d) {
  const size_t T = d.tokens > 0 ? d.tokens : 0, E = d.score_cols > 0 ? d.score_cols : 0;
  auto r = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t prune = gate_prune_applicable(d) ? gate_prune_workspace_bytes(d) : 0;
  switch (d.kind) {
    case FSMOE_GATE_NOISY_TOPK: return std::max(r(8 * T * E) * 2, prune);
    case FSMOE_GATE_SIGMOID_TOPK: return std::max(r(8 * T * E), prune);
    case FSMOE_GATE_COSINE_TOPK: return r(8 * T * (d.proj_rows > 0 ? d.proj_rows : 0)) + r(8 * E);
    case FSMOE_GATE_EXPERT_CHOICE: return r(8 * T * E);
    default: return 0;
  }
}

}  // namespace fsmoe

// ------------------------------------------------------------ libm audit --
// fsmoe_libm_eval: the gate's transcendental functions on the device, either
// the glibc restatement the gate uses (impl 0, glibc_libm.cuh) or CUDA's own
// libm (impl 1), for the parity audit against the host's glibc
// (tests/test_noise_exact_gpu.py).
namespace {
__global__ void libm_eval_kernel(int fn, int impl, const double* __restrict__ x,
                                 const double* __restrict__ x2, double* __restrict__ y, long long n) {
  using namespace fsmoe_libm;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double a = x[i];
    double r = 0.0;
    if (impl == 0) {
      switch (fn) {
        case 0: r = gl_log(a); break;
        case 1: r = gl_exp(a); break;
        case 2: r = gl_log1p(a); break;
        case 3: r = gl_cos(a); break;
        case 4: r = gl_normal(a, x2[i]); break;
        default: r = gl_softplus(a); break;
      }
    } else {
      const double two_pi = 2.0 * 3.141592653589793238462643383279502884;
      switch (fn) {
        case 0: r = log(a); break;
        case 1: r = exp(a); break;
        case 2: r = log1p(a); break;
        case 3: r = cos(a); break;
        case 4: r = __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, log(a))), cos(__dmul_rn(two_pi, x2[i]))); break;
        default: r = log1p(exp(a)); break;
      }
    }
    y[i] = r;
  }
}
}  // namespace

extern "C" int fsmoe_libm_eval(int fn, int impl, const double* x, const double* x2, double* y,
                               long long n, void* stream) {
  if (fn < 0 || fn > 5 || impl < 0 || impl > 1 || (n > 0 && (!x || !y)) || (fn == 4 && n > 0 && !x2))
    return fsmoe::config_error("libm eval: fn in [0, 5], impl 0 | 1, x and y required (x2 for fn 4)");
  if (n <= 0) return FSMOE_OK;
  const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
  libm_eval_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(fn, impl, x, x2, y, n);
  fsmoe::count_launch();
  return fsmoe::cuda_status(cudaGetLastError(), "fsmoe_libm_eval");
}
