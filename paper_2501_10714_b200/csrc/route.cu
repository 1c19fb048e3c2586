// route.cu — K2 capacity assignment, K3 dispatch (Order), K5 combine
// (I-Order) and their backward, for /root/reference/proj/src/workload.cpp:
//   dispatch_tokens 237-264  ->  assign_{count,rank}_kernel + dispatch_kernel
//   combine_tokens  266-282  ->  combine_kernel
//
// Assignment is a stable per-expert rank over the pick sequence (the
// reference's sequential fill loop): ranks inside 32-pick warp windows come
// from __match_any_sync, across warps/rounds from shared-memory prefix sums,
// across tiles from per-tile expert histograms. No atomics decide order, so
// slot_of_pick / fill / dropped are bit-identical to the reference.
//
// Permutation kernels move one buffer row per warp with 16-byte vector
// accesses (rows are contiguous, so each warp-instruction covers 512 B).
// Combine / dispatch-backward gather the (<= k) rows of a token and reduce in
// pick order; fp64 uses separately rounded multiply and add exactly as the
// reference (y[t] += w * buf[slot]).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <atomic>
#include <type_traits>
#include <cstdlib>

#include "host_once.h"
#include "capi_common.h"
#include "kernels.h"
#include "route_common.cuh"
#include "sm100.cuh"

namespace fsmoe {
namespace {

using namespace fsmoe_dev;

constexpr int AS_THREADS = 1024;
constexpr int AS_TILE = AS_THREADS;  // picks per tile (one round per block)
constexpr int AS_MAX_E = 256;
constexpr int AS_CNT_CACHE = 2048;  // tile histograms kept in shared memory (ints)

// cnt[tile][e] = picks of expert e inside the tile; flags bad picks.
__global__ void __launch_bounds__(AS_THREADS)
    assign_count_kernel(long long P, const int* __restrict__ ptok, const int* __restrict__ pexp,
                        int T, int E, int* __restrict__ cnt, int* __restrict__ status,
                        int* __restrict__ pick_of_slot, long long n_slots) {
  fsmoe_dev::pdl_enter();
  // every slot starts empty (assign_rank, the next kernel, fills the kept ones)
  for (long long i = blockIdx.x * static_cast<long long>(AS_THREADS) + threadIdx.x; i < n_slots;
       i += static_cast<long long>(gridDim.x) * AS_THREADS)
    pick_of_slot[i] = -1;
  __shared__ int h[AS_MAX_E];
  for (int i = threadIdx.x; i < E; i += AS_THREADS) h[i] = 0;
  __syncthreads();
  const long long base = static_cast<long long>(blockIdx.x) * AS_TILE;
  for (int i = threadIdx.x; i < AS_TILE; i += AS_THREADS) {
    long long p = base + i;
    if (p >= P) break;
    int e = pexp[p], t = ptok[p];
    if (e < 0 || e >= E || t < 0 || t >= T) {
      if (status) atomicOr(status, 8);
      continue;
    }
    atomicAdd(&h[e], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += AS_THREADS) cnt[blockIdx.x * E + i] = h[i];
}

__global__ void __launch_bounds__(AS_THREADS)
    assign_rank_kernel(long long P, const int* __restrict__ pexp, int E, long long C,
                       const int* __restrict__ cnt, int ntiles, int* __restrict__ slot_of_pick,
                       int* __restrict__ pick_of_slot, long long* __restrict__ fill,
                       long long* __restrict__ dropped) {
  fsmoe_dev::pdl_enter();
  __shared__ int base[AS_MAX_E];
  __shared__ int wc[AS_THREADS / 32][AS_MAX_E];
  __shared__ int cs[AS_CNT_CACHE];
  __shared__ long long drop_acc;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // every tile's histogram in one parallel load (not a dependent load per
  // tile), then per-expert prefix / totals from shared memory
  const int ncnt = ntiles * E;
  const bool cached = ncnt <= AS_CNT_CACHE;
  if (cached)
    for (int i = threadIdx.x; i < ncnt; i += AS_THREADS) cs[i] = cnt[i];
  if (threadIdx.x == 0) drop_acc = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += AS_THREADS) {
    int b = 0;
    long long tot = 0;
    for (int tl = 0; tl < ntiles; ++tl) {
      const int v = cached ? cs[tl * E + e] : cnt[tl * E + e];
      if (tl < static_cast<int>(blockIdx.x)) b += v;
      tot += v;
    }
    base[e] = b;
    if (blockIdx.x == 0) {
      fill[e] = tot < C ? tot : C;
      if (tot > C) atomicAdd(reinterpret_cast<unsigned long long*>(&drop_acc),
                             static_cast<unsigned long long>(tot - C));
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) *dropped = drop_acc;
  const long long tile0 = static_cast<long long>(blockIdx.x) * AS_TILE;
  for (int r = 0; r < AS_TILE / AS_THREADS; ++r) {
    for (int i = threadIdx.x; i < (AS_THREADS / 32) * E; i += AS_THREADS) wc[i / E][i % E] = 0;
    __syncthreads();
    long long p = tile0 + static_cast<long long>(r) * AS_THREADS + threadIdx.x;
    int e = -1;
    if (p < P) {
      e = pexp[p];
      if (e < 0 || e >= E) e = -1;
    }
    unsigned same = __match_any_sync(0xffffffffu, e);
    int in_warp = __popc(same & ((1u << lane) - 1u));
    if (e >= 0 && in_warp == 0) wc[wid][e] = __popc(same);
    __syncthreads();
    if (e >= 0) {
      int rank = base[e] + in_warp;
      for (int w = 0; w < wid; ++w) rank += wc[w][e];
      if (rank < C) {
        long long slot = static_cast<long long>(e) * C + rank;
        slot_of_pick[p] = static_cast<int>(slot);
        pick_of_slot[slot] = static_cast<int>(p);
      } else {
        slot_of_pick[p] = -1;
      }
    } else if (p < P) {
      slot_of_pick[p] = -1;
    }
    __syncthreads();
    for (int ee = threadIdx.x; ee < E; ee += AS_THREADS) {
      int s = 0;
      for (int w = 0; w < AS_THREADS / 32; ++w) s += wc[w][ee];
      base[ee] += s;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------ token index (CSR) --

__global__ void tok_token_major_kernel(int T, int k, int* __restrict__ ptr, int* __restrict__ idx) {
  fsmoe_dev::pdl_enter();
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i <= T) ptr[i] = static_cast<int>(i * k);
  if (i < static_cast<long long>(T) * k) idx[i] = static_cast<int>(i);
}

__global__ void tok_count_kernel(long long P, const int* __restrict__ ptok, int T,
                                 int* __restrict__ cnt) {
  long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (p < P) {
    int t = ptok[p];
    if (t >= 0 && t < T) atomicAdd(&cnt[t], 1);
  }
}

// Single-block exclusive scan of n ints (n up to a few 1e5; used once per layer).
__global__ void __launch_bounds__(1024) scan_excl_kernel(const int* __restrict__ in, int n,
                                                         int* __restrict__ out) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int b = 0; b < n; b += 1024) {
    int i = b + threadIdx.x;
    int v = i < n ? in[i] : 0;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = warp_tot[lane];
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;
    }
    __syncthreads();
    int before = (wid > 0 ? warp_tot[wid - 1] : 0) + carry;
    if (i < n) out[i] = before + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_tot[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

__global__ void tok_place_kernel(long long P, const int* __restrict__ ptok, int T,
                                 const int* __restrict__ ptr, int* __restrict__ cursor,
                                 int* __restrict__ idx) {
  long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (p < P) {
    int t = ptok[p];
    if (t >= 0 && t < T) idx[ptr[t] + atomicAdd(&cursor[t], 1)] = static_cast<int>(p);
  }
}

// Per-token insertion sort: lists are short (<= experts), restores pick order.
__global__ void tok_sort_kernel(int T, const int* __restrict__ ptr, int* __restrict__ idx) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  int a = ptr[t], b = ptr[t + 1];
  for (int i = a + 1; i < b; ++i) {
    int v = idx[i], j = i - 1;
    while (j >= a && idx[j] > v) {
      idx[j + 1] = idx[j];
      --j;
    }
    idx[j + 1] = v;
  }
}

// --------------------------------------------------------------- dispatch --

// buffers[row(s)] = x[token(pick_of_slot[s])] or 0; one warp per slot row.
template <typename V>
__global__ void __launch_bounds__(256)
    dispatch_kernel(long long n_slots, int row_vecs, int E, long long C, int chunks,
                    const int* __restrict__ pick_of_slot, const int* __restrict__ ptok,
                    const V* __restrict__ x, const PeerRows buf, const RowRange rr) {
  fsmoe_dev::pdl_enter();
  const long long s = blockIdx.x * 8LL + (threadIdx.x >> 5);
  if (s >= n_slots || !in_range(rr, s)) return;
  const int lane = threadIdx.x & 31;
  const int p = pick_of_slot[s];
  V* dst = reinterpret_cast<V*>(
      peer_row(buf, slot_row(s, E, C, chunks), static_cast<long long>(row_vecs) * sizeof(V)));
  if (p < 0) {
    V z;
    memset(&z, 0, sizeof(V));
    for (int i = lane; i < row_vecs; i += 32) dst[i] = z;
    return;
  }
  const V* src = x + static_cast<long long>(ptok[p]) * row_vecs;
  for (int i = lane; i < row_vecs; i += 32) dst[i] = src[i];
}

// Row moves through the TMA engine: lane r of the block's warp owns row r,
// bulk-loads its source row (global -> shared) and bulk-stores it to the
// destination (local or a peer's buffer over NVLink). One instruction moves a
// whole row, so the LSU / register path that limits the warp-per-row copy
// (long-scoreboard + lg_throttle stalls, ncu) drops out.
constexpr int BK_ROWS = 32;  // rows per group (one per lane)

__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem_src))), "r"(bytes)
               : "memory");
}

__global__ void __launch_bounds__(32)
    dispatch_bulk_kernel(long long n_slots, int row_bytes, int E, long long C, int chunks,
                         const int* __restrict__ pick_of_slot, const int* __restrict__ ptok,
                         const uint8_t* __restrict__ x, const PeerRows buf, const RowRange rr) {
  fsmoe_dev::pdl_enter();
  extern __shared__ __align__(128) uint8_t sm[];  // [BK_ROWS][row_bytes] + one zero row
  // one mbarrier per lane: a row's store leaves as soon as that row has landed
  // instead of after the whole group of BK_ROWS rows
  __shared__ __align__(8) uint64_t bar[BK_ROWS];
  const int lane = threadIdx.x;
  uint8_t* zero = sm + BK_ROWS * row_bytes;
  for (int i = lane * 16; i < row_bytes; i += 32 * 16) *reinterpret_cast<uint4*>(zero + i) = make_uint4(0, 0, 0, 0);
  if (lane < BK_ROWS) {
    fsmoe_dev::mbar_init(&bar[lane], 1);
    fsmoe_dev::fence_barrier_init();
  }
  fsmoe_dev::fence_proxy_async_smem();  // the zero row (generic writes) -> async proxy
  __syncwarp();
  uint8_t* mine = sm + (lane % BK_ROWS) * row_bytes;
  const long long ngroups = (n_slots + BK_ROWS - 1) / BK_ROWS;
  uint32_t phase = 0;
  // persistent: a block walks groups of BK_ROWS slots (lanes >= BK_ROWS idle)
  for (long long g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const long long s = g * BK_ROWS + lane;
    const bool valid = lane < BK_ROWS && s < n_slots && in_range(rr, s);
    const int p = valid ? pick_of_slot[s] : -1;
    if (p >= 0) {
      fsmoe_dev::mbar_arrive_expect_tx(&bar[lane], static_cast<uint32_t>(row_bytes));
      fsmoe_dev::bulk_load(mine, x + static_cast<long long>(ptok[p]) * row_bytes, static_cast<uint32_t>(row_bytes), &bar[lane]);
      fsmoe_dev::mbar_wait(&bar[lane], phase);
      phase ^= 1u;
    }
    if (valid) {
      char* dst = peer_row(buf, slot_row(s, E, C, chunks), row_bytes);
      bulk_store(dst, p >= 0 ? mine : zero, static_cast<uint32_t>(row_bytes));
      fsmoe_dev::bulk_commit();
    }
    fsmoe_dev::bulk_wait_read<0>();  // this lane's row buffer is free for the next group
  }
  fsmoe_dev::bulk_wait<0>();  // shared memory must outlive the stores
  __syncwarp();
}

// dst[i] = src[idx[i]] (idx < 0: zero row), i < n_rows, through the TMA
// engine like dispatch_bulk_kernel; dst through a peer map (identity for a
// local buffer). The I-order / order-backward permutations of a top-1
// softmax gate (every kept weight is exactly 1.0) are such gathers.
__global__ void __launch_bounds__(32)
    gather_bulk_kernel(long long n_rows, int row_bytes, const int* __restrict__ idx,
                       const uint8_t* __restrict__ src, const PeerRows dst) {
  fsmoe_dev::pdl_enter();
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[BK_ROWS];  // one per lane, as in dispatch_bulk_kernel
  const int lane = threadIdx.x;
  uint8_t* zero = sm + BK_ROWS * row_bytes;
  for (int b = lane * 16; b < row_bytes; b += 32 * 16) *reinterpret_cast<uint4*>(zero + b) = make_uint4(0, 0, 0, 0);
  if (lane < BK_ROWS) {
    fsmoe_dev::mbar_init(&bar[lane], 1);
    fsmoe_dev::fence_barrier_init();
  }
  fsmoe_dev::fence_proxy_async_smem();
  __syncwarp();
  uint8_t* mine = sm + (lane % BK_ROWS) * row_bytes;
  const long long ngroups = (n_rows + BK_ROWS - 1) / BK_ROWS;
  uint32_t phase = 0;
  for (long long g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const long long i = g * BK_ROWS + lane;
    const bool valid = lane < BK_ROWS && i < n_rows;
    const int s = valid ? idx[i] : -1;
    if (s >= 0) {
      fsmoe_dev::mbar_arrive_expect_tx(&bar[lane], static_cast<uint32_t>(row_bytes));
      fsmoe_dev::bulk_load(mine, src + static_cast<long long>(s) * row_bytes, static_cast<uint32_t>(row_bytes), &bar[lane]);
      fsmoe_dev::mbar_wait(&bar[lane], phase);
      phase ^= 1u;
    }
    if (valid) {
      bulk_store(peer_row(dst, i, row_bytes), s >= 0 ? mine : zero, static_cast<uint32_t>(row_bytes));
      fsmoe_dev::bulk_commit();
    }
    fsmoe_dev::bulk_wait_read<0>();
  }
  fsmoe_dev::bulk_wait<0>();
  __syncwarp();
}

// persistent grid for the bulk row movers: every resident block slot, at
// most one block per group
// (occupancy cached per kernel, device and shared-memory size)
template <typename K>
int bulk_grid(K kern, int smem, long long ngroups) {
  static std::mutex mu;
  static int cached_smem[kMaxDevices], cached_per_sm[kMaxDevices];
  static bool valid[kMaxDevices];
  const int dev = current_device();
  int per_sm = 1;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (valid[dev] && cached_smem[dev] == smem) {
      per_sm = cached_per_sm[dev];
    } else {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
      cached_smem[dev] = smem;
      cached_per_sm[dev] = per_sm;
      valid[dev] = true;
    }
  }
  const long long slots = static_cast<long long>(per_sm) * device_sms();
  return static_cast<int>(ngroups < slots ? ngroups : slots);
}

// ---------------------------------------------------------------- combine --

template <typename T>
struct Acc;
template <>
struct Acc<double> {
  using type = double;
  static __device__ __forceinline__ double ld(const double* p, int i) { return p[i]; }
  static __device__ __forceinline__ void st(double* p, int i, double v) { p[i] = v; }
};
template <>
struct Acc<float> {
  using type = float;
  static __device__ __forceinline__ float ld(const float* p, int i) { return p[i]; }
  static __device__ __forceinline__ void st(float* p, int i, float v) { p[i] = v; }
};
template <>
struct Acc<__nv_bfloat16> {
  using type = float;
  static __device__ __forceinline__ float ld(const __nv_bfloat16* p, int i) {
    return __bfloat162float(p[i]);
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, int i, float v) {
    p[i] = __float2bfloat16(v);
  }
};

__device__ __forceinline__ double madd(double acc, double w, double b) {
  return __dadd_rn(acc, __dmul_rn(w, b));
}
__device__ __forceinline__ float madd(float acc, float w, float b) { return fmaf(w, b, acc); }

// 8 consecutive elements per lane per vector (16 B bf16 / 32 B fp32 / 64 B fp64),
// 4 vectors in flight per lane: one warp covers 1024 columns per pass.
constexpr int CV = 8;
constexpr int NV = 4;

template <typename T>
struct Vec8;
template <>
struct Vec8<__nv_bfloat16> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16* p, float* o) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      o[2 * i] = f.x;
      o[2 * i + 1] = f.y;
    }
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float* v) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <>
struct Vec8<float> {
  static __device__ __forceinline__ void ld(const float* p, float* o) {
    float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
  }
  static __device__ __forceinline__ void st(float* p, const float* v) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};
template <>
struct Vec8<double> {
  static __device__ __forceinline__ void ld(const double* p, double* o) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double2 d = reinterpret_cast<const double2*>(p)[i];
      o[2 * i] = d.x;
      o[2 * i + 1] = d.y;
    }
  }
  static __device__ __forceinline__ void st(double* p, const double* v) {
#pragma unroll
    for (int i = 0; i < 4; ++i) reinterpret_cast<double2*>(p)[i] = make_double2(v[2 * i], v[2 * i + 1]);
  }
};

// Load / store 8 elements at column j of a row; VEC: full aligned vector,
// otherwise bounds-checked scalars.
template <bool VEC, typename T, typename A>
__device__ __forceinline__ void ld8(const T* row, int j, int M, A* o) {
  if (VEC) {
    Vec8<T>::ld(row + j, o);
  } else {
#pragma unroll
    for (int v = 0; v < CV; ++v) o[v] = j + v < M ? Acc<T>::ld(row, j + v) : A(0);
  }
}
template <bool VEC, typename T, typename A>
__device__ __forceinline__ void st8(T* row, int j, int M, const A* x) {
  if (VEC) {
    Vec8<T>::st(row + j, x);
  } else {
#pragma unroll
    for (int v = 0; v < CV; ++v)
      if (j + v < M) Acc<T>::st(row, j + v, x[v]);
  }
}

// Raw 8-element vectors: loads stay packed (bf16: one uint4 = 8 values) until
// the element is used, which keeps the in-flight loads cheap in registers
// (fp32 staging of whole vectors cost 98 registers and 25 % occupancy).
template <typename T>
struct Raw8 {
  using type = typename Acc<T>::type[8];
};
template <>
struct Raw8<__nv_bfloat16> {
  using type = uint4;
};
template <bool VEC, typename T>
__device__ __forceinline__ void ldraw(const T* row, int j, int M, typename Raw8<T>::type& r) {
  if constexpr (std::is_same_v<T, __nv_bfloat16>) {
    if (VEC) {
      r = *reinterpret_cast<const uint4*>(row + j);
    } else {
      __nv_bfloat16 h[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) h[v] = j + v < M ? row[j + v] : __float2bfloat16(0.f);
      r = *reinterpret_cast<uint4*>(h);
    }
  } else {
    ld8<VEC>(row, j, M, r);
  }
}
template <typename T, typename A>
__device__ __forceinline__ A rawget(const typename Raw8<T>::type& r, int v) {
  if constexpr (std::is_same_v<T, __nv_bfloat16>) {
    const uint32_t w = (&r.x)[v >> 1];
    return __uint_as_float((v & 1) ? (w & 0xffff0000u) : (w << 16));
  } else {
    return r[v];
  }
}

// y[t] = sum_{kept picks of t, pick order} w * buf[row(slot)]; one warp per token.
template <typename T, bool VEC>
__global__ void __launch_bounds__(256)
    combine_kernel(int ntok, int M, int E, long long C, int chunks, const int* __restrict__ tptr,
                   const int* __restrict__ tpick, const int* __restrict__ slot_of_pick,
                   const double* __restrict__ pw, const T* __restrict__ buf, T* __restrict__ y) {
  fsmoe_dev::pdl_enter();
  using A = typename Acc<T>::type;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= ntok) return;
  const int lane = threadIdx.x & 31;
  const int a = tptr[t], b = tptr[t + 1];
  T* yr = y + static_cast<long long>(t) * M;
  for (int jb = 0; jb < M; jb += 32 * CV * NV) {
    A acc[NV][CV];
#pragma unroll
    for (int u = 0; u < NV; ++u)
#pragma unroll
      for (int v = 0; v < CV; ++v) acc[u][v] = A(0);
    for (int q = a; q < b; ++q) {
      const int p = tpick[q];
      const int s = slot_of_pick[p];
      if (s < 0) continue;
      const A w = static_cast<A>(pw[p]);
      const T* br = buf + slot_row(s, E, C, chunks) * M;
      typename Raw8<T>::type val[NV];
#pragma unroll
      for (int u = 0; u < NV; ++u) {
        const int j = jb + (u * 32 + lane) * CV;
        if (j < M) ldraw<VEC>(br, j, M, val[u]);
      }
#pragma unroll
      for (int u = 0; u < NV; ++u)
#pragma unroll
        for (int v = 0; v < CV; ++v) acc[u][v] = madd(acc[u][v], w, rawget<T, A>(val[u], v));
    }
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int j = jb + (u * 32 + lane) * CV;
      if (j < M) st8<VEC>(yr, j, M, acc[u]);
    }
  }
}

// dx[t] (+)= sum_{kept picks of t} dbuf[row(slot)]
template <typename T, bool VEC>
__global__ void __launch_bounds__(256)
    dispatch_bwd_kernel(int ntok, int M, int E, long long C, int chunks,
                        const int* __restrict__ tptr, const int* __restrict__ tpick,
                        const int* __restrict__ slot_of_pick, const T* __restrict__ dbuf,
                        T* __restrict__ dx, int accumulate) {
  fsmoe_dev::pdl_enter();
  using A = typename Acc<T>::type;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= ntok) return;
  const int lane = threadIdx.x & 31;
  const int a = tptr[t], b = tptr[t + 1];
  T* xr = dx + static_cast<long long>(t) * M;
  for (int jb = 0; jb < M; jb += 32 * CV * NV) {
    A acc[NV][CV];
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int j = jb + (u * 32 + lane) * CV;
      if (accumulate && j < M) {
        ld8<VEC>(xr, j, M, acc[u]);
      } else {
#pragma unroll
        for (int v = 0; v < CV; ++v) acc[u][v] = A(0);
      }
    }
    for (int q = a; q < b; ++q) {
      const int s = slot_of_pick[tpick[q]];
      if (s < 0) continue;
      const T* br = dbuf + slot_row(s, E, C, chunks) * M;
      typename Raw8<T>::type val[NV];
#pragma unroll
      for (int u = 0; u < NV; ++u) {
        const int j = jb + (u * 32 + lane) * CV;
        if (j < M) ldraw<VEC>(br, j, M, val[u]);
      }
#pragma unroll
      for (int u = 0; u < NV; ++u)
#pragma unroll
        for (int v = 0; v < CV; ++v) acc[u][v] = acc[u][v] + rawget<T, A>(val[u], v);
    }
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int j = jb + (u * 32 + lane) * CV;
      if (j < M) st8<VEC>(xr, j, M, acc[u]);
    }
  }
}

// dbuf[row(s)] = w_p * dy[t_p] (0 for padding); dw[p] = <dy[t_p], buf[row(s)]>.
template <typename T, bool VEC>
__global__ void __launch_bounds__(256)
    combine_bwd_kernel(long long n_slots, int M, int E, long long C, int chunks,
                       const int* __restrict__ pick_of_slot, const int* __restrict__ ptok,
                       const double* __restrict__ pw, const T* __restrict__ dy,
                       const T* __restrict__ buf, const PeerRows dbuf, double* __restrict__ dw,
                       const RowRange rr) {
  fsmoe_dev::pdl_enter();
  using A = typename Acc<T>::type;
  const long long s = blockIdx.x * 8LL + (threadIdx.x >> 5);
  if (s >= n_slots || !in_range(rr, s)) return;
  const int lane = threadIdx.x & 31;
  const int p = pick_of_slot[s];
  const long long row = slot_row(s, E, C, chunks);
  T* dr = reinterpret_cast<T*>(peer_row(dbuf, row, static_cast<long long>(M) * sizeof(T)));
  if (p < 0) {
    A z[CV];
#pragma unroll
    for (int v = 0; v < CV; ++v) z[v] = A(0);
    for (int j = lane * CV; j < M; j += 32 * CV) st8<VEC>(dr, j, M, z);
    return;
  }
  const A w = static_cast<A>(pw[p]);
  const T* g = dy + static_cast<long long>(ptok[p]) * M;
  const T* o = buf + row * M;
  A dot = A(0);
  for (int jb = 0; jb < M; jb += 32 * CV * NV) {
    typename Raw8<T>::type gv[NV], ov[NV];
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int j = jb + (u * 32 + lane) * CV;
      if (j < M) {
        ldraw<VEC>(g, j, M, gv[u]);
        ldraw<VEC>(o, j, M, ov[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int j = jb + (u * 32 + lane) * CV;
      if (j >= M) continue;
      A out[CV];
#pragma unroll
      for (int v = 0; v < CV; ++v) {
        const A gvv = rawget<T, A>(gv[u], v);
        out[v] = static_cast<A>(w * gvv);
        dot = madd(dot, gvv, rawget<T, A>(ov[u], v));
      }
      st8<VEC>(dr, j, M, out);
    }
  }
  for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
  if (lane == 0) dw[p] = static_cast<double>(dot);
}

template <typename F>
int by_dtype(int dtype, F&& f) {
  switch (dtype) {
    case FSMOE_F64: f(double{}); return 0;
    case FSMOE_F32: f(float{}); return 0;
    case FSMOE_BF16: f(__nv_bfloat16{}); return 0;
    default: return -1;
  }
}

int elem_size(int dtype) { return dtype == FSMOE_F64 ? 8 : dtype == FSMOE_F32 ? 4 : 2; }

}  // namespace

// dst[r] = 0 for the rows r with idx[r] < 0; one warp per row
__global__ void __launch_bounds__(256)
    zero_rows_kernel(long long n_rows, int row_vecs, const int* __restrict__ idx, uint4* __restrict__ dst) {
  fsmoe_dev::pdl_enter();
  const long long r = blockIdx.x * 8LL + (threadIdx.x >> 5);
  if (r >= n_rows || idx[r] >= 0) return;
  uint4* d = dst + r * row_vecs;
  for (int v = threadIdx.x & 31; v < row_vecs; v += 32) d[v] = make_uint4(0u, 0u, 0u, 0u);
}

// ------------------------------------------------------------------ host ---

size_t assign_workspace_bytes(long long P, int E) {
  long long ntiles = (P + AS_TILE - 1) / AS_TILE;
  if (ntiles < 1) ntiles = 1;
  return static_cast<size_t>(ntiles) * (E > 0 ? E : 1) * sizeof(int) + 256;
}

int assign_launch(long long P, const int* ptok, const int* pexp, int T, int E, long long C,
                  int* slot_of_pick, long long* fill, long long* dropped, int* pick_of_slot,
                  int* status, void* ws, cudaStream_t st) {
  if (E > AS_MAX_E) return config_error("dispatch: at most 256 experts per rank supported");
  if (P <= 0) {
    FSMOE_CUDA_TRY(cudaMemsetAsync(pick_of_slot, 0xFF, sizeof(int) * E * C, st), "assign memset");
    FSMOE_CUDA_TRY(cudaMemsetAsync(fill, 0, sizeof(long long) * E, st), "assign memset");
    FSMOE_CUDA_TRY(cudaMemsetAsync(dropped, 0, sizeof(long long), st), "assign memset");
    return FSMOE_OK;
  }
  int ntiles = static_cast<int>((P + AS_TILE - 1) / AS_TILE);
  int* cnt = static_cast<int*>(ws);
  pdl_launch(assign_count_kernel, ntiles, AS_THREADS, 0, st, P, ptok, pexp, T, E, cnt, status, pick_of_slot,
             static_cast<long long>(E) * C); ::fsmoe::count_launch();
  pdl_launch(assign_rank_kernel, ntiles, AS_THREADS, 0, st, P, pexp, E, C, cnt, ntiles, slot_of_pick,
                                                    pick_of_slot, fill, dropped); ::fsmoe::count_launch();
  return cuda_status(cudaGetLastError(), "fsmoe_assign");
}

size_t token_index_workspace_bytes(long long, int T) {
  return static_cast<size_t>(T + 1) * sizeof(int) * 2 + 256;
}

int token_index_launch(long long P, const int* ptok, int T, int k, int* tptr, int* tpick,
                       void* ws, cudaStream_t st) {
  if (k > 0) {
    long long n = (static_cast<long long>(T) * k > T + 1) ? static_cast<long long>(T) * k : T + 1;
    pdl_launch(tok_token_major_kernel, static_cast<int>((n + 255) / 256), 256, 0, st, T, k, tptr, tpick); ::fsmoe::count_launch();
    return cuda_status(cudaGetLastError(), "fsmoe_token_index");
  }
  int* cnt = static_cast<int*>(ws);
  int* cursor = cnt + (T + 1);
  FSMOE_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int) * (T + 1) * 2, st), "token_index memset");
  int pb = static_cast<int>((P + 255) / 256);
  if (pb > 0) { tok_count_kernel<<<pb, 256, 0, st>>>(P, ptok, T, cnt); ::fsmoe::count_launch(); }
  scan_excl_kernel<<<1, 1024, 0, st>>>(cnt, T, tptr); ::fsmoe::count_launch();
  if (pb > 0) { tok_place_kernel<<<pb, 256, 0, st>>>(P, ptok, T, tptr, cursor, tpick); ::fsmoe::count_launch(); }
  tok_sort_kernel<<<(T + 255) / 256, 256, 0, st>>>(T, tptr, tpick); ::fsmoe::count_launch();
  return cuda_status(cudaGetLastError(), "fsmoe_token_index");
}

int zero_rows_launch(long long n_rows, long long row_bytes, const int* idx, void* dst, cudaStream_t st) {
  if (n_rows <= 0) return FSMOE_OK;
  if (row_bytes % 16 != 0) return config_error("zero_rows: row bytes must be a multiple of 16");
  pdl_launch(zero_rows_kernel, static_cast<int>((n_rows + 7) / 8), 256, 0, st, n_rows,
             static_cast<int>(row_bytes / 16), idx, static_cast<uint4*>(dst));
  ::fsmoe::count_launch();
  return cuda_status(cudaGetLastError(), "fsmoe_zero_rows");
}

int gather_rows_launch(long long n_rows, long long row_bytes, const int* idx, const void* src,
                       const PeerRows& dst, cudaStream_t st) {
  if (n_rows <= 0) return FSMOE_OK;
  if (row_bytes % 16 != 0 || row_bytes > 4096)
    return config_error("gather_rows: row bytes must be a multiple of 16 and at most 4096");
  static DeviceOnce attr;
  once_on_device(attr, [&] { cudaFuncSetAttribute(gather_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 33 * 4096); });
  const int smem = static_cast<int>((BK_ROWS + 1) * row_bytes);
  pdl_launch(gather_bulk_kernel, bulk_grid(gather_bulk_kernel, smem, (n_rows + BK_ROWS - 1) / BK_ROWS), 32, smem, st, 
      n_rows, static_cast<int>(row_bytes), idx, static_cast<const uint8_t*>(src), dst);
  ::fsmoe::count_launch();
  return cuda_status(cudaGetLastError(), "fsmoe_gather_rows");
}

int dispatch_launch(int dtype, int M, int E, long long C, int chunks, const int* pick_of_slot,
                    const int* ptok, const void* x, const PeerRows& buf, cudaStream_t st,
                    const RowRange& rr) {
  const long long n_slots = static_cast<long long>(E) * C;
  if (n_slots <= 0 || M <= 0) return FSMOE_OK;
  const long long row_bytes = static_cast<long long>(M) * elem_size(dtype);
  const int grid = static_cast<int>((n_slots + 7) / 8);
  static const bool nobulk = getenv("FSMOE_ROUTE_NOBULK") != nullptr;  // measurement switch, read once
  if (row_bytes % 16 == 0 && row_bytes <= 4096 && !nobulk) {
    const int smem = static_cast<int>((BK_ROWS + 1) * row_bytes);
    static DeviceOnce attr;
    once_on_device(attr, [&] { cudaFuncSetAttribute(dispatch_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 33 * 4096); });
    pdl_launch(dispatch_bulk_kernel, bulk_grid(dispatch_bulk_kernel, smem, (n_slots + BK_ROWS - 1) / BK_ROWS), 32, smem, st, 
        n_slots, static_cast<int>(row_bytes), E, C, chunks, pick_of_slot, ptok,
        static_cast<const uint8_t*>(x), buf, rr);
    ::fsmoe::count_launch();
  } else if (row_bytes % 16 == 0) {
    pdl_launch(dispatch_kernel<uint4>, grid, 256, 0, st, n_slots, static_cast<int>(row_bytes / 16), E, C,
                                                 chunks, pick_of_slot, ptok,
                                                 static_cast<const uint4*>(x), buf, rr); ::fsmoe::count_launch();
  } else if (row_bytes % 8 == 0) {
    pdl_launch(dispatch_kernel<uint2>, grid, 256, 0, st, n_slots, static_cast<int>(row_bytes / 8), E, C,
                                                 chunks, pick_of_slot, ptok,
                                                 static_cast<const uint2*>(x), buf, rr); ::fsmoe::count_launch();
  } else {
    pdl_launch(dispatch_kernel<uint16_t>, grid, 256, 0, st, 
        n_slots, static_cast<int>(row_bytes / 2), E, C, chunks, pick_of_slot, ptok,
        static_cast<const uint16_t*>(x), buf, rr); ::fsmoe::count_launch();
  }
  return cuda_status(cudaGetLastError(), "fsmoe_dispatch");
}

int combine_launch(int dtype, int T, int M, int E, long long C, int chunks, const int* tptr,
                   const int* tpick, const int* slot_of_pick, const double* pw, const void* buf,
                   void* y, cudaStream_t st) {
  if (T <= 0 || M <= 0) return FSMOE_OK;
  const int grid = (T + 7) / 8;
  int rc = by_dtype(dtype, [&](auto tag) {
    using Tt = decltype(tag);
    if (M % CV == 0)
      pdl_launch(combine_kernel<Tt, true>, grid, 256, 0, st, T, M, E, C, chunks, tptr, tpick, slot_of_pick,
                                                     pw, static_cast<const Tt*>(buf), static_cast<Tt*>(y));
    else
      pdl_launch(combine_kernel<Tt, false>, grid, 256, 0, st, T, M, E, C, chunks, tptr, tpick, slot_of_pick,
                                                      pw, static_cast<const Tt*>(buf), static_cast<Tt*>(y));
    ::fsmoe::count_launch();
  });
  if (rc) return config_error("combine: unknown dtype");
  return cuda_status(cudaGetLastError(), "fsmoe_combine");
}

int dispatch_bwd_launch(int dtype, int T, int M, int E, long long C, int chunks, const int* tptr,
                        const int* tpick, const int* slot_of_pick, const void* dbuf, void* dx,
                        int accumulate, cudaStream_t st) {
  if (T <= 0 || M <= 0) return FSMOE_OK;
  const int grid = (T + 7) / 8;
  int rc = by_dtype(dtype, [&](auto tag) {
    using Tt = decltype(tag);
    if (M % CV == 0)
      pdl_launch(dispatch_bwd_kernel<Tt, true>, grid, 256, 0, st, T, M, E, C, chunks, tptr, tpick, slot_of_pick,
                                                          static_cast<const Tt*>(dbuf),
                                                          static_cast<Tt*>(dx), accumulate);
    else
      pdl_launch(dispatch_bwd_kernel<Tt, false>, grid, 256, 0, st, T, M, E, C, chunks, tptr, tpick, slot_of_pick,
                                                           static_cast<const Tt*>(dbuf),
                                                           static_cast<Tt*>(dx), accumulate);
    ::fsmoe::count_launch();
  });
  if (rc) return config_error("dispatch_bwd: unknown dtype");
  return cuda_status(cudaGetLastError(), "fsmoe_dispatch_bwd");
}

int combine_bwd_launch(int dtype, int M, int E, long long C, int chunks, long long P,
                       const int* pick_of_slot, const int* ptok, const double* pw,
                       const void* dy, const void* buf, const PeerRows& dbuf, double* dw,
                       cudaStream_t st, const RowRange& rr) {
  const long long n_slots = static_cast<long long>(E) * C;
  // (a range launch leaves dw of the other slots' picks alone)
  if (P > 0 && !rr.excl && rr.lo <= 0 && rr.hi >= static_cast<long long>(E) * C)
    FSMOE_CUDA_TRY(cudaMemsetAsync(dw, 0, sizeof(double) * P, st), "combine_bwd memset");
  if (n_slots <= 0 || M <= 0) return FSMOE_OK;
  const int grid = static_cast<int>((n_slots + 7) / 8);
  int rc = by_dtype(dtype, [&](auto tag) {
    using Tt = decltype(tag);
    if (M % CV == 0)
      pdl_launch(combine_bwd_kernel<Tt, true>, grid, 256, 0, st, n_slots, M, E, C, chunks, pick_of_slot, ptok, pw,
                                                         static_cast<const Tt*>(dy),
                                                         static_cast<const Tt*>(buf),
                                                         dbuf, dw, rr);
    else
      pdl_launch(combine_bwd_kernel<Tt, false>, grid, 256, 0, st, n_slots, M, E, C, chunks, pick_of_slot, ptok, pw,
                                                          static_cast<const Tt*>(dy),
                                                          static_cast<const Tt*>(buf),
                                                          dbuf, dw, rr);
    ::fsmoe::count_launch();
  });
  if (rc) return config_error("combine_bwd: unknown dtype");
  return cuda_status(cudaGetLastError(), "fsmoe_combine_bwd");
}

}  // namespace fsmoe
