// peer.cu — arrival flags for the peer-memory AlltoAll (include/fsmoe_cuda.h
// fsmoe_peer_signal / fsmoe_peer_wait).
//
// The MoE layer's dispatch / combine exchanges are stores into the owning
// rank's buffers, issued by the producing kernel itself over NVLink
// (CUDA-IPC-mapped peer pointers). What remains of the "collective" is one
// ordering edge per exchange: the producer's stream raises flag[slot][rank]
// on every peer after its data stores, the consumer's stream spins until all
// sources have raised flag[slot][*] to the exchange's sequence number.
//
//   signal:  (optional small payload rows) -> bar.sync -> fence.sc.sys ->
//            red.release.sys.add(flag, 1)          one thread per peer
//   wait:    ld.acquire.sys(flag) >= target        one thread per source
//
// The stores of the kernels before `signal` in stream order are complete at
// its start (kernel boundary); the system-scope fence orders them, and the
// payload, before the flag for the remote observer. Counters only grow, so a
// flag is never reset and a late waiter cannot miss an increment.
//
// A peer that never signals (crashed rank) would spin the waiter forever; the
// wait gives up after fsmoe_peer_flags::timeout_ns (the layer takes it from
// FSMOE_PEER_TIMEOUT_S, default 600 s; 0 = never) and traps so the process
// fails instead of wedging the GPU. A legitimately late peer (checkpoint,
// evaluation, first-step initialisation) stays well inside the default.
//
// With fsmoe_peer_flags::wait_ns set, every wait adds the time it spent
// spinning (globaltimer, first thread in to last flag seen) to that counter:
// the untraced per-rank exposed-exchange time the bench reports.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>

#include "capi_common.h"
#include "kernels.h"

namespace fsmoe {
namespace {

using namespace fsmoe_dev;

struct Flags {
  unsigned long long* base[MAX_PEERS];
  int world, rank, nslots;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_sys_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void peer_signal_kernel(Flags f, int slot, const unsigned long long* __restrict__ put,
                                   int put_words, PeerRows put_dst, int put_rows) {
  // payload: rows of put_words 8-byte words, [world][el] rows, capacity 1
  const long long total = static_cast<long long>(put_rows) * put_words;
  for (long long i = threadIdx.x; i < total; i += blockDim.x) {
    const long long r = i / put_words;
    const int w = static_cast<int>(i - r * put_words);
    unsigned long long* d =
        reinterpret_cast<unsigned long long*>(peer_row(put_dst, r, 8LL * put_words));
    d[w] = put[i];
  }
  __syncthreads();
  const int p = threadIdx.x;
  if (p < f.world) {
    __threadfence_system();
    red_release_sys_add(f.base[p] + static_cast<long long>(slot) * f.world + f.rank, 1ULL);
  }
}

__global__ void peer_wait_kernel(const unsigned long long* __restrict__ flags, int world, int slot,
                                 unsigned long long target, unsigned long long* wait_ns,
                                 unsigned long long timeout_ns) {
  const int src = threadIdx.x;
  const unsigned long long t0 = global_ns();
  if (src < world) {
    const unsigned long long* fl = flags + static_cast<long long>(slot) * world + src;
    while (ld_acquire_sys(fl) < target) {
      __nanosleep(64);
      if (timeout_ns && global_ns() - t0 > timeout_ns) {
        printf("fsmoe_peer_wait: rank-%d flag of slot %d stuck below %llu (peer lost?)\n", src,
               slot, target);
        __trap();
      }
    }
  }
  __syncthreads();
  if (wait_ns && src == 0) atomicAdd(wait_ns, global_ns() - t0);
}

template <class T>
struct Srcs {
  const T* p[MAX_PEERS];
};

template <class T>
__global__ void sum_buffers_kernel(Srcs<T> s, int n_src, long long n, T* __restrict__ dst) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    T v = s.p[0][i];
    for (int k = 1; k < n_src; ++k) v += s.p[k][i];
    dst[i] = v;
  }
}

int check_flags(const fsmoe_peer_flags* f, int slot) {
  if (!f) return config_error("peer flags: null");
  if (f->world < 1 || f->world > MAX_PEERS || f->rank < 0 || f->rank >= f->world)
    return config_error("peer flags: world must be in [1, 8] and rank in [0, world)");
  if (slot < 0 || slot >= f->nslots) return config_error("peer flags: slot out of range");
  for (int p = 0; p < f->world; ++p)
    if (!f->base[p]) return config_error("peer flags: missing peer flag array");
  return FSMOE_OK;
}

}  // namespace
}  // namespace fsmoe

using namespace fsmoe;

extern "C" int fsmoe_peer_signal(const fsmoe_peer_flags* f, int slot, const void* put_src,
                                 long long put_row_bytes, const fsmoe_peer_rows* put_dst,
                                 void* stream) {
  if (int rc = check_flags(f, slot)) return rc;
  Flags k{};
  for (int p = 0; p < f->world; ++p) k.base[p] = f->base[p];
  k.world = f->world;
  k.rank = f->rank;
  k.nslots = f->nslots;
  fsmoe_dev::PeerRows dst{};
  int rows = 0, words = 0;
  if (put_src) {
    if (!put_dst || put_row_bytes <= 0 || put_row_bytes % 8 || put_dst->capacity != 1)
      return config_error("peer signal: payload rows must be 8-byte words with a capacity-1 map");
    dst = peer_rows_of(put_dst);
    rows = put_dst->world * put_dst->experts_local;
    words = static_cast<int>(put_row_bytes / 8);
  }
  peer_signal_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      k, slot, static_cast<const unsigned long long*>(put_src), words, dst, rows);
  count_launch();
  return cuda_status(cudaGetLastError(), "fsmoe_peer_signal");
}

extern "C" int fsmoe_sum_buffers(int dtype, int n_src, const void* const* src, long long n, void* dst,
                                 void* stream) {
  if (n_src < 1 || n_src > MAX_PEERS || !src || (n > 0 && !dst))
    return config_error("sum buffers: need 1..8 sources and a destination");
  if (dtype != FSMOE_F64 && dtype != FSMOE_F32) return config_error("sum buffers: dtype must be f64 or f32");
  if (n <= 0) return FSMOE_OK;
  const int threads = 256;
  const int blocks = static_cast<int>(std::min<long long>((n + threads - 1) / threads, 148LL * 8));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == FSMOE_F64) {
    Srcs<double> s{};
    for (int k = 0; k < n_src; ++k) s.p[k] = static_cast<const double*>(src[k]);
    sum_buffers_kernel<<<blocks, threads, 0, st>>>(s, n_src, n, static_cast<double*>(dst));
  } else {
    Srcs<float> s{};
    for (int k = 0; k < n_src; ++k) s.p[k] = static_cast<const float*>(src[k]);
    sum_buffers_kernel<<<blocks, threads, 0, st>>>(s, n_src, n, static_cast<float*>(dst));
  }
  count_launch();
  return cuda_status(cudaGetLastError(), "fsmoe_sum_buffers");
}

extern "C" int fsmoe_peer_wait(const fsmoe_peer_flags* f, int slot, unsigned long long target,
                               void* stream) {
  if (int rc = check_flags(f, slot)) return rc;
  peer_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(f->base[f->rank], f->world, slot,
                                                                  target, f->wait_ns, f->timeout_ns);
  count_launch();
  return cuda_status(cudaGetLastError(), "fsmoe_peer_wait");
}

// ----------------------------------------------------- copy-engine exchange --
// The chunked pipeline's dispatch-side exchanges (FSMoE's D_0..D_{r-1} on the
// inter link, schedule_sim.cpp:182-216) without SM work: the permutation
// kernel leaves the peers' rows in a canonical [E][C] send buffer, the copy
// engines move pipeline chunk i (rows [lo, hi) of every block) into each
// peer's receive buffer while the expert GEMMs of chunk i-1 hold every SM,
// and a stream memory operation raises the chunk's arrival flag behind them.
namespace {

using PFN_writeValue64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

PFN_writeValue64 write_value_fn() {
  static PFN_writeValue64 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue64", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_writeValue64>(p);
  });
  return fn;
}

}  // namespace

extern "C" int fsmoe_peer_copy_rows(const void* send, long long row_bytes, const fsmoe_peer_rows* dst,
                                    long long lo, long long hi, int include_self, void* stream) {
  if (!send || !dst || row_bytes <= 0 || lo < 0 || hi > dst->capacity || lo > hi)
    return config_error("peer copy rows: send, map, row bytes > 0 and 0 <= lo <= hi <= capacity required");
  if (dst->world < 1 || dst->world > MAX_PEERS || dst->rank < 0 || dst->rank >= dst->world)
    return config_error("peer copy rows: world must be in [1, 8] and rank in [0, world)");
  if (hi == lo) return FSMOE_OK;
  const int P = dst->world, El = dst->experts_local, me = dst->rank;
  const size_t pitch = static_cast<size_t>(dst->capacity * row_bytes);
  const size_t width = static_cast<size_t>((hi - lo) * row_bytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int k = 0; k < P; ++k) {
    const int p = (me + k) % P;  // start with the next rank: spread the copies over the links
    if (p == me && !include_self) continue;
    if (!dst->base[p]) return config_error("peer copy rows: missing peer base");
    // this rank's E_l blocks for p: send rows [(p El + el) C + lo, ... + hi)
    const char* s = static_cast<const char*>(send) + (static_cast<size_t>(p) * El * dst->capacity + lo) * row_bytes;
    // land in p's [rank][el][C] blocks
    char* d = static_cast<char*>(dst->base[p]) + (static_cast<size_t>(me) * El * dst->capacity + lo) * row_bytes;
    cudaError_t e = cudaMemcpy2DAsync(d, pitch, s, pitch, width, static_cast<size_t>(El),
                                      cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_status(e, "fsmoe_peer_copy_rows");
  }
  return FSMOE_OK;
}

extern "C" int fsmoe_peer_flag_write(const fsmoe_peer_flags* f, int slot, unsigned long long value,
                                     void* stream) {
  if (int rc = check_flags(f, slot)) return rc;
  PFN_writeValue64 wv = write_value_fn();
  if (!wv) return config_error("peer flag write: cuStreamWriteValue64 unavailable");
  for (int p = 0; p < f->world; ++p) {
    unsigned long long* a = f->base[p] + static_cast<long long>(slot) * f->world + f->rank;
    // default flags: a system-scope memory fence orders the stream's earlier
    // work (the copies) before the write
    CUresult r = wv(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(a), value, 0);
    if (r != CUDA_SUCCESS) return cuda_status(cudaErrorUnknown, "fsmoe_peer_flag_write");
  }
  return FSMOE_OK;
}
