// route_common.cuh — shared device helpers for the routing kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace fsmoe_dev {

// Element load as double (exact upcast of bf16 / fp32 / fp64).
template <int DT>
__device__ __forceinline__ double load_as_double(const void* base, long long i);
template <>
__device__ __forceinline__ double load_as_double<0>(const void* base, long long i) {
  return static_cast<const double*>(base)[i];
}
template <>
__device__ __forceinline__ double load_as_double<1>(const void* base, long long i) {
  return static_cast<double>(static_cast<const float*>(base)[i]);
}
template <>
__device__ __forceinline__ double load_as_double<2>(const void* base, long long i) {
  return static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(base)[i]));
}

// Programmatic dependent launch (host side: fsmoe::pdl_launch): let the
// stream's next kernel be scheduled now, then wait until every prior grid has
// completed and its memory is visible. Must precede any global-memory access
// of a kernel launched with the PDL attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Reference arithmetic: acc + a*b with a separately rounded product (no FMA).
__device__ __forceinline__ double mul_add_rn(double acc, double a, double b) {
  return __dadd_rn(acc, __dmul_rn(a, b));
}

// Slot -> row of the (possibly chunk-major) dispatch buffer. See
// fsmoe_slot_row in include/fsmoe_cuda.h.
__host__ __device__ __forceinline__ long long slot_row(long long slot, int experts,
                                                        long long cap, int chunks) {
  if (chunks <= 1) return slot;
  long long e = slot / cap;
  long long c = slot - e * cap;
  // chunk i covers [floor(i*cap/r), floor((i+1)*cap/r))
  long long i = (c * chunks + chunks - 1) / cap;  // candidate, fix up below
  if (i >= chunks) i = chunks - 1;
  while (i > 0 && (i * cap) / chunks > c) --i;
  while (i + 1 < chunks && ((i + 1) * cap) / chunks <= c) ++i;
  long long lo = (i * cap) / chunks;
  long long hi = ((i + 1) * cap) / chunks;
  return static_cast<long long>(experts) * lo + e * (hi - lo) + (c - lo);
}

// Destination of a row of a [P][E_l][C] block buffer written to peer memory
// (include/fsmoe_cuda.h fsmoe_peer_rows): row r of block b = p*E_l + e_l goes
// to base[p] at row (rank*E_l + e_l)*C + r%C -- the receiver's layout is the
// same [P][E_l][C] indexed by source rank. world 1 / rank 0 is the identity.
constexpr int MAX_PEERS = 8;
struct PeerRows {
  char* base[MAX_PEERS];
  int world, rank, el;
  long long cap;
};
__device__ __forceinline__ char* peer_row(const PeerRows& m, long long row, long long row_bytes) {
  if (m.world <= 1) return m.base[0] + row * row_bytes;
  const long long b = row / m.cap;
  const long long c = row - b * m.cap;
  const int p = static_cast<int>(b / m.el);
  const long long e = b - static_cast<long long>(p) * m.el;
  return m.base[p] + ((static_cast<long long>(m.rank) * m.el + e) * m.cap + c) * row_bytes;
}

// Which rows / slots / blocks a launch covers: [lo, hi), or everything but
// that range when excl. Lets the EP layer run its local share of a
// permutation or GEMM first and the peers' share on a second stream.
struct RowRange {
  long long lo, hi;
  int excl;
};
__host__ __device__ __forceinline__ bool in_range(const RowRange& r, long long i) {
  return (i >= r.lo && i < r.hi) != (r.excl != 0);
}
__host__ __device__ __forceinline__ RowRange all_rows() { return RowRange{0, (1LL << 62), 0}; }

// Monotone map double -> uint64 (a < b  <=>  key(a) < key(b)) for non-NaN.
__device__ __forceinline__ uint64_t order_key(double v) {
  if (v == 0.0) v = 0.0;  // -0.0 == +0.0 in the reference's comparisons
  uint64_t u = static_cast<uint64_t>(__double_as_longlong(v));
  return (u & 0x8000000000000000ULL) ? ~u : (u | 0x8000000000000000ULL);
}

}  // namespace fsmoe_dev
