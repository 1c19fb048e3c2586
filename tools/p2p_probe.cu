// p2p_probe.cu — NVLink peer-store microbenchmark (two GPUs, one process,
// cudaDeviceEnablePeerAccess). Measures how fast SM stores reach a peer's
// HBM for the access patterns the MoE layer's fused producers can use:
//   rowthread: one thread per row, 64 B per store group, rows 2 KB apart
//              (the GEMM epilogue's TMEM 32x32b fragment order)
//   coalesced: a warp writes 512 contiguous bytes (16 B per lane)
//   bulk:      smem -> global cp.async.bulk, 512 B rows issued by one lane
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_probe p2p_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));         \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

constexpr long long ROW = 2048;  // bytes per row (M = 1024 bf16)

__global__ void rowthread(const uint4* __restrict__ src, char* __restrict__ dst, long long rows) {
  // thread t: row r = t / 32 * 32 + lane, column chunk c = (t / 32) % 32 ... cover all
  const long long nthreads = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long units = rows * (ROW / 64);  // 64-byte units
  for (long long u = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; u < units;
       u += nthreads) {
    // consecutive lanes -> consecutive rows, same column chunk
    const long long lane = u & 31, grp = u >> 5;
    const long long chunks = ROW / 64;
    const long long c = grp % chunks, rblk = grp / chunks;
    const long long r = rblk * 32 + lane;
    const uint4* s = src + (r * ROW + c * 64) / 16;
    uint4* d = reinterpret_cast<uint4*>(dst + r * ROW + c * 64);
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = s[i];
  }
}

__global__ void coalesced(const uint4* __restrict__ src, uint4* __restrict__ dst, long long n16) {
  const long long nthreads = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n16;
       i += 4 * nthreads) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * nthreads < n16) v[k] = src[i + k * nthreads];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * nthreads < n16) dst[i + k * nthreads] = v[k];
  }
}

// segments of SEG bytes per row (rows ROW apart), a warp covers 512/SEG rows
template <int SEG>
__global__ void segmented(const uint4* __restrict__ src, char* __restrict__ dst, long long rows) {
  constexpr int LPS = SEG / 16;  // lanes per segment
  const long long nthreads = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long segs_per_row = ROW / SEG;
  const long long units = rows * segs_per_row * LPS;
  for (long long u = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; u < units;
       u += nthreads) {
    const long long l = u % LPS, sg = u / LPS;
    // consecutive segments -> consecutive rows (same column block), like a
    // transposed epilogue tile
    const long long r = sg % rows, cb = sg / rows;
    const long long off = r * ROW + cb * SEG + l * 16;
    *reinterpret_cast<uint4*>(dst + off) = src[off / 16];
  }
}

__global__ void bulk(const char* __restrict__ src, char* __restrict__ dst, long long bytes) {
  extern __shared__ __align__(128) char sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int nw = blockDim.x / 32;
  char* my = sm + warp * 4096;
  const long long nchunk = bytes / 4096;
  for (long long ch = blockIdx.x * static_cast<long long>(nw) + warp; ch < nchunk;
       ch += static_cast<long long>(gridDim.x) * nw) {
    const uint4* s = reinterpret_cast<const uint4*>(src + ch * 4096);
    // previous bulk store must have read smem
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
    for (int i = lane; i < 256; i += 32) reinterpret_cast<uint4*>(my)[i] = s[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      for (int k = 0; k < 8; ++k) {
        unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(my + k * 512));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(
                         dst + ch * 4096 + k * 512),
                     "r"(sa)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("need 2 GPUs\n");
    return 1;
  }
  const long long bytes = 16LL << 20;
  char *src, *dloc, *dpeer;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&dpeer, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&src, bytes));
  CK(cudaMalloc(&dloc, bytes));
  CK(cudaMemset(src, 1, bytes));
  CK(cudaFuncSetAttribute(bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int grids[] = {16, 32, 148};
  for (int dst_i = 0; dst_i < 2; ++dst_i) {
    char* dst = dst_i ? dpeer : dloc;
    for (int g : grids) {
      for (int kind = 0; kind < 6; ++kind) {
        auto run = [&] {
          if (kind == 0) rowthread<<<g, 256>>>(reinterpret_cast<const uint4*>(src), dst, bytes / ROW);
          if (kind == 1)
            coalesced<<<g, 256>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst),
                                  bytes / 16);
          if (kind == 2) bulk<<<g, 256, 8 * 4096>>>(src, dst, bytes);
          if (kind == 3) segmented<128><<<g, 256>>>(reinterpret_cast<const uint4*>(src), dst, bytes / ROW);
          if (kind == 4) segmented<256><<<g, 256>>>(reinterpret_cast<const uint4*>(src), dst, bytes / ROW);
          if (kind == 5) segmented<512><<<g, 256>>>(reinterpret_cast<const uint4*>(src), dst, bytes / ROW);
        };
        for (int w = 0; w < 3; ++w) run();
        CK(cudaEventRecord(a));
        const int reps = 20;
        for (int r = 0; r < reps; ++r) run();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        ms /= reps;
        const char* kn[] = {"rowthread", "coalesced", "bulk", "seg128", "seg256", "seg512"};
        printf("%s grid %4d %-10s %8.1f us  %7.1f GB/s\n", dst_i ? "peer " : "local", g, kn[kind],
               ms * 1e3, bytes / (ms * 1e-3) / 1e9);
      }
    }
  }
  // bidirectional: both GPUs push 16 MB into each other at once
  char *src1, *dpeer0;
  CK(cudaMalloc(&dpeer0, bytes));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&src1, bytes));
  cudaStream_t s1;
  CK(cudaStreamCreate(&s1));
  cudaEvent_t a1, b1;
  CK(cudaEventCreate(&a1));
  CK(cudaEventCreate(&b1));
  CK(cudaSetDevice(0));
  for (int kind : {0, 3, 4, 5}) {
    for (int g : {32, 148}) {
      auto run2 = [&](int dev, cudaStream_t st, const char* s, char* d) {
        CK(cudaSetDevice(dev));
        if (kind == 0) rowthread<<<g, 256, 0, st>>>(reinterpret_cast<const uint4*>(s), d, bytes / ROW);
        if (kind == 3) segmented<128><<<g, 256, 0, st>>>(reinterpret_cast<const uint4*>(s), d, bytes / ROW);
        if (kind == 4) segmented<256><<<g, 256, 0, st>>>(reinterpret_cast<const uint4*>(s), d, bytes / ROW);
        if (kind == 5) segmented<512><<<g, 256, 0, st>>>(reinterpret_cast<const uint4*>(s), d, bytes / ROW);
      };
      for (int w = 0; w < 3; ++w) { run2(0, 0, src, dpeer); run2(1, s1, src1, dpeer0); }
      CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(0)); CK(cudaEventRecord(a, 0));
      CK(cudaSetDevice(1)); CK(cudaEventRecord(a1, s1));
      for (int r = 0; r < 20; ++r) { run2(0, 0, src, dpeer); run2(1, s1, src1, dpeer0); }
      CK(cudaSetDevice(0)); CK(cudaEventRecord(b, 0));
      CK(cudaSetDevice(1)); CK(cudaEventRecord(b1, s1));
      CK(cudaEventSynchronize(b1));
      CK(cudaSetDevice(0)); CK(cudaEventSynchronize(b));
      float ms0 = 0, ms1 = 0;
      CK(cudaEventElapsedTime(&ms0, a, b));
      CK(cudaSetDevice(1)); CK(cudaEventElapsedTime(&ms1, a1, b1));
      CK(cudaSetDevice(0));
      const char* kn[] = {"rowthread", "", "", "seg128", "seg256", "seg512"};
      printf("bidir grid %4d %-10s gpu0 %7.1f GB/s gpu1 %7.1f GB/s\n", g, kn[kind],
             bytes / (ms0 / 20 * 1e-3) / 1e9, bytes / (ms1 / 20 * 1e-3) / 1e9);
    }
  }
  // copy engines: one large cudaMemcpyAsync into the peer's buffer (no SMs)
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaSetDevice(0));
    for (int w = 0; w < 3; ++w) CK(cudaMemcpyAsync(dpeer, src, bytes, cudaMemcpyDeviceToDevice, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a, 0));
    for (int r = 0; r < 20; ++r) CK(cudaMemcpyAsync(dpeer, src, bytes, cudaMemcpyDeviceToDevice, 0));
    CK(cudaEventRecord(b, 0));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("copy engine peer 16 MB: %7.1f GB/s\n", bytes / (ms / 20 * 1e-3) / 1e9);
  }
  // both directions at once
  CK(cudaSetDevice(0));
  CK(cudaEventRecord(a, 0));
  CK(cudaSetDevice(1));
  CK(cudaEventRecord(a1, s1));
  for (int r = 0; r < 20; ++r) {
    CK(cudaSetDevice(0));
    CK(cudaMemcpyAsync(dpeer, src, bytes, cudaMemcpyDeviceToDevice, 0));
    CK(cudaSetDevice(1));
    CK(cudaMemcpyAsync(dpeer0, src1, bytes, cudaMemcpyDeviceToDevice, s1));
  }
  CK(cudaSetDevice(0));
  CK(cudaEventRecord(b, 0));
  CK(cudaSetDevice(1));
  CK(cudaEventRecord(b1, s1));
  CK(cudaEventSynchronize(b1));
  CK(cudaSetDevice(0));
  CK(cudaEventSynchronize(b));
  {
    float ms0 = 0, ms1 = 0;
    CK(cudaEventElapsedTime(&ms0, a, b));
    CK(cudaSetDevice(1));
    CK(cudaEventElapsedTime(&ms1, a1, b1));
    printf("copy engine bidir: gpu0 %7.1f GB/s gpu1 %7.1f GB/s\n", bytes / (ms0 / 20 * 1e-3) / 1e9,
           bytes / (ms1 / 20 * 1e-3) / 1e9);
  }
  return 0;
}
