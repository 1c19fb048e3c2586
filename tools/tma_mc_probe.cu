// tma_mc_probe.cu — does TMA multicast raise the L2 -> SM operand delivery
// rate that bounds the expert GEMMs (ncu: lts2xbar ~85 % of peak)?
// Every CTA (one per SM, persistent) streams 16 KB SW128 boxes (64 bf16 x
// 128 rows, the GEMM's per-stage A/B box) from an L2-resident tensor into
// an 8-stage ring; a consumer warp releases each stage as soon as it lands.
//   mode 0 UC-distinct: each CTA loads its own boxes
//   mode 1 UC-same:     all CTAs of a cluster load the same box at once
//   mode 2 MC:          each CTA of a cluster loads 1/CS of the box and
//                       multicasts it to the whole cluster
// Reports delivered bytes/s (all SMs' smem fills) for cluster sizes 1,2,4,8.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_mc_probe tma_mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));         \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

constexpr int MAX_STAGES = 13;
constexpr int BOX_ROWS = 128;
constexpr int BOX_BYTES = BOX_ROWS * 128;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* b, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(su32(b)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ unsigned long long g_clk[2];

__global__ void __launch_bounds__(160) probe(const __grid_constant__ CUtensorMap map, int mode,
                                            int iters, int ntiles, int STAGES, const uint8_t* raw) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[MAX_STAGES], empty[MAX_STAGES];
  const uint32_t cs = nctarank(), rank = ctarank();
  const int cluster = blockIdx.x / cs;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], mode == 2 ? cs : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync();
  unsigned long long c0 = clock64(), t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  // producers: warp 0 (+ warps 2.. for modes 5 / 6: 2 / 4 issuing threads)
  const int nprod = mode == 5 ? 2 : mode == 6 ? 4 : 1;
  const int pidx = warp == 0 ? 0 : warp - 1;
  if (warp != 1 && pidx < nprod && lane == 0) {
    for (int i = pidx; i < iters; i += nprod) {
      const int s = i % STAGES;
      if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
      mbar_expect(&full[s], BOX_BYTES);
      int tile;
      if (mode == 0) tile = (blockIdx.x * 7 + i) % ntiles;
      else tile = (cluster * 7 + i) % ntiles;
      uint8_t* dst = smem + s * BOX_BYTES;
      if (mode == 2) {
        const int rows = BOX_ROWS / cs;
        // my slice: rows [rank*rows, (rank+1)*rows) of the box, to all CTAs
        const uint16_t mask = static_cast<uint16_t>((1u << cs) - 1);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
            " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(su32(dst + rank * rows * 128)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(su32(&full[s])), "r"(0),
            "r"(static_cast<int>(rank) * rows), "r"(tile), "h"(mask)
            : "memory");
      } else if (mode == 3) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(dst)),
            "l"(raw + static_cast<size_t>(tile) * BOX_BYTES), "r"(BOX_BYTES), "r"(su32(&full[s]))
            : "memory");
      } else if (mode == 4) {
        for (int part = 0; part < 2; ++part)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(dst + part * BOX_BYTES / 2)),
              "l"(reinterpret_cast<uint64_t>(&map)), "r"(su32(&full[s])), "r"(0), "r"(part * BOX_ROWS / 2),
              "r"(tile)
              : "memory");
      } else {
        for (int part = 0; part < 1; ++part)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(dst)),
              "l"(reinterpret_cast<uint64_t>(&map)), "r"(su32(&full[s])), "r"(0), "r"(0), "r"(tile)
              : "memory");
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      if (mode == 2) {
        for (uint32_t r = 0; r < cs; ++r) mbar_arrive_remote(&empty[s], r);
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
      }
    }
  }
  cluster_sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    g_clk[0] = clock64() - c0;
    g_clk[1] = t1 - t0;
  }
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  // tensor: [ntiles][BOX_ROWS rows][64 bf16], 16 KB per box; default 1536
  // boxes = 24 MB (L2 resident, spread over every slice)
  const int ntiles = argc > 1 ? atoi(argv[1]) : 1536;
  void* buf;
  const size_t bytes = static_cast<size_t>(ntiles) * BOX_BYTES;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  CUtensorMap map;
  cuuint64_t dims[3] = {64, BOX_ROWS, static_cast<cuuint64_t>(ntiles)};
  cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(BOX_BYTES)};
  const int iters = 20000;
  const int smem = MAX_STAGES * BOX_BYTES + 1024;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const int only_uc = argc > 2;
  for (int stages : {4, 8, 13})
  for (int cs : {1, 2, 4, 8}) {
    for (int mode = 0; mode < 7; ++mode) {
      if (cs == 1 && (mode == 1 || mode == 2)) continue;
      if (cs > 1 && mode > 2) continue;
      if (only_uc && (cs > 1 || mode == 1 || mode == 2)) continue;
      if (!only_uc && stages != 8) continue;
      cuuint32_t box[3] = {64, static_cast<cuuint32_t>(mode == 2 ? BOX_ROWS / cs : mode == 4 ? BOX_ROWS / 2 : BOX_ROWS), 1};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", static_cast<int>(r));
        return 1;
      }
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cfg.blockDim = dim3(160);
      cfg.dynamicSmemBytes = smem;
      int max_clusters = 0;
      cfg.gridDim = dim3(cs * 64);
      CK(cudaOccupancyMaxActiveClusters(&max_clusters, probe, &cfg));
      const int grid = std::min(max_clusters, sms / cs) * cs;
      cfg.gridDim = dim3(grid);
      cudaEvent_t a, b;
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
      CK(cudaLaunchKernelEx(&cfg, probe, map, mode, 200, ntiles, stages, (const uint8_t*)buf));
      CK(cudaEventRecord(a));
      CK(cudaLaunchKernelEx(&cfg, probe, map, mode, iters, ntiles, stages, (const uint8_t*)buf));
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      const double delivered = static_cast<double>(grid) * iters * BOX_BYTES;
      const double l2_reads = mode == 1 ? delivered : delivered / (mode == 2 ? 1.0 : 1.0);
      unsigned long long clk[2];
      CK(cudaMemcpyFromSymbol(clk, g_clk, sizeof(clk)));
      const double ghz = static_cast<double>(clk[0]) / clk[1];
      printf("%.3f GHz, %.1f B/clk/SM | ", ghz, delivered / grid / (ms * 1e-3) / (ghz * 1e9));
      printf("stages %d cluster %d mode %s: grid %d (max clusters %d), delivered %.2f TB/s (%.1f GB/s per SM)\n", stages, cs,
             mode == 0 ? "UC-distinct" : mode == 1 ? "UC-same    " : mode == 2 ? "MC         " : mode == 3 ? "bulk-1d    " : mode == 4 ? "2 half-box " : mode == 5 ? "2 producers" : "4 producers", grid, max_clusters,
             delivered / ms / 1e9, delivered / ms / 1e6 / grid);
      (void)l2_reads;
    }
  }
  return 0;
}
