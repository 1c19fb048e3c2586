// gemm_sm100.cu — persistent, warp-specialised grouped GEMM on 5th-gen tensor
// cores (tcgen05.mma kind::f16, bf16 x bf16 -> fp32 in TMEM), operands staged
// by TMA (128-byte swizzle) through a 4-stage mbarrier ring, accumulators
// double-buffered in TMEM so the epilogue of tile i overlaps the MMAs of
// tile i+1. Epilogues fuse the expert FFN activations (GELU / SwiGLU) forward
// and backward. This is the only dense contraction on the MoE path (expert
// FFN: absent in the reference, which only counts GEMMs,
// proj/src/workload.cpp:70).
//
// Warp roles (256 threads, 1 CTA per SM):
//   warp 0      TMA producer (one elected lane)
//   warp 1      MMA issuer (one elected lane)
//   warp 2      TMEM allocator
//   warps 4..11 epilogue: TMEM -> registers -> activation -> global; warp w
//               reads TMEM lane quarter w%4 and column half (w-4)/4
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>

#include "gemm.h"
#include "sm100.cuh"

namespace fsmoe {
namespace {

using namespace fsmoe_dev;

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_STAGE_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int NUM_THREADS = 384;
constexpr int EPI_THREADS = 256;  // 8 epilogue warps
constexpr int TMEM_COLS = 512;  // 2 accumulators x 256 fp32 columns
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

struct KParams {
  int kind;  // GemmKind
  int nblk, rows, K, N, Mo, No, n_w;
  int b_mn;
  const long long* valid;
  int m_tiles, n_tiles, n_groups, num_tiles;
  int epi;
  void* D;
  void* D2;
  const void* Zin;
  long long ldd, ldd2, ldz;
  int rows_total, row0;  // block row window (see gemm.h)
  int accumulate;
  int out_rows, out_cols;  // valid output extent per group
};

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Valid rows of block b inside the processed window [row0, row0 + rows).
__device__ __forceinline__ int valid_of(const KParams& p, int b) {
  if (!p.valid) return p.rows;
  long long v = p.valid[b] - p.row0;
  return v < 0 ? 0 : (v > p.rows ? p.rows : static_cast<int>(v));
}

struct TileInfo {
  int g, mt, nt;
  bool skip;
};

__device__ __forceinline__ TileInfo decode_tile(const KParams& p, int t) {
  TileInfo ti;
  int per_g = p.m_tiles * p.n_tiles;
  ti.g = t / per_g;
  int rem = t - ti.g * per_g;
  ti.mt = rem / p.n_tiles;
  ti.nt = rem - ti.mt * p.n_tiles;
  ti.skip = false;
  if (p.kind == 0) ti.skip = ti.mt * BM >= valid_of(p, ti.g);
  return ti;
}

// Number of BK-wide k-blocks of block b (k-grouped) -- rows up to round_up(valid, 64).
__device__ __forceinline__ int kblocks_of_block(const KParams& p, int b) {
  int v = valid_of(p, b);
  return ceil_div(v, BK);
}

__device__ __forceinline__ int total_kblocks(const KParams& p, int g) {
  if (p.kind == 0) return ceil_div(p.K, BK);
  int n = 0;
  for (int b = g; b < p.nblk; b += p.n_w) n += kblocks_of_block(p, b);
  return n;
}

__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }

__device__ __forceinline__ float gelu_f(float z) {
  return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f));
}
__device__ __forceinline__ float gelu_grad_f(float z) {
  float cdf = 0.5f * (1.0f + erff(z * 0.70710678118654752f));
  float pdf = 0.39894228040143268f * __expf(-0.5f * z * z);
  return cdf + z * pdf;
}
__device__ __forceinline__ float sigmoid_f(float z) { return 1.0f / (1.0f + __expf(-z)); }

__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float* v) {
  uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[i * 8 + 2 * j], v[i * 8 + 2 * j + 1]);
    d4[i] = *reinterpret_cast<uint4*>(h);
  }
}

__device__ __forceinline__ void load_bf16x32(const __nv_bfloat16* src, float* v) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 u = s4[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(h[j]);
      v[i * 8 + 2 * j] = f.x;
      v[i * 8 + 2 * j + 1] = f.y;
    }
  }
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const KParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const bool a_mn = (p.kind == 1);
  const bool b_mn = (p.kind == 1) || p.b_mn;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], EPI_THREADS);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        TileInfo ti = decode_tile(p, t);
        if (ti.skip) continue;
        if (p.kind == 0) {
          const int nkb = ceil_div(p.K, BK);
          const int w = ti.g % p.n_w;
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&empty_bar[s], ph ^ 1);
            uint8_t* sa = smem + s * STAGE_BYTES;
            uint8_t* sb = sa + A_STAGE_BYTES;
            mbar_arrive_expect_tx(&full_bar[s], STAGE_BYTES);
            tma_load_3d(sa, &tmA, &full_bar[s], kb * BK, p.row0 + ti.mt * BM, ti.g);
            if (!b_mn) {
              tma_load_3d(sb, &tmB, &full_bar[s], kb * BK, ti.nt * BN, w);
            } else {
#pragma unroll
              for (int i = 0; i < BN / 64; ++i)
                tma_load_3d(sb + i * 8192, &tmB, &full_bar[s], ti.nt * BN + i * 64, kb * BK, w);
            }
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
        } else {
          for (int b = ti.g; b < p.nblk; b += p.n_w) {
            const int nkb = kblocks_of_block(p, b);
            for (int kb = 0; kb < nkb; ++kb) {
              mbar_wait(&empty_bar[s], ph ^ 1);
              uint8_t* sa = smem + s * STAGE_BYTES;
              uint8_t* sb = sa + A_STAGE_BYTES;
              mbar_arrive_expect_tx(&full_bar[s], STAGE_BYTES);
#pragma unroll
              for (int i = 0; i < BM / 64; ++i)
                tma_load_3d(sa + i * 8192, &tmA, &full_bar[s], ti.mt * BM + i * 64, p.row0 + kb * BK, b);
#pragma unroll
              for (int i = 0; i < BN / 64; ++i)
                tma_load_3d(sb + i * 8192, &tmB, &full_bar[s], ti.nt * BN + i * 64, p.row0 + kb * BK, b);
              if (++s == STAGES) { s = 0; ph ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t idesc = make_idesc_bf16(BM, BN, a_mn, b_mn);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t aph = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      TileInfo ti = decode_tile(p, t);
      if (ti.skip) continue;
      const int nkb = total_kblocks(p, ti.g);
      mbar_wait(&tempty_bar[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t dtmem = tmem_base + acc * BN;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t sb = sa + A_STAGE_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t ad = a_mn ? make_sdesc_sw128(sa + k * 2048, 8192, 1024)
                               : make_sdesc_sw128(sa + k * 32, 16, 1024);
            uint64_t bd = b_mn ? make_sdesc_sw128(sb + k * 2048, 8192, 1024)
                               : make_sdesc_sw128(sb + k * 32, 16, 1024);
            umma_bf16(dtmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty_bar[s]);
        }
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
      if (elect_one()) {
        if (nkb > 0) umma_commit(&tfull_bar[acc]);
        else mbar_arrive(&tfull_bar[acc]);
      }
      __syncwarp();
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;  // which 128 accumulator columns
    const int lane = threadIdx.x & 31;
    int acc = 0;
    uint32_t aph = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      TileInfo ti = decode_tile(p, t);
      if (ti.skip) continue;
      const int nkb = total_kblocks(p, ti.g);
      mbar_wait(&tfull_bar[acc], aph);
      tc_fence_after();
      const int row = ti.mt * BM + q * 32 + lane;  // within the processed window
      const bool row_ok = row < p.out_rows;
      const long long orow = p.kind == 0
                                 ? static_cast<long long>(ti.g) * p.rows_total + p.row0 + row
                                 : static_cast<long long>(ti.g) * p.Mo + row;
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      uint32_t r[32];
      float v[32];
      if (p.epi == static_cast<int>(Epi::SwigluFwd)) {
        // tile cols: [0,128) gate units, [128,256) up units (same 128 units)
        __nv_bfloat16* Z = static_cast<__nv_bfloat16*>(p.D) + orow * p.ldd;
        __nv_bfloat16* H = static_cast<__nv_bfloat16*>(p.D2) +
                           orow * p.ldd2;
        for (int c = 2 * half; c < 2 * half + 2; ++c) {
          float g[32];
          if (nkb > 0) {
            tmem_ld_32x32b_x32(tbase + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) g[i] = __uint_as_float(r[i]);
            tmem_ld_32x32b_x32(tbase + 128 + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) g[i] = v[i] = 0.f;
          }
          const int gcol = ti.nt * BN + c * 32;
          const int unit = ti.nt * (BN / 2) + c * 32;
          if (row_ok && gcol < p.out_cols) {
            store_bf16x32(Z + gcol, g);
            store_bf16x32(Z + gcol + 128, v);
            float h[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              float gb = bf2f(__float2bfloat16(g[i]));
              float ub = bf2f(__float2bfloat16(v[i]));
              h[i] = gb * sigmoid_f(gb) * ub;
            }
            store_bf16x32(H + unit, h);
          }
        }
      } else {
        for (int c = 4 * half; c < 4 * half + 4; ++c) {
          const int col = ti.nt * BN + c * 32;
          if (nkb > 0) {
            tmem_ld_32x32b_x32(tbase + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
          if (!row_ok || col >= p.out_cols) continue;
          switch (p.epi) {
            case static_cast<int>(Epi::StoreBF16): {
              __nv_bfloat16* D = static_cast<__nv_bfloat16*>(p.D) + orow * p.ldd;
              store_bf16x32(D + col, v);
              break;
            }
            case static_cast<int>(Epi::StoreF32): {
              float* D = static_cast<float*>(p.D) + orow * p.ldd + col;
              float4* d4 = reinterpret_cast<float4*>(D);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                float4 o = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                if (p.accumulate) {
                  float4 e = d4[i];
                  o.x += e.x; o.y += e.y; o.z += e.z; o.w += e.w;
                }
                d4[i] = o;
              }
              break;
            }
            case static_cast<int>(Epi::GeluFwd): {
              __nv_bfloat16* Z = static_cast<__nv_bfloat16*>(p.D) + orow * p.ldd;
              __nv_bfloat16* H = static_cast<__nv_bfloat16*>(p.D2) +
                                 orow * p.ldd2;
              store_bf16x32(Z + col, v);
              float h[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) h[i] = gelu_f(bf2f(__float2bfloat16(v[i])));
              store_bf16x32(H + col, h);
              break;
            }
            case static_cast<int>(Epi::GeluBwd): {
              const __nv_bfloat16* Z = static_cast<const __nv_bfloat16*>(p.Zin) +
                                       orow * p.ldz;
              __nv_bfloat16* dZ = static_cast<__nv_bfloat16*>(p.D) + orow * p.ldd;
              float z[32];
              load_bf16x32(Z + col, z);
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] *= gelu_grad_f(z[i]);
              store_bf16x32(dZ + col, v);
              break;
            }
            case static_cast<int>(Epi::SwigluBwd): {
              const int unit = col;
              const int gcol = (unit / 128) * 256 + (unit % 128);
              const __nv_bfloat16* Z = static_cast<const __nv_bfloat16*>(p.Zin) +
                                       orow * p.ldz;
              __nv_bfloat16* dZ = static_cast<__nv_bfloat16*>(p.D) + orow * p.ldd;
              float g[32], u[32], dg[32];
              load_bf16x32(Z + gcol, g);
              load_bf16x32(Z + gcol + 128, u);
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                float sg = sigmoid_f(g[i]);
                float silu = g[i] * sg;
                dg[i] = v[i] * u[i] * sg * (1.0f + g[i] * (1.0f - sg));
                u[i] = v[i] * silu;
              }
              store_bf16x32(dZ + gcol, dg);
              store_bf16x32(dZ + gcol + 128, u);
              break;
            }
            default:
              break;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------ host --

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &ptr, 12000,
                                         cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 3-D bf16 tensor map: dims {d0 (contiguous), d1, d2}, box {b0, b1, 1}.
bool make_map3(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
               uint32_t b0, uint32_t b1) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 2, d0 * d1 * 2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

int gemm_sm100_launch(const GemmProblem& pr, cudaStream_t stream) {
  KParams p{};
  CUtensorMap ta, tb;
  p.kind = static_cast<int>(pr.kind);
  p.nblk = pr.nblk;
  p.rows = pr.rows;
  p.K = pr.K;
  p.N = pr.N;
  p.Mo = pr.Mo;
  p.No = pr.No;
  p.n_w = pr.n_w > 0 ? pr.n_w : 1;
  p.b_mn = pr.b_mn_major ? 1 : 0;
  p.valid = pr.valid_rows;
  p.epi = static_cast<int>(pr.epi);
  p.D = pr.D;
  p.D2 = pr.D2;
  p.Zin = pr.Zin;
  p.ldd = pr.ldd;
  p.ldd2 = pr.ldd2;
  p.ldz = pr.ldz;
  p.accumulate = pr.accumulate ? 1 : 0;
  p.rows_total = pr.rows_total > 0 ? pr.rows_total : pr.rows;
  p.row0 = pr.row0;
  if (pr.nblk <= 0 || pr.rows <= 0) return cudaSuccess;
  if (p.row0 < 0 || p.row0 + pr.rows > p.rows_total || p.row0 % 64) return cudaErrorInvalidValue;
  if (pr.kind == GemmKind::KGrouped && p.row0 + pr.rows < p.rows_total && pr.rows % 64)
    return cudaErrorInvalidValue;  // the K window must end on a 64-row boundary
  if (pr.kind == GemmKind::RowGrouped) {
    if (pr.K % 8 || pr.N % 64 || pr.K <= 0 || pr.N <= 0) return cudaErrorInvalidValue;
    p.m_tiles = (pr.rows + BM - 1) / BM;
    p.n_tiles = (pr.N + BN - 1) / BN;
    p.n_groups = pr.nblk;
    p.out_rows = pr.rows;
    // SwigluBwd's output columns are the interleaved dZ (2N); masking is on N units.
    p.out_cols = pr.N;
    if (!make_map3(&ta, pr.A, pr.K, p.rows_total, pr.nblk, BK, BM)) return cudaErrorInvalidValue;
    if (!pr.b_mn_major) {
      if (!make_map3(&tb, pr.B, pr.K, pr.N, p.n_w, BK, BN)) return cudaErrorInvalidValue;
    } else {
      if (!make_map3(&tb, pr.B, pr.N, pr.K, p.n_w, 64, BK)) return cudaErrorInvalidValue;
    }
  } else {
    if (pr.Mo % 64 || pr.No % 64 || pr.nblk % p.n_w) return cudaErrorInvalidValue;
    p.m_tiles = (pr.Mo + BM - 1) / BM;
    p.n_tiles = (pr.No + BN - 1) / BN;
    p.n_groups = p.n_w;
    p.out_rows = pr.Mo;
    p.out_cols = pr.No;
    if (!make_map3(&ta, pr.A, pr.Mo, p.rows_total, pr.nblk, 64, BK)) return cudaErrorInvalidValue;
    if (!make_map3(&tb, pr.B, pr.No, p.rows_total, pr.nblk, 64, BK)) return cudaErrorInvalidValue;
  }
  p.num_tiles = p.n_groups * p.m_tiles * p.n_tiles;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(grouped_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SMEM_BYTES);
    attr_set = true;
  }
  int grid = p.num_tiles < num_sms() ? p.num_tiles : num_sms();
  grouped_gemm_kernel<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(ta, tb, p); ::fsmoe::count_launch();
  return static_cast<int>(cudaGetLastError());
}

}  // namespace fsmoe
