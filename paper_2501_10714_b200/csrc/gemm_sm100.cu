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
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gemm.h"
#include "host_once.h"
#include "sm100.cuh"

namespace fsmoe {
namespace {

using namespace fsmoe_dev;

constexpr int BM = 128;
constexpr int BN_MAX = 256;  // tile columns: 256, or 128 when 256 leaves a ragged last wave
constexpr int BK = 64;
constexpr int NUM_THREADS = 384;
constexpr int EPI_THREADS = 256;  // 8 epilogue warps

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
  int use_peers;           // row-grouped plain stores through `peers`
  fsmoe_dev::PeerRows peers;
  fsmoe_dev::RowRange blocks;  // row-grouped: the blocks this launch covers
  int band_m, band_n;  // tile order: bands of band_m m-tiles (n walked inside) or band_n n-tiles
  const int* scatter;  // StoreBF16 row scatter (fsmoe_gemm_desc::scatter_rows), or null
  void* sdst;
  long long sld;
  int dbg;  // measurement only (fsmoe_gemm_desc::dbg): 1 no epilogue after the TMEM reads,
            // 2 no TMEM reads either, 4 everything but the TMA stores
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

// GELU and its derivative from one exponential: Phi(z) = 0.5 (1 + erf(z/sqrt2))
// with erf by Abramowitz-Stegun 7.1.26 (|error| <= 1.5e-7, i.e. fp32-exact
// for bf16 outputs): erf(x) = 1 - poly(t) e^{-x^2}, t = 1 / (1 + p x), x >= 0.
// e^{-z^2/2} is both that exponential and sqrt(2 pi) * phi(z), so
//   gelu(z) = z Phi(z),  gelu'(z) = Phi(z) + z phi(z)
// cost 2 MUFU (rcp, ex2) + ~12 FMA instead of erff + expf per value.
__device__ __forceinline__ void gelu_and_grad(float z, float& h, float& g) {
  const float x = fabsf(z) * 0.70710678118654752f;
  const float t = __fdividef(1.0f, fmaf(0.3275911f, x, 1.0f));
  float poly = fmaf(1.061405429f, t, -1.453152027f);
  poly = fmaf(poly, t, 1.421413741f);
  poly = fmaf(poly, t, -0.284496736f);
  poly = fmaf(poly, t, 0.254829592f);
  poly *= t;
  const float e = __expf(-0.5f * z * z);
  const float tail = 0.5f * poly * e;  // 0.5 (1 - erf(x))
  const float cdf = z >= 0.f ? 1.0f - tail : tail;
  h = z * cdf;
  g = fmaf(z * 0.39894228040143268f, e, cdf);
}
// Packed fp32 pairs (FFMA2 / FMUL2 / FADD2, sm_100): two IEEE operations per
// instruction, which halves the epilogue's FP32 issue count.
__device__ __forceinline__ unsigned long long f2u(float2 v) {
  return *reinterpret_cast<unsigned long long*>(&v);
}
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }

__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// gelu_and_grad on a pair of values, same formula in paired arithmetic with
// the branch-free Phi(z) = 0.5 + sign(z) (0.5 - tail), tail = 0.5 poly(t) e
// (the 0.5 folded into the coefficients): ~13 instructions per value.
__device__ __forceinline__ void gelu_and_grad2(float2 z, float2& h, float2& g) {
  const float2 az = make_float2(fabsf(z.x), fabsf(z.y));
  const float2 den = fma2(az, bc2(0.3275911f * 0.70710678118654752f), bc2(1.0f));
  const float2 t = make_float2(rcp_approx(den.x), rcp_approx(den.y));
  float2 poly = fma2(bc2(0.5f * 1.061405429f), t, bc2(0.5f * -1.453152027f));
  poly = fma2(poly, t, bc2(0.5f * 1.421413741f));
  poly = fma2(poly, t, bc2(0.5f * -0.284496736f));
  poly = fma2(poly, t, bc2(0.5f * 0.254829592f));
  poly = mul2(poly, t);
  const float2 q = mul2(mul2(z, bc2(-0.5f * 1.4426950408889634f)), z);
  const float2 e = make_float2(ex2_approx(q.x), ex2_approx(q.y));
  const float2 u = fma2(mul2(poly, e), bc2(-1.0f), bc2(0.5f));  // 0.5 - tail >= 0
  const float2 su = make_float2(copysignf(u.x, z.x), copysignf(u.y, z.y));
  const float2 cdf = add2(su, bc2(0.5f));
  h = mul2(z, cdf);
  g = fma2(mul2(z, bc2(0.39894228040143268f)), e, cdf);
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

// CTAS = 1: one CTA computes a 128 x 256 tile (tcgen05 cta_group::1).
// CTAS = 2: a CTA pair (cluster of 2 on one TPC) computes a 256 x 256 tile
// with cta_group::2: each CTA stages its 128 rows of A and 128 of the 256
// B rows; the leader issues the MMAs and both TMEMs hold their 128 rows.
template <int CTAS, int BN_ = BN_MAX>
struct TileCfg {
  static constexpr int BM = 128 * CTAS;      // tile rows (whole pair)
  static constexpr int BN = BN_;             // tile columns
  // one tcgen05.mma covers at most 256 columns: a 512-column pair tile issues
  // two per K step, each over its own 256-row B segment (split over the pair)
  static constexpr int MMA_N = BN < 256 ? BN : 256;
  static constexpr int NSEG = BN / MMA_N;
  static constexpr int SEG_ROWS = MMA_N / CTAS;                // B rows per CTA per segment
  static constexpr int SEG_BYTES = SEG_ROWS * BK * 2;
  static constexpr int BN_CTA = BN / CTAS;   // B rows staged per CTA
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = BN_CTA * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STG_PER_WARP = 8192;                     // two 4 KB SW128 boxes
  static constexpr int STG_TOTAL = (EPI_THREADS / 32) * STG_PER_WARP;
  // as many stages as fit next to the epilogue boxes (<= 6)
  static constexpr int NS_FIT = (227 * 1024 - 2048 - STG_TOTAL) / STAGE;
  static constexpr int NSTAGE = NS_FIT > 6 ? 6 : NS_FIT;
  static constexpr int STG_OFF = NSTAGE * STAGE + 1024;         // after the barrier block
  static constexpr int SMEM = STG_OFF + STG_TOTAL + 1024;
  // double-buffered accumulator when two fit in the 512 TMEM columns; the
  // 512-column tile has one (the MMAs of the next tile wait for the drain)
  static constexpr int ACC_BUFS = 2 * BN <= 512 ? 2 : 1;
  static constexpr int TMEM_COLS = ACC_BUFS * BN;
};

// Epilogue tensor maps (TMA stores / loads of 32-row x 128-byte SW128 boxes):
// d = main output, d2 = GeluFwd's H, z = GeluBwd's saved gelu', peer[p] =
// rank p's receive buffer when the output rows belong to other GPUs.
struct EpiMaps {
  CUtensorMap d, d2, z;
  CUtensorMap peer[fsmoe_dev::MAX_PEERS];
};

template <int CTAS>
__device__ __forceinline__ TileInfo decode_tile_c(const KParams& p, int t) {
  // Tile order inside a group: bands of TILE_GM m-tiles, walked column by
  // column (m fastest), so the tiles in flight at once share a few A row
  // blocks and B column blocks that stay in L2 -- with m-major order every
  // m-tile streamed the whole B (a 235 MB Mixtral W1) again from HBM.
  // Only for wide problems (n-tiles > 2 bands): with few n-tiles the m-major
  // order already keeps the whole B in flight, and banding measured worse
  // there (ncu dram reads of the N = 4096 launches grew 1.4-2x).
  TileInfo ti;
  int per_g = p.m_tiles * p.n_tiles;
  ti.g = t / per_g;
  int rem = t - ti.g * per_g;
  if (p.band_m > 0) {
    const int bm = p.band_m;
    const int band = rem / (bm * p.n_tiles);
    const int m0 = band * bm;
    const int gm = min(bm, p.m_tiles - m0);
    const int idx = rem - band * bm * p.n_tiles;
    ti.mt = m0 + idx % gm;
    ti.nt = idx / gm;
  } else if (p.band_n > 0) {
    // bands of band_n n-tiles (a B panel set stays in L2), m walked inside
    const int bn = p.band_n;
    const int band = rem / (bn * p.m_tiles);
    const int n0 = band * bn;
    const int gn = min(bn, p.n_tiles - n0);
    const int idx = rem - band * bn * p.m_tiles;
    ti.nt = n0 + idx % gn;
    ti.mt = idx / gn;
  } else {
    ti.mt = rem / p.n_tiles;
    ti.nt = rem - ti.mt * p.n_tiles;
  }
  ti.skip = p.kind == 0 &&
            (ti.mt * TileCfg<CTAS>::BM >= valid_of(p, ti.g) || !fsmoe_dev::in_range(p.blocks, ti.g));
  return ti;
}

template <int CTAS, int BN_>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const KParams p,
                        const __grid_constant__ EpiMaps em) {
  using Cfg = TileCfg<CTAS, BN_>;
  constexpr int NS = Cfg::NSTAGE;
  constexpr int BN = BN_;
  constexpr int CPH = BN / 64;  // 32-column TMEM chunks per epilogue warp (half the tile)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + NS * Cfg::STAGE);
  uint64_t* empty_bar = full_bar + NS;
  uint64_t* tfull_bar = empty_bar + NS;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint64_t* zbar = tempty_bar + 3;        // [8 epilogue warps][2 boxes]: GeluBwd loads

  const int warp = threadIdx.x / 32;
  const bool a_mn = (p.kind == 1);
  const bool b_mn = (p.kind == 1) || p.b_mn;
  const uint32_t rank = CTAS == 2 ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int unit = blockIdx.x / CTAS;          // tile-scheduling unit (CTA or pair)
  const int nunits = gridDim.x / CTAS;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], (EPI_THREADS / 32) * CTAS);  // one arrive per epilogue warp
    }
    for (int i = 0; i < 2 * (EPI_THREADS / 32); ++i) mbar_init(&zbar[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CTAS == 2) tmem_alloc_pair<Cfg::TMEM_COLS>(tmem_slot);
    else tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (CTAS == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic dependent launch: the prologue above (barriers, TMEM,
  // descriptor prefetch) overlapped the previous kernel's tail; nothing
  // below may touch global memory before it has completed
  fsmoe_dev::pdl_enter();

  if (warp == 0) {
    // ===================== TMA producer (every CTA loads its half) ==========
    if (elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      const int arow = static_cast<int>(rank) * 128;          // this CTA's A rows in the tile
      const int brow = static_cast<int>(rank) * Cfg::SEG_ROWS;  // this CTA's B rows per segment
      auto issue = [&](uint8_t* dst, const CUtensorMap* m, int c0, int c1, int c2) {
        if constexpr (CTAS == 2) tma_load_3d_pair(dst, m, mapa_shared(&full_bar[s], 0), c0, c1, c2);
        else tma_load_3d(dst, m, &full_bar[s], c0, c1, c2);
      };
      auto begin_stage = [&]() {
        mbar_wait(&empty_bar[s], ph ^ 1);
        if (leader) mbar_arrive_expect_tx(&full_bar[s], Cfg::STAGE * CTAS);
      };
      for (int t = unit; t < p.num_tiles; t += nunits) {
        TileInfo ti = decode_tile_c<CTAS>(p, t);
        if (ti.skip) continue;
        if (p.kind == 0) {
          const int nkb = ceil_div(p.K, BK);
          const int w = ti.g % p.n_w;
          for (int kb = 0; kb < nkb; ++kb) {
            begin_stage();
            uint8_t* sa = smem + s * Cfg::STAGE;
            uint8_t* sb = sa + Cfg::A_BYTES;
            issue(sa, &tmA, kb * BK, p.row0 + ti.mt * Cfg::BM + arow, ti.g);
#pragma unroll
            for (int h = 0; h < Cfg::NSEG; ++h) {
              const int nrow = ti.nt * BN + h * Cfg::MMA_N + brow;
              uint8_t* sbh = sb + h * Cfg::SEG_BYTES;
              if (!b_mn) {
                issue(sbh, &tmB, kb * BK, nrow, w);
              } else {
#pragma unroll
                for (int i = 0; i < Cfg::SEG_ROWS / 64; ++i)
                  issue(sbh + i * 8192, &tmB, nrow + i * 64, kb * BK, w);
              }
            }
            if (++s == NS) { s = 0; ph ^= 1; }
          }
        } else {
          for (int b = ti.g; b < p.nblk; b += p.n_w) {
            const int nkb = kblocks_of_block(p, b);
            for (int kb = 0; kb < nkb; ++kb) {
              begin_stage();
              uint8_t* sa = smem + s * Cfg::STAGE;
              uint8_t* sb = sa + Cfg::A_BYTES;
#pragma unroll
              for (int i = 0; i < 2; ++i)
                issue(sa + i * 8192, &tmA, ti.mt * Cfg::BM + arow + i * 64, p.row0 + kb * BK, b);
#pragma unroll
              for (int h = 0; h < Cfg::NSEG; ++h)
#pragma unroll
                for (int i = 0; i < Cfg::SEG_ROWS / 64; ++i)
                  issue(sb + h * Cfg::SEG_BYTES + i * 8192, &tmB,
                        ti.nt * BN + h * Cfg::MMA_N + brow + i * 64, p.row0 + kb * BK, b);
              if (++s == NS) { s = 0; ph ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    if (leader) {
      const uint32_t idesc = make_idesc_bf16(Cfg::BM, Cfg::MMA_N, a_mn, b_mn);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int t = unit; t < p.num_tiles; t += nunits) {
        TileInfo ti = decode_tile_c<CTAS>(p, t);
        if (ti.skip) continue;
        const int nkb = total_kblocks(p, ti.g);
        mbar_wait(&tempty_bar[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t dtmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = smem_u32(smem + s * Cfg::STAGE);
            const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              uint64_t ad = a_mn ? make_sdesc_sw128(sa + k * 2048, 8192, 1024)
                                 : make_sdesc_sw128(sa + k * 32, 16, 1024);
#pragma unroll
              for (int h = 0; h < Cfg::NSEG; ++h) {
                const uint32_t sbh = sb + h * Cfg::SEG_BYTES;
                uint64_t bd = b_mn ? make_sdesc_sw128(sbh + k * 2048, 8192, 1024)
                                   : make_sdesc_sw128(sbh + k * 32, 16, 1024);
                const uint32_t dt = dtmem + h * Cfg::MMA_N;
                if constexpr (CTAS == 2) umma_bf16_pair(dt, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
                else umma_bf16(dt, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
              }
            }
            if constexpr (CTAS == 2) umma_commit_pair(&empty_bar[s], 0x3);
            else umma_commit(&empty_bar[s]);
          }
          __syncwarp();
          if (++s == NS) { s = 0; ph ^= 1; }
        }
        if (elect_one()) {
          if (nkb > 0) {
            if constexpr (CTAS == 2) umma_commit_pair(&tfull_bar[acc], 0x3);
            else umma_commit(&tfull_bar[acc]);
          } else {
            for (int r = 0; r < CTAS; ++r) mbar_arrive_cluster(mapa_shared(&tfull_bar[acc], r));
          }
        }
        __syncwarp();
        if (++acc == Cfg::ACC_BUFS) { acc = 0; aph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue (every CTA: its 128 TMEM lanes) ========
    // Warp (q, half) owns accumulator rows [32q, 32q+32) of this CTA and
    // columns [128 half, 128 half + 128) of the tile. Outputs leave through
    // TMA: the warp writes a 32-row x 128-byte box into shared memory in the
    // SW128 layout (16-byte unit k of row r at k ^ (r & 7): conflict-free with
    // one row per lane) and one lane issues the tensor store (or, for
    // accumulating fp32 wgrad outputs, the tensor reduce-add). Two boxes per
    // warp alternate so the next box is written while the last is in flight.
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int lane = threadIdx.x & 31;
    const int wi = warp - 4;
    uint8_t* stg = smem + Cfg::STG_OFF + wi * Cfg::STG_PER_WARP;
    uint64_t* zb = zbar + 2 * wi;
    uint32_t zph[2] = {0u, 0u};
    const uint32_t tempty_leader = mapa_shared(&tempty_bar[0], 0);
    const bool tma_epi = p.epi == static_cast<int>(Epi::StoreBF16) ||
                         p.epi == static_cast<int>(Epi::StoreF32) ||
                         p.epi == static_cast<int>(Epi::GeluFwd) ||
                         p.epi == static_cast<int>(Epi::GeluBwd) ||
                         p.epi == static_cast<int>(Epi::AddBF16);
    // GeluBwd and AddBF16 combine the accumulator with a loaded bf16 box
    const bool zbox_epi = p.epi == static_cast<int>(Epi::GeluBwd) || p.epi == static_cast<int>(Epi::AddBF16);
    // this lane's row inside a box: unit k of the row lives at (k ^ (lane & 7))
    auto box_row = [&](uint8_t* box) { return reinterpret_cast<uint4*>(box + lane * 128); };
    auto store_box = [&](const CUtensorMap* m, const void* box, int x0, int x1, int x2) {
      if (p.dbg != 4) tma_store_3d(m, box, x0, x1, x2);
    };
    const int sw = lane & 7;
    int acc = 0;
    uint32_t aph = 0;
    for (int t = unit; t < p.num_tiles; t += nunits) {
      TileInfo ti = decode_tile_c<CTAS>(p, t);
      if (ti.skip) continue;
      const int nkb = total_kblocks(p, ti.g);
      const int rloc = ti.mt * Cfg::BM + static_cast<int>(rank) * 128 + q * 32;  // first row of the warp
      // TMA box coordinates of the warp's rows: (col, row, block)
      int c1 = p.kind == 0 ? p.row0 + rloc : rloc;
      int c2 = ti.g;
      const CUtensorMap* md = &em.d;
      if (p.use_peers) {
        const int pp = ti.g / p.peers.el;
        c2 = p.peers.rank * p.peers.el + (ti.g - pp * p.peers.el);
        md = &em.peer[pp];
      }
      if (p.epi == static_cast<int>(Epi::SwigluBwd)) {
        // prefetch this warp's first saved gate / up box pair while the MMAs run
        const int col = ti.nt * BN + CPH * half * 32;
        if (lane == 0 && col < p.out_cols) {
          const int gcol = (col / 128) * 256 + (col % 128);
          bulk_wait_read<0>();  // the previous tile's stores have left the boxes
          mbar_arrive_expect_tx(&zb[0], 4096);
          tma_load_3d(stg, &em.z, &zb[0], gcol, c1, ti.g);
          mbar_arrive_expect_tx(&zb[1], 4096);
          tma_load_3d(stg + 4096, &em.z, &zb[1], gcol + 128, c1, ti.g);
        }
        __syncwarp();
      }
      if (zbox_epi) {
        // prefetch this warp's saved gelu'(Z) (or addend) boxes while the MMAs still run
        if (lane == 0) {
          bulk_wait_read<0>();  // the previous tile's stores have left the boxes
#pragma unroll
          for (int pc = 0; pc < CPH / 2; ++pc) {
            const int col = ti.nt * BN + (CPH * half + 2 * pc) * 32;
            if (col < p.out_cols) {
              mbar_arrive_expect_tx(&zb[pc], 4096);
              tma_load_3d(stg + pc * 4096, &em.z, &zb[pc], col, c1, ti.g);
            }
          }
        }
        __syncwarp();
      }
      mbar_wait(&tfull_bar[acc], aph);
      tc_fence_after();
      const int row = rloc + lane;
      const bool row_ok = row < p.out_rows;
      const long long orow = p.kind == 0
                                 ? static_cast<long long>(ti.g) * p.rows_total + p.row0 + row
                                 : static_cast<long long>(ti.g) * p.Mo + row;
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      // row scatter: this lane's output row goes to row sdst_row of p.sdst
      const int sdst_row = (p.scatter && row_ok) ? p.scatter[orow] : -1;
      uint32_t r[32];
      float v[32];
      // hand the accumulator back to the MMA warp as soon as this warp's last
      // TMEM read of the tile has landed (the rest works from registers)
      bool released = false;
      auto release_acc = [&]() {
        tc_fence_before();
        __syncwarp();
        // the tcgen05 fence orders this warp's (completed) TMEM reads before
        // the hand-off; nothing else needs ordering, so the arrive is relaxed
        // (a release arrive costs a MEMBAR + ERRBAR per warp per tile)
        if (lane == 0) {
          if constexpr (CTAS == 2) mbar_arrive_cluster_relaxed(tempty_leader + acc * 8);
          else mbar_arrive_relaxed(&tempty_bar[acc]);
        }
        released = true;
      };
      if (tma_epi && p.epi == static_cast<int>(Epi::StoreF32)) {
        // fp32: one 32-column TMEM chunk = one box
        for (int c = CPH * half; c < CPH * half + CPH; ++c) {
          const int col = ti.nt * BN + c * 32;
          if (p.dbg == 2) break;
          if (nkb > 0) {
            tmem_ld_32x32b_x32(tbase + c * 32, r);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = 0u;
          }
          if (c == CPH * half + CPH - 1) release_acc();
          if (col >= p.out_cols) continue;  // warp-uniform
          if (p.dbg == 1) {
            if (lane == 0 && (r[0] ^ r[31]) == 0x7fc00001u) r[1] = 0;  // keep the loads
            continue;
          }
          uint8_t* box = stg + (c & 1) * 4096;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          uint4* br = box_row(box);
#pragma unroll
          for (int k = 0; k < 8; ++k) br[k ^ sw] = make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (p.accumulate) tma_reduce_add_3d(md, box, col, c1, c2);
            else store_box(md, box, col, c1, c2);
            bulk_commit();
          }
        }
      } else if (tma_epi) {
        // bf16: two TMEM chunks (64 columns) = one box
        for (int pc = 0; pc < CPH / 2; ++pc) {
          const int c = CPH * half + 2 * pc;
          const int col = ti.nt * BN + c * 32;
          uint32_t r2[32];
          if (p.dbg == 2) break;
          if (nkb > 0) {
            tmem_ld_32x32b_x32(tbase + c * 32, r);
            tmem_ld_32x32b_x32(tbase + (c + 1) * 32, r2);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = r2[i] = 0u;
          }
          if (pc == CPH / 2 - 1) release_acc();
          if (col >= p.out_cols) continue;  // warp-uniform
          auto pk = [&](float a, float b) {
            __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
            return *reinterpret_cast<uint32_t*>(&h);
          };
          auto val = [&](int i) { return __uint_as_float(i < 32 ? r[i] : r2[i - 32]); };
          if (p.dbg == 1) {
            if (lane == 0 && (r[0] ^ r2[31]) == 0x7fc00001u) r[1] = 0;  // keep the loads
            continue;
          }
          if (p.epi == static_cast<int>(Epi::StoreBF16) && p.scatter) {
            // top-1 combine fused: the row's 64 columns straight to its token
            // row (one full 128-byte line per lane); dropped / padding rows skip
            if (sdst_row >= 0) {
              uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.sdst) +
                                                  static_cast<long long>(sdst_row) * p.sld + col);
#pragma unroll
              for (int k = 0; k < 8; ++k)
                o[k] = make_uint4(pk(val(8 * k), val(8 * k + 1)), pk(val(8 * k + 2), val(8 * k + 3)),
                                  pk(val(8 * k + 4), val(8 * k + 5)), pk(val(8 * k + 6), val(8 * k + 7)));
            }
          } else if (p.epi == static_cast<int>(Epi::StoreBF16)) {
            uint8_t* box = stg + (pc & 1) * 4096;
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            uint4* br = box_row(box);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              br[k ^ sw] = make_uint4(pk(val(8 * k), val(8 * k + 1)), pk(val(8 * k + 2), val(8 * k + 3)),
                                      pk(val(8 * k + 4), val(8 * k + 5)), pk(val(8 * k + 6), val(8 * k + 7)));
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              store_box(md, box, col, c1, c2);
              bulk_commit();
            }
          } else if (p.epi == static_cast<int>(Epi::GeluFwd)) {
            // box 0: gelu'(Z) (saved for the backward), box 1: H = gelu(Z)
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
            uint4* bg = box_row(stg);
            uint4* bh = box_row(stg + 4096);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              uint32_t hp[4], gp[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                // the bf16-rounded Z (what the backward sees) as a pair
                __nv_bfloat162 zb = __floats2bfloat162_rn(val(8 * k + 2 * j), val(8 * k + 2 * j + 1));
                float2 h2, g2;
                gelu_and_grad2(__bfloat1622float2(zb), h2, g2);
                hp[j] = pk(h2.x, h2.y);
                gp[j] = pk(g2.x, g2.y);
              }
              bg[k ^ sw] = make_uint4(gp[0], gp[1], gp[2], gp[3]);
              bh[k ^ sw] = make_uint4(hp[0], hp[1], hp[2], hp[3]);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              store_box(md, stg, col, c1, c2);
              store_box(&em.d2, stg + 4096, col, c1, c2);
              bulk_commit();
            }
          } else {  // GeluBwd: dZ = dH * gelu'(Z); AddBF16: D = acc + Zin; over the loaded box
            uint8_t* box = stg + pc * 4096;
            mbar_wait(&zb[pc], zph[pc]);
            zph[pc] ^= 1u;
            uint4* br = box_row(box);
            const bool add = p.epi == static_cast<int>(Epi::AddBF16);
            auto op = [&](float a, float z) { return add ? a + z : a * z; };
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              uint4 gw = br[k ^ sw];
              const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gw);
              float2 g0 = __bfloat1622float2(g2[0]), g1 = __bfloat1622float2(g2[1]);
              float2 g2f = __bfloat1622float2(g2[2]), g3 = __bfloat1622float2(g2[3]);
              br[k ^ sw] = make_uint4(pk(op(val(8 * k), g0.x), op(val(8 * k + 1), g0.y)),
                                      pk(op(val(8 * k + 2), g1.x), op(val(8 * k + 3), g1.y)),
                                      pk(op(val(8 * k + 4), g2f.x), op(val(8 * k + 5), g2f.y)),
                                      pk(op(val(8 * k + 6), g3.x), op(val(8 * k + 7), g3.y)));
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              store_box(md, box, col, c1, c2);
              bulk_commit();
            }
          }
        }
      } else if (p.epi == static_cast<int>(Epi::SwigluFwd)) {
        // every 256 tile columns: [0,128) gate units, [128,256) up units (the
        // same 128 units). A 256-column tile splits its 128 units over the two
        // warp halves; a 512-column tile gives each half one 256-column block.
        // Per 64 units (two 32-column TMEM chunks): the bf16 gate and up
        // pre-activations go out as two 32-row x 128-byte TMA boxes (Z), then
        // H = silu(gate) * up (from the bf16-rounded values the backward
        // sees) as a third box through the first buffer once its store read.
        constexpr int NSUB = BN >= 256 ? BN / 256 : 1;
        const int sub = NSUB == 2 ? half : 0;
        const int c_lo = NSUB == 2 ? 0 : 2 * half;
        const int c_hi = c_lo + (NSUB == 2 ? 4 : 2);
        const uint32_t tsub = tbase + sub * 256;
        uint4* bz0 = box_row(stg);
        uint4* bz1 = box_row(stg + 4096);
        for (int c = c_lo; c < c_hi; c += 2) {
          const int gcol = ti.nt * BN + sub * 256 + c * 32;
          const int hcol = ti.nt * (BN / 2) + sub * 128 + c * 32;
          if (lane == 0) bulk_wait_read<0>();  // both buffers free
          __syncwarp();
          uint32_t gp[32];  // bf16 pairs: gate of the two chunks
          uint32_t hp[32];  // bf16 pairs: H of the two chunks
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (nkb > 0) {
              tmem_ld_32x32b_x32(tsub + (c + j) * 32, r);
              tmem_ld_wait();
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) r[i] = 0u;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
              gp[16 * j + i] = *reinterpret_cast<uint32_t*>(&h2);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
              bz0[(4 * j + k) ^ sw] = make_uint4(gp[16 * j + 4 * k], gp[16 * j + 4 * k + 1],
                                                 gp[16 * j + 4 * k + 2], gp[16 * j + 4 * k + 3]);
            if (nkb > 0) {
              tmem_ld_32x32b_x32(tsub + 128 + (c + j) * 32, r);
              tmem_ld_wait();
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) r[i] = 0u;
            }
            if (j == 1 && c + 2 >= c_hi) release_acc();
            uint32_t up[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              __nv_bfloat162 u2 = __floats2bfloat162_rn(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
              up[i] = *reinterpret_cast<uint32_t*>(&u2);
              const float2 gb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gp[16 * j + i]));
              const float2 ub = __bfloat1622float2(u2);
              __nv_bfloat162 h2 = __floats2bfloat162_rn(gb.x * sigmoid_f(gb.x) * ub.x,
                                                        gb.y * sigmoid_f(gb.y) * ub.y);
              hp[16 * j + i] = *reinterpret_cast<uint32_t*>(&h2);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
              bz1[(4 * j + k) ^ sw] = make_uint4(up[4 * k], up[4 * k + 1], up[4 * k + 2], up[4 * k + 3]);
          }
          if (gcol >= p.out_cols) continue;  // warp-uniform (after the TMEM reads)
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            store_box(md, stg, gcol, c1, c2);
            store_box(md, stg + 4096, gcol + 128, c1, c2);
            bulk_commit();
            bulk_wait_read<0>();
          }
          __syncwarp();
#pragma unroll
          for (int k = 0; k < 8; ++k)
            bz0[k ^ sw] = make_uint4(hp[4 * k], hp[4 * k + 1], hp[4 * k + 2], hp[4 * k + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            store_box(&em.d2, stg, hcol, c1, c2);
            bulk_commit();
          }
        }
      } else {  // SwigluBwd: acc = dH over H units; dZ at the interleaved gate/up columns
        // Per 64 units: the saved bf16 gate / up boxes come in by TMA (the
        // first pair was prefetched while the MMAs ran), dG / dU are written
        // over them and go back out to the same place (dZ over Z).
        for (int pc = 0; pc < CPH / 2; ++pc) {
          const int c = CPH * half + 2 * pc;
          const int col = ti.nt * BN + c * 32;
          const int gcol = (col / 128) * 256 + (col % 128);
          uint32_t r2[32];
          if (nkb > 0) {
            tmem_ld_32x32b_x32(tbase + c * 32, r);
            tmem_ld_32x32b_x32(tbase + (c + 1) * 32, r2);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = r2[i] = 0u;
          }
          if (pc == CPH / 2 - 1) release_acc();
          if (col >= p.out_cols) continue;  // warp-uniform
          if (pc > 0) {  // this pair was not prefetched: load it now
            if (lane == 0) {
              bulk_wait_read<0>();
              mbar_arrive_expect_tx(&zb[0], 4096);
              tma_load_3d(stg, &em.z, &zb[0], gcol, c1, ti.g);
              mbar_arrive_expect_tx(&zb[1], 4096);
              tma_load_3d(stg + 4096, &em.z, &zb[1], gcol + 128, c1, ti.g);
            }
            __syncwarp();
          }
          mbar_wait(&zb[0], zph[0]);
          zph[0] ^= 1u;
          mbar_wait(&zb[1], zph[1]);
          zph[1] ^= 1u;
          uint4* bg = box_row(stg);
          uint4* bu = box_row(stg + 4096);
          auto dv = [&](int i) { return __uint_as_float(i < 32 ? r[i] : r2[i - 32]); };
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            uint4 gw = bg[k ^ sw], uw = bu[k ^ sw];
            const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gw);
            const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uw);
            uint32_t og[4], ou[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 g = __bfloat1622float2(g2[j]);
              const float2 u = __bfloat1622float2(u2[j]);
              const float d0 = dv(8 * k + 2 * j), d1 = dv(8 * k + 2 * j + 1);
              const float s0 = sigmoid_f(g.x), s1 = sigmoid_f(g.y);
              __nv_bfloat162 dg = __floats2bfloat162_rn(d0 * u.x * s0 * (1.0f + g.x * (1.0f - s0)),
                                                        d1 * u.y * s1 * (1.0f + g.y * (1.0f - s1)));
              __nv_bfloat162 du = __floats2bfloat162_rn(d0 * (g.x * s0), d1 * (g.y * s1));
              og[j] = *reinterpret_cast<uint32_t*>(&dg);
              ou[j] = *reinterpret_cast<uint32_t*>(&du);
            }
            bg[k ^ sw] = make_uint4(og[0], og[1], og[2], og[3]);
            bu[k ^ sw] = make_uint4(ou[0], ou[1], ou[2], ou[3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            store_box(md, stg, gcol, c1, c2);
            store_box(md, stg + 4096, gcol + 128, c1, c2);
            bulk_commit();
          }
        }
      }
      if (!released) release_acc();
      if (++acc == Cfg::ACC_BUFS) { acc = 0; aph ^= 1; }
    }
    if (lane == 0) bulk_wait<0>();  // outputs written before the kernel retires
    __syncwarp();
  }

  tc_fence_before();
  if constexpr (CTAS == 2) cluster_sync();
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CTAS == 2) tmem_dealloc_pair<Cfg::TMEM_COLS>(tmem_base);
    else tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
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

// General 3-D map: element type, dims {d0 (contiguous), d1, d2}, byte strides of
// dims 1 and 2, box {b0, b1, 1}, 128-byte swizzle (the epilogue box layout).
bool make_map3s(CUtensorMap* m, const void* base, bool f32, uint64_t d0, uint64_t d1, uint64_t d2,
                uint64_t s1, uint64_t s2, uint32_t b0, uint32_t b1) {
  auto enc = get_encode_fn();
  if (!enc || !base) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  return device_sms();
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
  p.dbg = pr.dbg;
  p.scatter = pr.scatter_rows;
  p.sdst = pr.scatter_out;
  p.sld = pr.scatter_ld;
  p.D = pr.D;
  p.D2 = pr.D2;
  p.Zin = pr.Zin;
  p.ldd = pr.ldd;
  p.ldd2 = pr.ldd2;
  p.ldz = pr.ldz;
  p.accumulate = pr.accumulate ? 1 : 0;
  p.use_peers = pr.use_peers ? 1 : 0;
  p.peers = pr.peers;
  p.blocks = pr.blocks;
  p.rows_total = pr.rows_total > 0 ? pr.rows_total : pr.rows;
  p.row0 = pr.row0;
  if (pr.nblk <= 0 || pr.rows <= 0) return cudaSuccess;
  if (p.row0 < 0 || p.row0 + pr.rows > p.rows_total || p.row0 % 64) return cudaErrorInvalidValue;
  if (pr.kind == GemmKind::KGrouped && p.row0 + pr.rows < p.rows_total && pr.rows % 64)
    return cudaErrorInvalidValue;  // the K window must end on a 64-row boundary
  // Tile shape: CTA pairs (256 x 256, cta_group::2) unless the problem is too
  // small to give every SM pair work; fsmoe_gemm_desc::force_ctas forces a variant.
  const int units_rows = pr.kind == GemmKind::RowGrouped ? pr.rows : pr.Mo;
  const int units_cols = pr.kind == GemmKind::RowGrouped ? pr.N : pr.No;
  const int groups = pr.kind == GemmKind::RowGrouped ? pr.nblk : p.n_w;
  long long pair_tiles = static_cast<long long>(groups) * ((units_rows + 255) / 256) *
                         ((units_cols + BN_MAX - 1) / BN_MAX);
  int ctas = pair_tiles >= num_sms() / 4 ? 2 : 1;
  if (pr.force_ctas) ctas = pr.force_ctas == 1 ? 1 : 2;
  // Tile width. Pairs take 512-column tiles (two MMAs per K step, one
  // accumulator: 25 % less operand traffic per flop than 256 columns) for the
  // plain bf16 and fp32 epilogues when that still gives every pair a tile:
  // measured 2-3 % faster on the configs[1] launches and 8-18 % on the
  // configs[2] ones (profiles/r01_gemm_bn512.md). The GELU / SwiGLU epilogues
  // keep 256 columns and double-buffered accumulators (their epilogue is long
  // enough that the single-accumulator drain shows). 128-column tiles
  // (force_bn = 128) measured slower everywhere. force_bn = 128|256|512
  // forces a width (512: every epilogue but GELU-backward).
  int BN = BN_MAX;
  const bool plain_epi = pr.epi == Epi::StoreBF16 || pr.epi == Epi::StoreF32;
  if (ctas == 2 && plain_epi) {
    const long long tiles512 = static_cast<long long>(groups) * ((units_rows + 255) / 256) *
                               ((units_cols + 511) / 512);
    if (tiles512 >= num_sms() / 2) BN = 512;
  }
  if (pr.force_bn) {
    const int want = pr.force_bn;
    if (want == 128 && pr.epi != Epi::SwigluFwd && pr.epi != Epi::SwigluBwd) BN = 128;
    else if (want == 256) BN = 256;
    else if (want == 512 && ctas == 2 && pr.epi != Epi::GeluBwd && pr.epi != Epi::AddBF16) BN = 512;
  }
  const int bm = 128 * ctas, bn_seg = (BN < 256 ? BN : 256) / ctas;  // B box rows per segment
  if (pr.kind == GemmKind::RowGrouped) {
    if (pr.K % 8 || pr.N % 64 || pr.K <= 0 || pr.N <= 0) return cudaErrorInvalidValue;
    p.m_tiles = (pr.rows + bm - 1) / bm;
    p.n_tiles = (pr.N + BN - 1) / BN;
    p.n_groups = pr.nblk;
    p.out_rows = pr.rows;
    // SwigluBwd's output columns are the interleaved dZ (2N); masking is on N units.
    p.out_cols = pr.N;
    if (!make_map3(&ta, pr.A, pr.K, p.rows_total, pr.nblk, BK, 128)) return cudaErrorInvalidValue;
    if (!pr.b_mn_major) {
      if (!make_map3(&tb, pr.B, pr.K, pr.N, p.n_w, BK, bn_seg)) return cudaErrorInvalidValue;
    } else {
      if (!make_map3(&tb, pr.B, pr.N, pr.K, p.n_w, 64, BK)) return cudaErrorInvalidValue;
    }
  } else {
    if (pr.Mo % 64 || pr.No % 64 || pr.nblk % p.n_w) return cudaErrorInvalidValue;
    p.m_tiles = (pr.Mo + bm - 1) / bm;
    p.n_tiles = (pr.No + BN - 1) / BN;
    p.n_groups = p.n_w;
    p.out_rows = pr.Mo;
    p.out_cols = pr.No;
    if (!make_map3(&ta, pr.A, pr.Mo, p.rows_total, pr.nblk, 64, BK)) return cudaErrorInvalidValue;
    if (!make_map3(&tb, pr.B, pr.No, p.rows_total, pr.nblk, 64, BK)) return cudaErrorInvalidValue;
  }
  p.num_tiles = p.n_groups * p.m_tiles * p.n_tiles;
  // Tile order inside a group. Default: bands of 8 m-tiles walked column by
  // column for wide launches (> 16 n-tiles), m-major otherwise (see
  // decode_tile_c). fsmoe_gemm_desc::band_m / band_n override it (band_m < 0:
  // plain m-major).
  p.band_m = p.m_tiles >= 16 && p.n_tiles > 16 ? 8 : 0;
  p.band_n = 0;
  if (pr.band_m > 0) {
    p.band_m = pr.band_m;
  } else if (pr.band_n > 0) {
    p.band_m = 0;
    p.band_n = pr.band_n;
  } else if (pr.band_m < 0) {
    p.band_m = 0;
  }
  // epilogue maps: 32-row boxes of 128 bytes (64 bf16 / 32 fp32 columns); the
  // row extent ends at the window so TMA clips rows outside [row0, row0+rows)
  EpiMaps em;
  memset(&em, 0, sizeof(em));
  {
    const bool f32 = pr.epi == Epi::StoreF32;
    const uint64_t es = f32 ? 4 : 2;
    const uint32_t bc = f32 ? 32 : 64;
    if (pr.epi == Epi::SwigluFwd || pr.epi == Epi::SwigluBwd) {
      // Z (2N interleaved gate / up columns, or N of them for the forward's
      // N = 2H launch) and H boxes: 32 rows x 64 bf16
      const uint64_t rows_end = static_cast<uint64_t>(p.row0) + pr.rows;
      const uint64_t zcols = pr.epi == Epi::SwigluFwd ? static_cast<uint64_t>(pr.N) : 2ULL * pr.N;
      if (!make_map3s(&em.d, pr.D, false, zcols, rows_end, pr.nblk, pr.ldd * 2,
                      static_cast<uint64_t>(p.rows_total) * pr.ldd * 2, 64, 32))
        return cudaErrorInvalidValue;
      if (pr.epi == Epi::SwigluFwd &&
          !make_map3s(&em.d2, pr.D2, false, pr.N / 2, rows_end, pr.nblk, pr.ldd2 * 2,
                      static_cast<uint64_t>(p.rows_total) * pr.ldd2 * 2, 64, 32))
        return cudaErrorInvalidValue;
      if (pr.epi == Epi::SwigluBwd &&
          !make_map3s(&em.z, pr.Zin, false, zcols, rows_end, pr.nblk, pr.ldz * 2,
                      static_cast<uint64_t>(p.rows_total) * pr.ldz * 2, 64, 32))
        return cudaErrorInvalidValue;
    }
    const bool tma_epi = pr.epi == Epi::StoreBF16 || pr.epi == Epi::StoreF32 ||
                         pr.epi == Epi::GeluFwd || pr.epi == Epi::GeluBwd || pr.epi == Epi::AddBF16;
    if (tma_epi) {
      if (pr.kind == GemmKind::RowGrouped) {
        const uint64_t rows_end = static_cast<uint64_t>(p.row0) + pr.rows;
        const uint64_t s1 = pr.ldd * es, s2 = static_cast<uint64_t>(p.rows_total) * pr.ldd * es;
        if (pr.use_peers) {
          const int blocks = pr.peers.world * pr.peers.el;
          for (int pp = 0; pp < pr.peers.world; ++pp)
            if (!make_map3s(&em.peer[pp], pr.peers.base[pp], f32, pr.N, rows_end, blocks, s1, s2, bc, 32))
              return cudaErrorInvalidValue;
        } else if (!pr.scatter_rows && !make_map3s(&em.d, pr.D, f32, pr.N, rows_end, pr.nblk, s1, s2, bc, 32)) {
          return cudaErrorInvalidValue;
        }
        if (pr.epi == Epi::GeluFwd &&
            !make_map3s(&em.d2, pr.D2, false, pr.N, rows_end, pr.nblk, pr.ldd2 * 2,
                        static_cast<uint64_t>(p.rows_total) * pr.ldd2 * 2, 64, 32))
          return cudaErrorInvalidValue;
        if ((pr.epi == Epi::GeluBwd || pr.epi == Epi::AddBF16) &&
            !make_map3s(&em.z, pr.Zin, false, pr.N, rows_end, pr.nblk, pr.ldz * 2,
                        static_cast<uint64_t>(p.rows_total) * pr.ldz * 2, 64, 32))
          return cudaErrorInvalidValue;
      } else {
        if (!make_map3s(&em.d, pr.D, f32, pr.No, pr.Mo, p.n_w, pr.ldd * es,
                        static_cast<uint64_t>(pr.Mo) * pr.ldd * es, bc, 32))
          return cudaErrorInvalidValue;
      }
    }
  }
  const int sms = pr.max_sms > 0 && pr.max_sms < num_sms() ? pr.max_sms : num_sms();
  const int max_units = sms / ctas > 0 ? sms / ctas : 1;
  const int units = p.num_tiles < max_units ? p.num_tiles : max_units;
  static DeviceOnce smem_set[2][3];
  auto launch = [&](auto kern, int smem) -> cudaError_t {
    once_on_device(smem_set[ctas - 1][BN == 128 ? 0 : BN == 256 ? 1 : 2],
                   [&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(units * ctas);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (ctas == 2) {
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = ctas;
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = 1;
      ++na;
    }
    if (pdl_on()) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, ta, tb, p, em);
  };
  cudaError_t e;
  if (ctas == 1)
    e = BN == 256 ? launch(grouped_gemm_kernel<1, 256>, TileCfg<1, 256>::SMEM)
                  : launch(grouped_gemm_kernel<1, 128>, TileCfg<1, 128>::SMEM);
  else if (BN == 512)
    e = launch(grouped_gemm_kernel<2, 512>, TileCfg<2, 512>::SMEM);
  else
    e = BN == 256 ? launch(grouped_gemm_kernel<2, 256>, TileCfg<2, 256>::SMEM)
                  : launch(grouped_gemm_kernel<2, 128>, TileCfg<2, 128>::SMEM);
  if (e != cudaSuccess) return static_cast<int>(e);
  ::fsmoe::count_launch();
  return static_cast<int>(cudaGetLastError());
}

}  // namespace fsmoe
