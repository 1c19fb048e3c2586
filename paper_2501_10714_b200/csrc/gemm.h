// gemm.h — grouped expert GEMM problem description shared by the tcgen05
// kernel (bf16, gemm_sm100.cu) and the fp32 SIMT check-mode kernel
// (gemm_simt.cu). Host-side only types plus the launch entry points.
//
// Two problem shapes cover the whole expert FFN forward and backward
// (SURVEY.md Appendix D):
//
//  ROW-GROUPED (forward, dgrad):   D[b] (rows x N) = A[b] (rows x K) . B[w(b)] (K x N)
//    A: [nblk][rows][K] row-major (K contiguous)           -> K-major operand
//    B: K-major   [E_w][N][K]  (forward weights)
//       MN-major  [E_w][K][N]  (dgrad: the forward weight read transposed)
//    w(b) = b % E_w ; D: [nblk][rows][N]
//
//  K-GROUPED (wgrad):   D[e] (Mo x No) = sum_{b : b % E_w == e} A[b]^T . B[b]
//    A: [nblk][rows][Mo] (Mo contiguous) -> MN-major operand
//    B: [nblk][rows][No] (No contiguous) -> MN-major operand
//    D: [E_w][Mo][No] fp32, optionally accumulated (pipeline chunks).
//
// Row window: every block holds `rows_total` rows in memory (the capacity C);
// one launch processes rows [row0, row0 + rows) of each block (a pipeline
// chunk). Row-grouped outputs (and Zin / D2) use the same [nblk][rows_total]
// row addressing. row0 must be a multiple of 128 unless rows reaches the end.
//
// `valid_rows[b]` (optional, device int64 per block) is the dispatch fill of
// that block (absolute row count): row tiles entirely past it are skipped
// (their rows are capacity padding) and wgrad's K extent stops at
// round_up(valid, 64).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "route_common.cuh"

namespace fsmoe {

enum class GemmKind : int { RowGrouped = 0, KGrouped = 1 };

enum class Epi : int {
  StoreBF16 = 0,   // D bf16
  StoreF32 = 1,    // D fp32 (accumulate when `accumulate`)
  GeluFwd = 2,     // D = gelu'(acc) (bf16, what the backward needs), D2 = H = gelu(acc)
  SwigluFwd = 3,   // acc cols interleaved [gate128|up128]: Z = acc, H = silu(g)*u
  GeluBwd = 4,     // acc = dH; dZ = dH * Zin, Zin = the saved gelu'(Z)  N = H
  SwigluBwd = 5,   // acc = dH (N = H); writes dZ at interleaved gate/up columns
  AddBF16 = 6,     // D = bf16(acc + Zin) (Zin may alias D: in-place accumulation of a bf16 output)
};

struct GemmProblem {
  GemmKind kind = GemmKind::RowGrouped;
  int nblk = 0;        // A/B blocks (row-grouped: output blocks too)
  int rows = 0;        // rows per block processed by this launch
  int rows_total = 0;  // rows per block in memory (0 -> rows)
  int row0 = 0;        // first processed row of each block
  int K = 0;           // row-grouped reduction dim
  int N = 0;           // row-grouped output columns
  int Mo = 0, No = 0;  // k-grouped output dims
  int n_w = 1;         // weight (expert) count E_w; w(b) = b % n_w
  bool b_mn_major = false;  // row-grouped only (k-grouped: both MN-major)
  const void* A = nullptr;
  const void* B = nullptr;
  const long long* valid_rows = nullptr;  // [nblk] or null
  // epilogue
  Epi epi = Epi::StoreBF16;
  void* D = nullptr;         // main output
  void* D2 = nullptr;        // GeluFwd/SwigluFwd: H output
  const void* Zin = nullptr; // GeluBwd/SwigluBwd: saved pre-activation
  long long ldd = 0;         // D row stride (elements)
  long long ldd2 = 0;        // D2 row stride
  long long ldz = 0;         // Zin row stride
  bool accumulate = false;   // StoreF32: D += acc
  // Row-grouped StoreBF16 / StoreF32: output row r of [nblk][rows_total] goes
  // through this peer map (NVLink stores into the owning rank) instead of D.
  bool use_peers = false;
  fsmoe_dev::PeerRows peers{};
  fsmoe_dev::RowRange blocks = fsmoe_dev::all_rows();  // row-grouped: blocks processed
  int max_sms = 0;                                        // > 0: cap the persistent grid
  int force_ctas = 0, force_bn = 0, dbg = 0;              // fsmoe_gemm_desc overrides
  int band_m = 0, band_n = 0;                             // tile-order override
  // row-grouped StoreBF16: output row r -> row scatter_rows[r] of scatter_out
  // (stride scatter_ld elements; < 0 dropped) instead of D
  const int* scatter_rows = nullptr;
  void* scatter_out = nullptr;
  long long scatter_ld = 0;
};

// bf16 operands, fp32 accumulate in TMEM (tcgen05). Returns cudaError_t.
int gemm_sm100_launch(const GemmProblem& p, cudaStream_t stream);
// fp32 operands/outputs, SIMT FFMA; same problem semantics (check mode).
int gemm_simt_launch(const GemmProblem& p, cudaStream_t stream);

void count_launch();  // capi_gemm.cu

}  // namespace fsmoe
