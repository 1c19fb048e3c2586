// gemm_simt.cu — fp32 "check mode" grouped GEMM (SIMT FFMA, fp32 accumulate).
//
// Same problem semantics as the tcgen05 kernel (gemm.h) on fp32 tensors; used
// to verify the expert FFN forward/backward against the fp64 CPU restatement
// at tight tolerance. Only the StoreF32 epilogue is supported here; the
// activation epilogues run as separate elementwise kernels in check mode.
#include "gemm.h"

namespace fsmoe {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

struct SParams {
  int kind, nblk, rows, K, N, Mo, No, n_w, b_mn, rows_total, row0;
  const long long* valid;
  const float* A;
  const float* B;
  float* D;
  long long ldd;
  int accumulate;
  int use_peers;
  fsmoe_dev::PeerRows peers;
  fsmoe_dev::RowRange blocks;
};

__device__ __forceinline__ int valid_rows(const SParams& p, int b) {
  if (!p.valid) return p.rows;
  long long v = p.valid[b] - p.row0;
  return v < 0 ? 0 : (v > p.rows ? p.rows : static_cast<int>(v));
}

__global__ void __launch_bounds__(256) simt_gemm_kernel(SParams p) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int g = blockIdx.z;
  const int m0 = blockIdx.y * TM;
  const int n0 = blockIdx.x * TN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int out_rows = p.kind == 0 ? p.rows : p.Mo;
  const int out_cols = p.kind == 0 ? p.N : p.No;
  if (p.kind == 0 && (m0 >= valid_rows(p, g) || !fsmoe_dev::in_range(p.blocks, g))) return;
  float acc[4][4] = {};

  auto tile = [&](auto loadA, auto loadB, int klen) {
    for (int k0 = 0; k0 < klen; k0 += TK) {
      for (int i = threadIdx.x; i < TK * TM; i += 256) {
        int kk = i / TM, mm = i % TM;
        As[kk][mm] = loadA(m0 + mm, k0 + kk);
      }
      for (int i = threadIdx.x; i < TK * TN; i += 256) {
        int kk = i / TN, nn = i % TN;
        Bs[kk][nn] = loadB(n0 + nn, k0 + kk);
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
  };

  if (p.kind == 0) {
    const int w = g % p.n_w;
    const float* A = p.A + (static_cast<long long>(g) * p.rows_total + p.row0) * p.K;
    auto la = [&](int r, int k) -> float {
      return (r < p.rows && k < p.K) ? A[static_cast<long long>(r) * p.K + k] : 0.f;
    };
    auto lb = [&](int n, int k) -> float {
      if (n >= p.N || k >= p.K) return 0.f;
      return p.b_mn ? p.B[(static_cast<long long>(w) * p.K + k) * p.N + n]
                    : p.B[(static_cast<long long>(w) * p.N + n) * p.K + k];
    };
    tile(la, lb, p.K);
  } else {
    for (int b = g; b < p.nblk; b += p.n_w) {
      const int vr = valid_rows(p, b);
      const float* A = p.A + (static_cast<long long>(b) * p.rows_total + p.row0) * p.Mo;
      const float* B = p.B + (static_cast<long long>(b) * p.rows_total + p.row0) * p.No;
      auto la = [&](int m, int r) -> float {
        return (m < p.Mo && r < vr) ? A[static_cast<long long>(r) * p.Mo + m] : 0.f;
      };
      auto lb = [&](int n, int r) -> float {
        return (n < p.No && r < vr) ? B[static_cast<long long>(r) * p.No + n] : 0.f;
      };
      tile(la, lb, vr);
    }
  }


#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = m0 + ty * 4 + i;
    if (r >= out_rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int c = n0 + tx * 4 + j;
      if (c >= out_cols) continue;
      const long long orow = p.kind == 0 ? static_cast<long long>(g) * p.rows_total + p.row0 + r
                                         : static_cast<long long>(g) * p.Mo + r;
      float* d = (p.use_peers ? reinterpret_cast<float*>(fsmoe_dev::peer_row(p.peers, orow, p.ldd * 4))
                              : p.D + orow * p.ldd) + c;
      *d = p.accumulate ? *d + acc[i][j] : acc[i][j];
    }
  }
}

}  // namespace

int gemm_simt_launch(const GemmProblem& pr, cudaStream_t stream) {
  if (pr.epi != Epi::StoreF32) return cudaErrorInvalidValue;
  if (pr.nblk <= 0 || pr.rows <= 0) return cudaSuccess;
  SParams p{};
  p.kind = static_cast<int>(pr.kind);
  p.nblk = pr.nblk;
  p.rows = pr.rows;
  p.rows_total = pr.rows_total > 0 ? pr.rows_total : pr.rows;
  p.row0 = pr.row0;
  if (p.row0 < 0 || p.row0 + p.rows > p.rows_total) return cudaErrorInvalidValue;
  p.K = pr.K;
  p.N = pr.N;
  p.Mo = pr.Mo;
  p.No = pr.No;
  p.n_w = pr.n_w > 0 ? pr.n_w : 1;
  p.b_mn = pr.b_mn_major ? 1 : 0;
  p.valid = pr.valid_rows;
  p.A = static_cast<const float*>(pr.A);
  p.B = static_cast<const float*>(pr.B);
  p.D = static_cast<float*>(pr.D);
  p.ldd = pr.ldd;
  p.accumulate = pr.accumulate ? 1 : 0;
  p.use_peers = pr.use_peers ? 1 : 0;
  p.peers = pr.peers;
  p.blocks = pr.blocks;
  dim3 grid;
  if (pr.kind == GemmKind::RowGrouped) {
    grid = dim3((pr.N + TN - 1) / TN, (pr.rows + TM - 1) / TM, pr.nblk);
  } else {
    if (pr.nblk % p.n_w) return cudaErrorInvalidValue;
    grid = dim3((pr.No + TN - 1) / TN, (pr.Mo + TM - 1) / TM, p.n_w);
  }
  simt_gemm_kernel<<<grid, 256, 0, stream>>>(p); ::fsmoe::count_launch();
  return static_cast<int>(cudaGetLastError());
}

}  // namespace fsmoe
