// capi_gemm.cu — extern "C" error plumbing + expert-FFN GEMM entry points.
#include <atomic>
#include <cstdio>
#include <string>

#include "capi_common.h"
#include "gemm.h"
#include "kernels.h"

namespace fsmoe {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_last_error(const std::string& msg) { g_last_error = msg; }

int config_error(const std::string& msg) {
  g_last_error = msg;
  return FSMOE_CONFIG_ERROR;
}

int invariant_error(const std::string& msg) {
  g_last_error = msg;
  return FSMOE_INVARIANT_ERROR;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return FSMOE_OK;
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return FSMOE_CUDA_ERROR;
}

namespace {

__global__ void act_f32_kernel(int op, int nblk, int rows_total, int row0, int rows, int units,
                               const float* __restrict__ in0, const float* __restrict__ z0,
                               float* __restrict__ out0) {
  long long n = static_cast<long long>(nblk) * rows * units;
  for (long long li = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; li < n;
       li += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long lr = li / units;
    int u = static_cast<int>(li - lr * units);
    long long b = lr / rows;
    long long r = b * rows_total + row0 + (lr - b * rows);  // absolute row
    long long i = r * units + u;
    const float* in = in0;
    const float* z = z0;
    float* out = out0;
    int gcol = (u / 128) * 256 + (u % 128);  // interleaved gate/up column of unit u
    switch (op) {
      case 2: {  // gelu fwd: in = Z (rows x units) -> out = gelu(Z)
        float v = in[i];
        out[i] = 0.5f * v * (1.0f + erff(v * 0.70710678118654752f));
        break;
      }
      case 3: {  // swiglu fwd: in = Z (rows x 2*units interleaved) -> out = H
        const float* zr = in + r * 2LL * units;
        float g = zr[gcol], up = zr[gcol + 128];
        out[i] = g / (1.0f + expf(-g)) * up;
        break;
      }
      case 4: {  // gelu bwd: in = dH, z = Z -> out = dZ
        float v = z[i];
        float cdf = 0.5f * (1.0f + erff(v * 0.70710678118654752f));
        float pdf = 0.39894228040143268f * expf(-0.5f * v * v);
        out[i] = in[i] * (cdf + v * pdf);
        break;
      }
      case 5: {  // swiglu bwd: in = dH (rows x units), z = Z interleaved -> out = dZ interleaved
        const float* zr = z + r * 2LL * units;
        float* dr = out + r * 2LL * units;
        float g = zr[gcol], up = zr[gcol + 128];
        float sg = 1.0f / (1.0f + expf(-g));
        float dh = in[i];
        dr[gcol] = dh * up * sg * (1.0f + g * (1.0f - sg));
        dr[gcol + 128] = dh * g * sg;
        break;
      }
      default:
        break;
    }
  }
}

}  // namespace
}  // namespace fsmoe

extern "C" {

const char* fsmoe_last_error(void) { return fsmoe::g_last_error.c_str(); }

int fsmoe_abi_version(void) { return 1; }

long long fsmoe_launch_count(void) { return fsmoe::g_launches.load(); }

int fsmoe_copy_device(void* dst, const void* src, size_t bytes, void* stream) {
  FSMOE_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, fsmoe::as_stream(stream)),
                 "fsmoe_copy_device");
  return FSMOE_OK;
}

int fsmoe_set_device(int device) {
  FSMOE_CUDA_TRY(cudaSetDevice(device), "fsmoe_set_device");
  return FSMOE_OK;
}

int fsmoe_grouped_gemm(const fsmoe_gemm_desc* d, void* stream) {
  using namespace fsmoe;
  if (!d) return config_error("gemm: null descriptor");
  GemmProblem p;
  p.kind = d->kind == 1 ? GemmKind::KGrouped : GemmKind::RowGrouped;
  p.nblk = d->nblk;
  p.rows = d->rows;
  p.K = d->K;
  p.N = d->N;
  p.Mo = d->Mo;
  p.No = d->No;
  p.n_w = d->n_w;
  p.rows_total = d->rows_total;
  p.row0 = d->row0;
  p.b_mn_major = d->b_mn_major != 0;
  p.A = d->A;
  p.B = d->B;
  p.valid_rows = d->valid_rows;
  p.epi = static_cast<Epi>(d->epi);
  p.D = d->D;
  p.D2 = d->D2;
  p.Zin = d->Zin;
  p.ldd = d->ldd;
  p.ldd2 = d->ldd2;
  p.ldz = d->ldz;
  p.accumulate = d->accumulate != 0;
  if (d->epi < 0 || d->epi > 6) return config_error("gemm: unknown epilogue");
  p.max_sms = d->max_sms;
  p.force_ctas = d->force_ctas;
  p.force_bn = d->force_bn;
  p.dbg = d->dbg;
  p.band_m = d->band_m;
  p.band_n = d->band_n;
  if (d->scatter_rows) {
    if (d->kind != 0 || d->epi != 0 || d->precision != 0 || d->d_peers || !d->scatter_out || d->scatter_ld <= 0)
      return config_error("gemm: a row scatter needs a row-grouped bf16-store tcgen05 problem and an output");
    p.scatter_rows = d->scatter_rows;
    p.scatter_out = d->scatter_out;
    p.scatter_ld = d->scatter_ld;
  }
  if (d->blk_hi > 0) {
    if (d->kind != 0) return config_error("gemm: a block range needs a row-grouped problem");
    p.blocks = fsmoe_dev::RowRange{d->blk_lo, d->blk_hi, d->blk_exclude};
  }
  if (d->d_peers) {
    const fsmoe_peer_rows* m = d->d_peers;
    if (d->kind != 0 || d->epi > 1)
      return config_error("gemm: peer output needs a row-grouped plain-store epilogue");
    if (m->world < 1 || m->world > FSMOE_MAX_PEERS || m->rank < 0 || m->rank >= m->world ||
        m->experts_local * m->world != d->nblk || m->capacity != (d->rows_total > 0 ? d->rows_total : d->rows))
      return config_error("gemm: peer map does not match nblk / rows_total");
    p.use_peers = true;
    p.peers = peer_rows_of(m);
  }
  if (p.kind == GemmKind::KGrouped && p.epi != Epi::StoreF32)
    return config_error("gemm: k-grouped (wgrad) problems take the f32 store epilogue");
  int rc = d->precision == 1 ? gemm_simt_launch(p, as_stream(stream))
                             : gemm_sm100_launch(p, as_stream(stream));
  if (rc == cudaErrorInvalidValue) return config_error("gemm: unsupported problem shape");
  return cuda_status(static_cast<cudaError_t>(rc), "fsmoe_grouped_gemm");
}

int fsmoe_activation_f32(int op, int nblk, int rows_total, int row0, int rows, int units,
                         const float* in, const float* z, float* out, void* stream) {
  using namespace fsmoe;
  if (op < 2 || op > 5) return config_error("activation: unknown op");
  if (nblk <= 0 || rows <= 0 || units <= 0) return FSMOE_OK;
  if (row0 < 0 || row0 + rows > rows_total) return config_error("activation: bad row window");
  if ((op == 3 || op == 5) && units % 128) return config_error("activation: swiglu units % 128");
  long long n = static_cast<long long>(nblk) * rows * units;
  int grid = static_cast<int>((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  act_f32_kernel<<<grid, 256, 0, as_stream(stream)>>>(op, nblk, rows_total, row0, rows, units, in,
                                                      z, out); ::fsmoe::count_launch();
  return cuda_status(cudaGetLastError(), "fsmoe_activation_f32");
}

}  // extern "C"
