// Dependent-chain latency (cycles per op) of DADD, DMUL, DFMA, F2F.F64.F32
// and FADD on one thread, and DADD throughput with many independent chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_latency fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(int kind, int n, double* out, long long* cyc) {
  double a = out[0], b = out[1];
  float f = static_cast<float>(out[2]);
  long long t0 = clock64();
  if (kind == 0) for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
  if (kind == 1) for (int i = 0; i < n; ++i) a = __dmul_rn(a, b);
  if (kind == 2) for (int i = 0; i < n; ++i) a = __fma_rn(a, b, b);
  if (kind == 3) for (int i = 0; i < n; ++i) { a = static_cast<double>(f); f = static_cast<float>(a) + 1.0f; }
  if (kind == 4) for (int i = 0; i < n; ++i) f = __fadd_rn(f, 1.0f);
  long long t1 = clock64();
  out[3 + threadIdx.x] = a + f;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 4096 * 8); cudaMalloc(&c, 8);
  double h[3] = {1.0, 1e-9, 1.5};
  cudaMemcpy(d, h, 24, cudaMemcpyHostToDevice);
  const char* names[] = {"DADD", "DMUL", "DFMA", "F2F.F64.F32+F2F.F32.F64+FADD", "FADD"};
  const int n = 1 << 16;
  for (int k = 0; k < 5; ++k) {
    for (int threads : {1, 32, 128, 512, 1024}) {
      chain<<<1, threads>>>(k, n, d, c);
      chain<<<1, threads>>>(k, n, d, c);
      long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
      printf("%-30s threads %5d: %.2f cycles per dependent op per thread\n", names[k], threads, double(cy) / n);
    }
  }
  return 0;
}
