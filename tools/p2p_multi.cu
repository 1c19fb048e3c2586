// p2p_multi.cu — NVLink egress of one GPU writing to 1..3 peers at once, and
// of all GPUs writing to all peers at once (the AlltoAll pattern): is the
// ~550 GB/s seen to one peer a per-peer or a per-GPU limit?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_multi p2p_multi.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));         \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

struct Dsts {
  char* p[8];
  int n;
};

// block b writes its share of `bytes` to destination b % n (16-byte coalesced stores)
__global__ void scatter(const uint4* __restrict__ src, Dsts d, long long bytes) {
  const int k = blockIdx.x % d.n;
  const int nb = gridDim.x / d.n;  // blocks per destination
  const int bi = blockIdx.x / d.n;
  const long long n16 = bytes / 16;
  uint4* dst = reinterpret_cast<uint4*>(d.p[k]);
  for (long long i = static_cast<long long>(bi) * blockDim.x + threadIdx.x; i < n16;
       i += static_cast<long long>(nb) * blockDim.x)
    dst[i] = src[i];
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("need 2+ GPUs\n");
    return 1;
  }
  const long long bytes = 32LL << 20;  // per destination
  std::vector<char*> src(n);
  std::vector<std::vector<char*>> recv(n, std::vector<char*>(n, nullptr));  // recv[dst][src]
  for (int g = 0; g < n; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < n; ++h)
      if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMemset(src[g], 1, bytes));
    for (int h = 0; h < n; ++h) CK(cudaMalloc(&recv[g][h], bytes));
  }
  auto run = [&](int g, int npeers, cudaStream_t s) {
    Dsts d{};
    d.n = npeers;
    for (int k = 0, h = 0; k < npeers; ++h)
      if (h != g) d.p[k++] = recv[h][g];
    scatter<<<148 * 4 / npeers * npeers, 512, 0, s>>>(reinterpret_cast<const uint4*>(src[g]), d, bytes);
  };
  // one GPU -> 1..n-1 peers
  CK(cudaSetDevice(0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int np = 1; np < n; ++np) {
    run(0, np, 0);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int r = 0; r < 5; ++r) run(0, np, 0);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("gpu0 -> %d peer(s): %.1f GB/s egress\n", np, 5.0 * np * bytes / (ms * 1e-3) / 1e9);
  }
  // all GPUs -> all peers at once
  std::vector<cudaStream_t> st(n);
  std::vector<cudaEvent_t> e0(n), e1(n);
  for (int g = 0; g < n; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaStreamCreate(&st[g]));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  for (int rep = 0; rep < 2; ++rep) {
    for (int g = 0; g < n; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaDeviceSynchronize());
    }
    for (int g = 0; g < n; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventRecord(e0[g], st[g]));
      for (int r = 0; r < 5; ++r) run(g, n - 1, st[g]);
      CK(cudaEventRecord(e1[g], st[g]));
    }
    double worst = 0;
    for (int g = 0; g < n; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventSynchronize(e1[g]));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
      worst = ms > worst ? ms : worst;
    }
    if (rep) printf("all %d GPUs -> all peers: %.1f GB/s egress per GPU\n", n, 5.0 * (n - 1) * bytes / (worst * 1e-3) / 1e9);
  }
  return 0;
}
