// Dependent-chain latency of uniform-datapath vs vector integer code (one warp).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/uniform_bench.cu -o /tmp/ub && /tmp/ub
//
// Each iteration: x = (x * 3 + tab[x & 15]) ^ (x >> 3) -- a multiply, an
// indexed constant-bank read feeding the next add, a shift and a xor, all
// dependent.  U: x starts warp-uniform (shuffled) so ptxas may use UR
// registers; V: x depends on the lane so it stays in vector registers.
#include <cstdio>
#include <cuda_runtime.h>

struct Tab {
  int v[16];
};

template <bool U>
__global__ void chain_kernel(int iters, const __grid_constant__ Tab tab, int* out, unsigned long long* cyc) {
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  if (warp != 0) return;
  int x = U ? __shfl_sync(0xffffffffu, (int)blockIdx.x, 0) : (int)(threadIdx.x + blockIdx.x);
  const unsigned long long c0 = clock64();
  for (int i = 0; i < iters; ++i) x = (x * 3 + tab.v[x & 15]) ^ (x >> 3);
  const unsigned long long c1 = clock64();
  out[blockIdx.x * 32 + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}

int main() {
  Tab t;
  for (int i = 0; i < 16; ++i) t.v[i] = i * 7 + 1;
  int* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 148 * 32 * sizeof(int));
  cudaMalloc(&cyc, 148 * sizeof(unsigned long long));
  unsigned long long h[148];
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    chain_kernel<true><<<148, 64>>>(iters, t, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("uniform: %.1f cycles/iteration\n", (double)h[0] / iters);
    chain_kernel<false><<<148, 64>>>(iters, t, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("vector:  %.1f cycles/iteration\n", (double)h[0] / iters);
  }
  return 0;
}
