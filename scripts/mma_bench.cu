// tcgen05.mma (kind::f16, SS operands) issue-rate microbenchmark.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_23745_b200/csrc \
//        scripts/mma_bench.cu -o /tmp/mma_bench -lcuda && /tmp/mma_bench
//
// One warp per CTA issues `iters` rounds of `nacc` accumulators x `chain`
// dependent K-steps (128 x N x 16 each) from shared memory, commits once and
// waits; cycles per MMA per SM = elapsed SM cycles x CTAs per SM / MMAs per CTA.
// Operand values are irrelevant (zeros).  Variants: N, accumulators,
// chain length, CTAs per SM, whether A advances (distinct smem rows) per MMA.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "engine.hpp"
#include "tc_gemm.cuh"

using namespace syno::tc;

__global__ void mma_kernel(int n, int nacc, int chain, int iters, int a_rows_step, int commit_every,
                           unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t cols = 256u;  // <= 2 CTAs per SM
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  unsigned long long c0 = 0, c1 = 0;
  if (warp == 0) {
    const uint32_t idesc = idesc_bf16(128, n);
    const uint64_t db = sw128_desc(smem + 64 * 1024);
    c0 = clock64();
    uint32_t ncommit = 0;
    for (int it = 0; it < iters; ++it) {
      for (int a = 0; a < nacc; ++a) {
        const uint32_t dst = tmem + (uint32_t)(a * n) % cols;
        // A: a row-shifted view per accumulator/iteration (as the halo windows are)
        const uint64_t da = sw128_desc(smem, ((it * nacc + a) * a_rows_step) % 256);
        for (int k = 0; k < chain; ++k) mma_bf16(dst, da + (uint64_t)((k & 3) * 2), db + (uint64_t)((k & 3) * 2), idesc, 1u);
      }
      if (commit_every && (it + 1) % commit_every == 0) {
        mma_commit(&bar);
        ++ncommit;
      }
    }
    mma_commit(&bar);
    ++ncommit;
    // wait for the last commit (phase parity of the ncommit-th completion)
    mbar_wait(&bar, (ncommit - 1) & 1u);
    c1 = clock64();
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = c1 - c0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}


// Straight-line variants: CHAIN MMAs per round with compile-time descriptor
// offsets (the descriptors advance by adds only).  MODE 0: warp-wide issue
// with elect (mma_bf16); MODE 1: one thread issues (plain tcgen05.mma).
template <int CHAIN, int MODE>
__global__ void mma_fixed(int n, int iters, int commit_every, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t cols = 256u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  unsigned long long c0 = 0, c1 = 0;
  const uint32_t idesc = idesc_bf16(128, n);
  const uint64_t db = sw128_desc(smem + 64 * 1024);
  const uint64_t da0 = sw128_desc(smem);
  if (MODE == 0 && warp == 0) {
    c0 = clock64();
    uint32_t nc = 0;
    for (int it = 0; it < iters; ++it) {
      const uint64_t da = da0 + (uint64_t)((it & 7) * 8);  // 1 row = 128 B = 8 units
#pragma unroll
      for (int k = 0; k < CHAIN; ++k) mma_bf16(tmem, da + (uint64_t)((k & 3) * 2), db + (uint64_t)((k & 3) * 2), idesc, 1u);
      if (commit_every && (it + 1) % commit_every == 0) {
        mma_commit(&bar);
        ++nc;
      }
    }
    mma_commit(&bar);
    ++nc;
    mbar_wait(&bar, (nc - 1) & 1u);
    c1 = clock64();
  }
  if (MODE == 1 && threadIdx.x == 0) {
    c0 = clock64();
    uint32_t nc = 0;
    for (int it = 0; it < iters; ++it) {
      const uint64_t da = da0 + (uint64_t)((it & 7) * 8);
#pragma unroll
      for (int k = 0; k < CHAIN; ++k)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da + (uint64_t)((k & 3) * 2)), "l"(db + (uint64_t)((k & 3) * 2)), "r"(idesc), "r"(1));
      if (commit_every && (it + 1) % commit_every == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                     : "memory");
        ++nc;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    ++nc;
    mbar_wait(&bar, (nc - 1) & 1u);
    c1 = clock64();
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = c1 - c0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}

template <int CHAIN, int MODE>
static void run_fixed(int n, int iters, int commit_every, int per_sm, unsigned long long* d_out) {
  const size_t smem = 100 * 1024;
  cudaFuncSetAttribute(mma_fixed<CHAIN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = 148 * per_sm;
  for (int rep = 0; rep < 2; ++rep) mma_fixed<CHAIN, MODE><<<grid, 128, smem>>>(n, iters, commit_every, d_out);
  cudaDeviceSynchronize();
  static unsigned long long h[4096];
  cudaMemcpy(h, d_out, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < grid; ++i) mean += (double)h[i];
  mean /= grid;
  printf("fixed chain=%2d mode=%d N=%3d commit/it=%d ctas/SM=%d | %8.1f cycles/MMA/SM\n", CHAIN, MODE, n, commit_every,
         per_sm, mean / ((double)iters * CHAIN) / per_sm);
}

// MN-major operands (both A and B, as the grad-weight GEMM uses): one warp
// issues chains of 128 x N x 16 MMAs from 128-byte-swizzled MN-major tiles.
__global__ void mma_mn_kernel(int n, int chain, int iters, int per_sm_div, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  unsigned long long c0 = 0, c1 = 0;
  if (warp == 0) {
    const uint32_t idesc = idesc_bf16(128, n, 1, 1);
    const uint64_t da = sw128_mn_desc(smem, 8192), db = sw128_mn_desc(smem + 32768, 8192);
    c0 = clock64();
    uint32_t nc = 0;
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < chain; ++k)
        mma_bf16(tmem, da + (uint64_t)((k & 3) * 128), db + (uint64_t)((k & 3) * 128), idesc, 1u);
      mma_commit(&bar);
      ++nc;
    }
    mbar_wait(&bar, (nc - 1) & 1u);
    c1 = clock64();
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = c1 - c0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  {
    unsigned long long* d_o;
    cudaMalloc(&d_o, 4096 * sizeof(unsigned long long));
    static unsigned long long hh[4096];
    cudaFuncSetAttribute(mma_mn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int n : {64, 128, 256}) {
      for (int rep = 0; rep < 2; ++rep) mma_mn_kernel<<<148, 128, 100 * 1024>>>(n, 16, 128, 1, d_o);
      cudaDeviceSynchronize();
      cudaMemcpy(hh, d_o, 148 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double mean = 0;
      for (int i = 0; i < 148; ++i) mean += (double)hh[i];
      printf("MN-major A and B: N=%3d chain=16 | %8.1f cycles/MMA/SM (floor %d)\n", n, mean / 148 / (128.0 * 16),
             128 * n / 256);
    }
    cudaFree(d_o);
  }
  unsigned long long* d_out;
  cudaMalloc(&d_out, 4096 * sizeof(unsigned long long));
  unsigned long long h[4096];
  const size_t smem = 100 * 1024;  // two CTAs fit per SM
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  struct Cfg {
    int n, nacc, chain, iters, step, commit_every, per_sm;
  };
  const Cfg cfgs[] = {
      {64, 1, 4, 512, 0, 0, 1},   {64, 1, 4, 512, 0, 0, 2},   {64, 1, 4, 512, 1, 0, 1},  {64, 1, 4, 512, 1, 1, 1},
      {64, 1, 4, 512, 1, 1, 2},   {64, 2, 4, 256, 1, 1, 1},   {64, 4, 4, 128, 1, 1, 1},  {64, 1, 16, 128, 1, 0, 1},
      {64, 1, 36, 64, 1, 0, 1},   {128, 1, 4, 512, 1, 1, 1},  {128, 1, 4, 512, 1, 1, 2}, {128, 2, 4, 256, 1, 1, 1},
      {256, 1, 4, 512, 1, 1, 1},  {64, 1, 4, 512, 3, 1, 1},   {64, 1, 4, 512, 1, 4, 1},  {64, 1, 4, 512, 1, 4, 2},
  };
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("   N nacc chain iters step commit/it ctas/SM | cycles/MMA/SM  (SS 128xNx16; floor 128N/256)\n");
  for (const Cfg& c : cfgs) {
    const int grid = 148 * c.per_sm;
    for (int rep = 0; rep < 2; ++rep)
      mma_kernel<<<grid, 128, smem>>>(c.n, c.nacc, c.chain, c.iters, c.step, c.commit_every, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d_out, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < grid; ++i) mean += (double)h[i];
    mean /= grid;
    const double mmas = (double)c.iters * c.nacc * c.chain;
    printf("%4d %4d %5d %5d %4d %9d %7d | %8.1f\n", c.n, c.nacc, c.chain, c.iters, c.step, c.commit_every, c.per_sm,
           mean / mmas / c.per_sm);
  }
  for (int n : {64, 128, 256}) {
    run_fixed<4, 0>(n, 512, 1, 1, d_out);
    run_fixed<4, 1>(n, 512, 1, 1, d_out);
    run_fixed<16, 0>(n, 128, 1, 1, d_out);
    run_fixed<16, 1>(n, 128, 1, 1, d_out);
    run_fixed<4, 1>(n, 512, 1, 2, d_out);
    run_fixed<16, 1>(n, 128, 1, 2, d_out);
  }
  return 0;
}
