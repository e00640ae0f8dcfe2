// Producer -> MMA-warp hand-off cost (no TMA, optional MMAs): cycles per
// k-step of the ring protocol tc_gemm_kernel uses, under variants.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_23745_b200/csrc \
//        scripts/sync_bench.cu -o /tmp/sync_bench -lcuda && /tmp/sync_bench
//
// Warp 0 (producer): per step wait empty[s], arrive full[s].  Warp 1 (consumer):
// wait full[s], fence, [n_mma MMAs 128x256x16], commit empty[s] (tcgen05.commit)
// or a plain arrive.  Flags: bit0 consumer uses try_wait, bit1 producer uses
// try_wait, bit2 plain arrive instead of tcgen05.commit (no MMAs), bit3 no fence,
// bit4 second commit per step (as the A + B rings do), bit5 consumer alone
// (no producer: waits on a pre-completed phase), bit6 producer alone,
// bit7 relaxed try_wait, bit8 consumer does not wait, bit9 consumer does not release.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "engine.hpp"
#include "tc_gemm.cuh"

using namespace syno::tc;

__device__ __forceinline__ void wait_try(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void wait_relaxed(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__global__ void sync_kernel(int steps, int stages, int n_mma, int flags, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[8], empty[8], empty2[8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&empty2[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  unsigned long long c0 = clock64();
  if (warp == 0 && !(flags & 32)) {
    for (int i = 0; i < steps; ++i) {
      const int s = i % stages;
      const uint32_t ph = (flags & 64) ? 1u : ((i / stages) & 1) ^ 1;
      if (flags & 2) wait_try(&empty[s], ph);
      else mbar_wait(&empty[s], ph);
      if (flags & 16) {
        if (flags & 2) wait_try(&empty2[s], ph);
        else mbar_wait(&empty2[s], ph);
      }
      if (elect_one()) mbar_arrive(&full[s]);
      __syncwarp();
    }
  } else if (warp == 1 && !(flags & 64)) {
    const uint32_t idesc = idesc_bf16(128, 256);
    const uint64_t da = sw128_desc(smem), db = sw128_desc(smem + 32768);
    for (int i = 0; i < steps; ++i) {
      const int s = i % stages;
      const uint32_t ph = (flags & 32) ? 1u : (i / stages) & 1;  // alone: parity 1 of a fresh barrier completes at once
      if (flags & 256) {
        // no wait
      } else if (flags & 128) wait_relaxed(&full[s], ph);
      else if (flags & 1) wait_try(&full[s], ph);
      else mbar_wait(&full[s], ph);
      if (!(flags & 8)) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int k = 0; k < n_mma; ++k) mma_bf16(tmem, da + (uint64_t)((k & 3) * 2), db + (uint64_t)((k & 3) * 2), idesc, 1u);
      if (flags & 512) {
        // no release
      } else if (flags & 4) {
        if (elect_one()) {
          mbar_arrive(&empty[s]);
          if (flags & 16) mbar_arrive(&empty2[s]);
        }
        __syncwarp();
      } else {
        mma_commit(&empty[s]);
        if (flags & 16) mma_commit(&empty2[s]);
      }
    }
  }
  unsigned long long c1 = clock64();
  __syncthreads();
  if (threadIdx.x == 32) out[blockIdx.x] = c1 - c0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// Compile-time variants of the consumer loop alone (no producer): W wait
// (0 none, 1 test_wait, 2 try_wait), R release (0 none, 1 tcgen05.commit,
// 2 plain arrive), M MMAs per step; stages fixed at 4 (masking, no division).
struct Tab {
  int v[64];
};

// X: 0 none, 1 per-step indexed read of a __grid_constant__ array feeding the
// wait address, 2 the same array staged in shared memory, 3 runtime-bound
// inner loop over array entries (as the window loop), 4 = 3 with smem.
template <int W, int R, int M, int X = 0>
__global__ void cons_kernel(int steps, unsigned long long* out, const __grid_constant__ Tab tab) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[4], empty[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  __shared__ int stab[64];
  if (threadIdx.x < 64) stab[threadIdx.x] = tab.v[threadIdx.x];
  __syncthreads();
  const uint32_t tmem = tslot;
  const uint32_t idesc = idesc_bf16(128, 256);
  const uint64_t da = sw128_desc(smem), db = sw128_desc(smem + 32768);
  unsigned long long c0 = clock64();
  for (int i = 0; i < steps; ++i) {
    int s = i & 3;
    if (X == 1) s = tab.v[i & 63];
    if (X == 2) s = stab[i & 63];
    if (X == 3 || X == 4) {
      const int lo = X == 3 ? tab.v[(i & 31)] : stab[i & 31], hi = X == 3 ? tab.v[32 + (i & 31)] : stab[32 + (i & 31)];
      for (int j = lo; j < hi; ++j) s = (s + j) & 3;
    }
    if (W == 1) mbar_wait(&full[s], 1u);
    if (W == 2) wait_try(&full[s], 1u);
#pragma unroll
    for (int k = 0; k < M; ++k) mma_bf16(tmem, da + (uint64_t)((k & 3) * 2), db + (uint64_t)((k & 3) * 2), idesc, 1u);
    if (R == 1) mma_commit(&empty[s]);
    if (R == 2) {
      if (elect_one()) mbar_arrive(&empty[s]);
      __syncwarp();
    }
  }
  unsigned long long c1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = c1 - c0;
  mma_commit(&empty[0]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// Compile-time producer/consumer ping-pong over a 4-stage ring: R release
// (1 tcgen05.commit, 2 plain arrive), M MMAs per step, D data-ring pairs per
// step (1: one full/empty pair as one ring; 2: A and B rings as tc_gemm has).
template <int R, int M, int D>
__global__ void pp_kernel(int steps, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[2][4], empty[2][4];
  __shared__ uint32_t tslot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 2; ++d) {
        mbar_init(&full[d][s], 1);
        mbar_init(&empty[d][s], 1);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  unsigned long long c0 = clock64();
  if (warp == 0) {
    for (int i = 0; i < steps; ++i) {
      const int s = i & 3;
      const uint32_t ph = ((i >> 2) & 1) ^ 1;
      for (int d = 0; d < D; ++d) {
        mbar_wait(&empty[d][s], ph);
        if (elect_one()) mbar_arrive(&full[d][s]);
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16(128, 256);
    const uint64_t da = sw128_desc(smem), db = sw128_desc(smem + 32768);
    for (int i = 0; i < steps; ++i) {
      const int s = i & 3;
      const uint32_t ph = (i >> 2) & 1;
      for (int d = 0; d < D; ++d) mbar_wait(&full[d][s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int k = 0; k < M; ++k) mma_bf16(tmem, da + (uint64_t)((k & 3) * 2), db + (uint64_t)((k & 3) * 2), idesc, 1u);
      for (int d = 0; d < D; ++d) {
        if (R == 1) mma_commit(&empty[d][s]);
        if (R == 2) {
          if (elect_one()) mbar_arrive(&empty[d][s]);
          __syncwarp();
        }
      }
    }
  }
  unsigned long long c1 = clock64();
  __syncthreads();
  if (threadIdx.x == 32) out[blockIdx.x] = c1 - c0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int R, int M, int D>
static void run_pp(unsigned long long* d_out) {
  const int steps = 2048, grid = 148;
  cudaFuncSetAttribute(pp_kernel<R, M, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rep = 0; rep < 2; ++rep) pp_kernel<R, M, D><<<grid, 64, 100 * 1024>>>(steps, d_out);
  cudaDeviceSynchronize();
  static unsigned long long h[4096];
  cudaMemcpy(h, d_out, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < grid; ++i) mean += (double)h[i];
  printf("pingpong release=%d mma=%2d rings=%d | %8.1f cycles/step\n", R, M, D, mean / grid / steps);
}

template <int W, int R, int M, int X = 0>
static void run_cons(unsigned long long* d_out) {
  const int steps = 2048, grid = 148;
  Tab tab;
  for (int i = 0; i < 64; ++i) tab.v[i] = i < 32 ? 0 : 1;  // X 1/2: slot 0..; X 3/4: one inner iteration
  for (int i = 0; i < 32; ++i) tab.v[i] = 0;
  cudaFuncSetAttribute(cons_kernel<W, R, M, X>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rep = 0; rep < 2; ++rep) cons_kernel<W, R, M, X><<<grid, 32, 100 * 1024>>>(steps, d_out, tab);
  cudaDeviceSynchronize();
  static unsigned long long h[4096];
  cudaMemcpy(h, d_out, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < grid; ++i) mean += (double)h[i];
  printf("cons wait=%d release=%d mma=%2d x=%d | %8.1f cycles/step\n", W, R, M, X, mean / grid / steps);
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 4096 * sizeof(unsigned long long));
  static unsigned long long h[4096];
  const size_t smem = 100 * 1024;
  cudaFuncSetAttribute(sync_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  struct Cfg {
    int stages, n_mma, flags, threads;
  };
  const Cfg cfgs[] = {
      {4, 0, 32, 64},        {4, 0, 32 | 256, 64},  {4, 0, 32 | 512, 64}, {4, 0, 32 | 256 | 512, 64},
      {4, 0, 32 | 128, 64},  {4, 0, 32 | 128 | 512, 64}, {4, 0, 32 | 256 | 4, 64}, {4, 0, 32 | 1 | 512, 64},
      {4, 0, 32 | 8 | 256 | 512, 64}, {4, 4, 32 | 256 | 512, 64}, {4, 4, 32 | 256, 64}, {4, 4, 128, 64},
      {4, 8, 128, 64},
  };
  printf("stages n_mma flags threads | cycles/step  (flags: 1 cons try_wait, 2 prod try_wait, 4 plain arrive, 8 no fence, 16 two commits)\n");
  for (const Cfg& c : cfgs) {
    const int steps = 2048, grid = 148;
    for (int rep = 0; rep < 2; ++rep) sync_kernel<<<grid, c.threads, smem>>>(steps, c.stages, c.n_mma, c.flags, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d_out, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < grid; ++i) mean += (double)h[i];
    mean /= grid;
    printf("%6d %5d %5d %7d | %8.1f\n", c.stages, c.n_mma, c.flags, c.threads, mean / steps);
  }
  run_cons<0, 0, 0>(d_out);
  run_cons<1, 0, 0>(d_out);
  run_cons<2, 0, 0>(d_out);
  run_cons<0, 1, 0>(d_out);
  run_cons<0, 2, 0>(d_out);
  run_cons<1, 1, 0>(d_out);
  run_cons<2, 1, 0>(d_out);
  run_cons<0, 0, 4>(d_out);
  run_cons<0, 1, 4>(d_out);
  run_cons<2, 1, 4>(d_out);
  run_cons<2, 1, 8>(d_out);
  run_cons<2, 1, 16>(d_out);
  run_cons<1, 1, 0, 1>(d_out);
  run_cons<1, 1, 0, 2>(d_out);
  run_cons<1, 1, 0, 3>(d_out);
  run_cons<1, 1, 0, 4>(d_out);
  run_cons<1, 1, 4, 1>(d_out);
  run_cons<1, 1, 4, 3>(d_out);
  run_cons<1, 1, 4, 4>(d_out);
  run_pp<1, 0, 1>(d_out);
  run_pp<2, 0, 1>(d_out);
  run_pp<1, 0, 2>(d_out);
  run_pp<1, 4, 1>(d_out);
  run_pp<1, 4, 2>(d_out);
  run_pp<1, 8, 2>(d_out);
  return 0;
}
