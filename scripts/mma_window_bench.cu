// tcgen05.mma rate with the implicit-GEMM window pattern of tc_gemm_kernel
// (MODE_ROWS, BN = 64, resident B): per tile, 9 windows x 4 K-steps of
// 128 x 64 x 16 into one accumulator; window w reads the A halo at a row
// shift s_w and its own resident 64 x 64 B tile; one commit per tile.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_23745_b200/csrc \
//        scripts/mma_window_bench.cu -o /tmp/mwb -lcuda && /tmp/mwb
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "engine.hpp"
#include "tc_gemm.cuh"

using namespace syno::tc;

// variant bits: 1 all shifts 0, 2 B always tile 0, 4 accumulate from the first MMA, 8 two accumulators alternate,
// 16 a second warp spins mbarrier.test_wait on a barrier the MMAs never complete, 32 the same with try_wait,
// 64 a producer warp streams 24 KB bulk copies global -> shared while the MMAs run,
// 128 eight epilogue warps loop tcgen05.ld of the second accumulator + bf16 global stores,
// 256 operands hold random bf16 values (else zeros), 512 window shifts read from a __grid_constant__
// parameter array with a dynamic index (as tc_gemm_kernel reads p.a_shift[w]), 1024 all 512 TMEM columns
// allocated and the accumulator at column 256, 2048 resident B at the top of a 200 KB allocation
struct ShiftParams {
  int pad[256];  // a large parameter block, as TcGemmParams is
  int shift[16];
};

__global__ void win_kernel(int n, int tiles, int variant, int kq, unsigned long long* out, const uint8_t* gsrc,
                           __nv_bfloat16* gdst, const __grid_constant__ ShiftParams sp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, never, cbar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  {
    // operand data: zeros, or N(0,1)-like random bf16 (variant 256)
    uint32_t* w32 = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < 104 * 1024 / 4; i += blockDim.x) {
      uint32_t v = 0;
      if (variant & 256) {
        uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 97u);
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        const float a = ((int)(h & 0xFFFF) - 32768) / 16384.0f, b = ((int)(h >> 16) - 32768) / 16384.0f;
        __nv_bfloat162 p2 = __floats2bfloat162_rn(a, b);
        v = *reinterpret_cast<uint32_t*>(&p2);
      }
      w32[i] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    done = 0;
    mbar_init(&never, 1);
    mbar_init(&cbar, 1);
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t cols = (variant & 1024) ? 512u : 256u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  unsigned long long c0 = 0, c1 = 0, g0 = 0, g1 = 0;
  const int shifts[9] = {0, 1, 2, 33, 34, 35, 66, 67, 68};
  if (warp == 0) {
    const uint32_t idesc = idesc_bf16(128, n);
    const uint32_t a_base = desc_lo(smem_u32(smem));
    const uint32_t b_base = desc_lo(smem_u32(smem + ((variant & 2048) ? 128 : 32) * 1024));
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    c0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t dst = tmem + ((variant & 8) ? (uint32_t)(t & 1) * 128u : 0u) + ((variant & 1024) ? 256u : 0u);
      if (!(variant & 4096)) {
#pragma unroll
      for (int w = 0; w < 9; ++w) {
        const uint32_t a_lo = a_base + (uint32_t)((variant & 1) ? 0 : shifts[w]) * 8u;
        const uint32_t b_lo = b_base + (uint32_t)((variant & 2) ? 0 : w) * (uint32_t)(n * 128 >> 4);
        for (int k = 0; k < kq; ++k)
          mma_lo<false>(dst, a_lo + (uint32_t)(k * 2), b_lo + (uint32_t)(k * 2), idesc,
                        ((variant & 4) || w > 0 || k > 0) ? 1u : 0u);
      }
      } else
#pragma unroll 1
      for (int w = 0; w < 9; ++w) {
        const int sh = (variant & 512) ? sp.shift[w] : shifts[w];
        const uint32_t a_lo = a_base + (uint32_t)((variant & 1) ? 0 : sh) * 8u;
        const uint32_t b_lo = b_base + (uint32_t)((variant & 2) ? 0 : w) * (uint32_t)(n * 128 >> 4);
        for (int k = 0; k < kq; ++k)
          mma_lo<false>(dst, a_lo + (uint32_t)(k * 2), b_lo + (uint32_t)(k * 2), idesc,
                        ((variant & 4) || w > 0 || k > 0) ? 1u : 0u);
      }
      mma_commit(&bar);
    }
    mbar_wait(&bar, (uint32_t)(tiles - 1) & 1u);
    c1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    done = 1;
  } else if (warp == 1 && (variant & 64)) {
    // producer: 24 KB bulk copies into [104 KB, 128 KB) of the dynamic smem, back to back
    uint32_t ph = 0;
    int i = 0;
    while (!done) {
      if (elect_one()) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&cbar)), "r"(24576));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(smem + 104 * 1024)),
                     "l"(gsrc + (size_t)((blockIdx.x * 64 + i) % 4096) * 24576), "r"(24576), "r"(smem_u32(&cbar))
                     : "memory");
      }
      __syncwarp();
      mbar_wait(&cbar, ph);
      ph ^= 1u;
      ++i;
    }
  } else if (warp >= 2 && (variant & 128)) {
    // epilogue: TMEM loads of columns [128, 192) + bf16 stores, 32 rows per warp
    const int q = warp & 3;
    float v[32];
    int it = 0;
    while (!done) {
      for (int c = 0; c < 2; ++c) {
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + 128u + (uint32_t)(c * 32), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32; ++j)
          gdst[((size_t)(blockIdx.x * 8 + (warp - 2)) * 64 + c * 32 + j) * 128 + (size_t)(it & 3) * 32 + (threadIdx.x & 31)] =
              __float2bfloat16(v[j]);
      }
      ++it;
    }
  } else if (warp == 1 && (variant & 48)) {
    // a producer-like warp polling a barrier while the MMAs run
    while (!done) {
      uint32_t ok;
      if (variant & 16)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&never)) : "memory");
      else
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0, %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&never)), "r"(1000) : "memory");
      if (ok) break;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x] = c1 - c0;
    out[2048 + blockIdx.x] = g1 - g0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 4096 * sizeof(unsigned long long));
  static unsigned long long h[4096];
  const size_t smem = 201 * 1024;
  uint8_t* d_src;
  __nv_bfloat16* d_dst;
  cudaMalloc(&d_src, (size_t)4096 * 24576 + 4096);
  cudaMalloc(&d_dst, (size_t)296 * 8 * 64 * 128 * 2);
  cudaFuncSetAttribute(win_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  ShiftParams sp{};
  const int shv[9] = {0, 1, 2, 33, 34, 35, 66, 67, 68};
  for (int i = 0; i < 9; ++i) sp.shift[i] = shv[i];
  printf("  N variant kq ctas/SM | cycles/MMA/SM (floor %s)\n", "128N/256");
  for (int n : {64, 128}) {
    for (int per_sm : {1}) {
      for (int variant : {0, 64, 128, 256, 448, 4096, 4096+64, 4096+128, 4096+256, 4096+448, 4096+192}) {
        for (int kq : {4}) {
          if (n == 128 && (per_sm == 2 || !(variant & 2))) continue;  // 9 B tiles of 16 KB do not fit
          const int tiles = 64, grid = 148 * per_sm;
          for (int rep = 0; rep < 2; ++rep) win_kernel<<<grid, 320, smem>>>(n, tiles, variant, kq, d_out, d_src, d_dst, sp);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          cudaMemcpy(h, d_out, 4096 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
          double mean = 0, ns = 0;
          for (int i = 0; i < grid; ++i) mean += (double)h[i], ns += (double)h[2048 + i];
          mean /= grid;
          ns /= grid;
          printf("%4d %7d %3d %7d | %8.1f   (%.0f MHz)\n", n, variant, kq, per_sm, mean / (tiles * 9.0 * kq) / per_sm,
                 mean / ns * 1e3);
        }
      }
    }
  }
  return 0;
}
