// tcgen05 implicit-GEMM kernel (sm_100a): TMA -> SMEM (128B swizzle) ->
// tcgen05.mma (bf16 x bf16 -> fp32 in TMEM) -> tcgen05.ld -> masked affine
// epilogue.  Both operands are K-major tiles fetched by TMA from packed
// operand layouts (tc.cu); the k-block schedule and the epilogue address
// map come from TcGemmParams, so one kernel serves forward (windows x
// channel blocks), grad-input (flipped windows) and grad-weight (split-K
// over pixels, one window per blockIdx.z group).
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner +
// MMA issuer (one elected lane), warps 2..5 = epilogue (TMEM lane quarter
// = warp % 4).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

namespace syno {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;                 // one 128-byte swizzle row of bf16
constexpr int STAGES = 4;
constexpr int MAXWIN = 64;
constexpr int THREADS = 192;

enum Mode : int32_t {
  MODE_ROWS = 0,   // A rows = flat padded pixels (+ window shift); k = (cblock, window)
  MODE_WGRAD = 1,  // M = C_out, N = C_in, k = pixel rows (MN-major channels-last tiles); window = group
};

enum OutKind : int32_t { OUT_BF16 = 0, OUT_F32 = 1, OUT_F32_ATOMIC = 2 };

struct alignas(64) TcGemmParams {
  CUtensorMap tma_a;   // 3-D: [K elems][rows][plane]
  CUtensorMap tma_b;   // 3-D: [K elems][rows][plane]
  int32_t mode;
  int32_t n_cblocks;   // MODE_ROWS: channel blocks of 64; MODE_WGRAD: pixel blocks per window
  int32_t n_win;       // windows per group (MODE_ROWS) or groups (MODE_WGRAD)
  int32_t ksplit;      // MODE_WGRAD split of the pixel blocks
  int32_t a_shift[MAXWIN];   // MODE_ROWS: row shift of A per window; MODE_WGRAD: B row (pixel) shift
  int32_t a_plane[MAXWIN];   // plane (phase) of the shifted operand per window
  int32_t b_plane[MAXWIN];   // MODE_ROWS: B plane (packed weight window) per window
  // groups (blockIdx.z): MODE_ROWS uses win_base[g]..win_base[g]+win_count[g]
  int32_t win_base[8], win_count[8];
  int64_t g_out_off[8];
  int32_t a_row_base;        // MODE_ROWS: first flat row of the M tile grid
  // epilogue: row index r of the M tile -> output coordinates
  //   MODE_ROWS: flat = mtile*128 + r + a_row_base; (img, hp, wp) by Hp, Wp; h = hp - lo_h ...
  //   MODE_WGRAD: row = C_out index
  int32_t Hp, Wp, lo_h, lo_w, H, W, n_img;
  int64_t o_img, o_h, o_w, o_n, o_m;   // output element strides (o_m used by MODE_WGRAD rows)
  int32_t m_ext, n_ext;
  int32_t out_kind;
  float scale;
  void* out;
  uint32_t tx_bytes;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// K-major, 128-byte swizzle smem descriptor (canonical ((8,m),(T,2)) : ((8T,SBO),(1,T))).
__device__ __forceinline__ uint64_t sw128_desc(const void* smem) {
  uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFF;              // start address
  d |= (uint64_t)(16 >> 4) << 16;         // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                 // sm100 descriptor version
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// MN-major, 128-byte swizzle descriptor (canonical ((8,n),(8,k)) : ((1,LBO),(8,SBO)) in
// 16-byte units): 64 MN elements per 128 B row, one row per k; MN atoms of
// 64 elements are `lbo` bytes apart, 8-row k groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_mn_desc(const void* smem, uint32_t lbo) {
  uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFF;
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32; majors 0 = K, 1 = MN.
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, int a_mn = 0, int b_mn = 0) {
  return (1u << 4)            // D format f32
         | (1u << 7)          // A bf16
         | (1u << 10)         // B bf16
         | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16)
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t addr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

template <int BN>
__global__ void __launch_bounds__(THREADS, 1) tc_gemm_kernel(const __grid_constant__ TcGemmParams p) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = BN * BK * 2;
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int mt = blockIdx.x, nt = blockIdx.y;
  int g = blockIdx.z, ks = 0;
  if (p.mode == MODE_WGRAD) {
    ks = blockIdx.z % p.ksplit;
    g = blockIdx.z / p.ksplit;
  }
  // k-block range of this CTA
  int kb0, kb1, win0 = 0;
  if (p.mode == MODE_ROWS) {
    win0 = p.win_base[g];
    kb0 = 0;
    kb1 = p.win_count[g] * p.n_cblocks;
  } else {
    int per = (p.n_cblocks + p.ksplit - 1) / p.ksplit;
    kb0 = ks * per;
    kb1 = min(p.n_cblocks, kb0 + per);
    if (kb1 < kb0) kb1 = kb0;
  }
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tma_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tma_b)) : "memory");
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        const int kb = kb0 + i;
        mbar_expect_tx(&full[s], p.tx_bytes);
        if (p.mode == MODE_ROWS) {
          // K-major tiles: A = 128 pixel rows x 64 channels, B = BN rows x 64 channels
          const int cb = kb % p.n_cblocks;
          const int w = win0 + kb / p.n_cblocks;
          tma_load_3d(sa + s * A_BYTES, &p.tma_a, &full[s], cb * BK, p.a_row_base + mt * BM + p.a_shift[w],
                      p.a_plane[w]);
          tma_load_3d(sb + s * B_BYTES, &p.tma_b, &full[s], cb * BK, nt * BN, p.b_plane[w]);
        } else {
          // MN-major tiles from channels-last operands: 64 pixel rows (k) x 64 channels per box;
          // the window is a pixel-row shift of the x operand.
#pragma unroll
          for (int h = 0; h < BM / 64; ++h)
            tma_load_3d(sa + s * A_BYTES + h * 8192, &p.tma_a, &full[s], mt * BM + h * 64, kb * BK, 0);
#pragma unroll
          for (int h = 0; h < BN / 64; ++h)
            tma_load_3d(sb + s * B_BYTES + h * 8192, &p.tma_b, &full[s], nt * BN + h * 64, kb * BK + p.a_shift[g],
                        p.a_plane[g]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const bool mn = p.mode == MODE_WGRAD;
      const uint32_t idesc = mn ? idesc_bf16(BM, BN, 1, 1) : idesc_bf16(BM, BN);
      // per UMMA_K = 16 step: K-major advances 32 B inside the swizzled row,
      // MN-major advances two 8-row k groups (2 x 1024 B)
      const uint64_t kstep = mn ? (2048 >> 4) : (32 >> 4);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = mn ? sw128_mn_desc(sa + s * A_BYTES, 8192) : sw128_desc(sa + s * A_BYTES);
        const uint64_t db = mn ? sw128_mn_desc(sb + s * B_BYTES, 8192) : sw128_desc(sb + s * B_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          mma_bf16(tmem, da + (uint64_t)k * kstep, db + (uint64_t)k * kstep, idesc, (i > 0 || k > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
      }
      if (nkb > 0) mma_commit(tfull);
      else mbar_arrive(tfull);
    }
    __syncwarp();
  } else {
    // epilogue: TMEM lane quarter = warp % 4
    const int q = warp & 3;
    const int r = q * 32 + lane;
    mbar_wait(tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    bool ok;
    int64_t off;
    if (p.mode == MODE_ROWS) {
      const int64_t flat = (int64_t)mt * BM + r;
      const int64_t wp = flat % p.Wp;
      const int64_t t = flat / p.Wp;
      const int64_t hp = t % p.Hp;
      const int64_t img = t / p.Hp;
      const int64_t h = hp - p.lo_h, w = wp - p.lo_w;
      ok = img < p.n_img && h >= 0 && h < p.H && w >= 0 && w < p.W;
      off = p.g_out_off[g] + img * p.o_img + h * p.o_h + w * p.o_w;
    } else {
      const int64_t row = (int64_t)mt * BM + r;
      ok = row < p.m_ext;
      off = p.g_out_off[g] + row * p.o_m;
    }
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
      if (ok && nkb > 0) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int n = nt * BN + c + j;
          if (n < p.n_ext) {
            const int64_t o = off + (int64_t)n * p.o_n;
            const float val = v[j] * p.scale;
            if (p.out_kind == OUT_BF16) reinterpret_cast<__nv_bfloat16*>(p.out)[o] = __float2bfloat16(val);
            else if (p.out_kind == OUT_F32) reinterpret_cast<float*>(p.out)[o] = val;
            else atomicAdd(reinterpret_cast<float*>(p.out) + o, val);
          }
        }
      } else if (ok && p.out_kind != OUT_F32_ATOMIC) {
        for (int j = 0; j < 32; ++j) {
          const int n = nt * BN + c + j;
          if (n < p.n_ext) {
            const int64_t o = off + (int64_t)n * p.o_n;
            if (p.out_kind == OUT_BF16) reinterpret_cast<__nv_bfloat16*>(p.out)[o] = __float2bfloat16(0.f);
            else reinterpret_cast<float*>(p.out)[o] = 0.f;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

template <int BN>
constexpr int smem_bytes() {
  return 1024 + STAGES * (BM * BK * 2 + BN * BK * 2) + 256;
}

}  // namespace tc
}  // namespace syno
