// Tensor-core path: operator matcher, operand packing, weight folding and
// the three tcgen05 GEMM launches (forward, grad-input, grad-weight).
//
// Geometry of one windowed pixel dim (unfold over a strided data dim,
// pgraph.py:390-403): output index h reads input  S*h + r - c  for window
// r in [0, K).  Write  r - c = S*delta(r) + phi(r)  (floor division): the
// input is phase plane phi(r) of x (P_phi[u] = x[S*u + phi]) at u = h +
// delta(r).  Zero-padding every plane by lo/hi rows puts all windows of
// all output pixels on ONE flat padded grid, so a window is a constant row
// shift  delta_h*Wp + delta_w  of a 2-D operand and TMA tiles it directly
// (its out-of-bounds fill supplies the reference's "out of range reads
// zero", codegen.py:14-16).
#include "tc.hpp"

#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <type_traits>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <tuple>

#include "tc_gemm.cuh"

namespace syno {

using namespace tc;

constexpr int MAXFW = 4;  // weights of a fast fold

// ---------------------------------------------------------------------------
// TMA descriptors
// ---------------------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q),
               "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
    if (!p || q != cudaDriverEntryPointSuccess) fail(SYNO_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 3-D bf16 map [d0 (K, contiguous)][d1 (rows)][d2 (planes)], box [64][box1][1], 128B swizzle.
struct MapSpec {
  uint64_t d0 = 0, d1 = 0, d2 = 0, p1 = 0, p2 = 0;
  uint32_t box1 = 0;
};

static CUtensorMap make_map(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t pitch1_elems,
                            uint64_t pitch2_elems, uint32_t box1) {
  CUtensorMap m;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {pitch1_elems * 2, pitch2_elems * 2};
  cuuint32_t box[3] = {(cuuint32_t)BK, box1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SYNO_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

static CUtensorMap make_map(const void* base, const MapSpec& m) {
  return make_map(base, m.d0, m.d1, m.d2, m.p1, m.p2, m.box1);
}

static MapSpec map_spec(uint64_t d0, uint64_t d1, uint64_t d2, uint64_t p1, uint64_t p2, uint32_t box1) {
  MapSpec m;
  m.d0 = d0;
  m.d1 = d1;
  m.d2 = d2;
  m.p1 = p1;
  m.p2 = p2;
  m.box1 = box1;
  return m;
}

// ---------------------------------------------------------------------------
// Packing kernels (bandwidth-bound layout transforms)
// ---------------------------------------------------------------------------

// fp32 operands run on the bf16 tensor cores as split pairs v = hi + lo
// (hi = bf16(v), lo = bf16(v - hi)); a product x*w is recovered to ~2^-17
// relative as xh*wh + xh*wl + xl*wh, i.e. a GEMM over THREE parts of the
// contraction dim with operand patterns A = (hi, hi, lo), B = (hi, lo, hi).
enum Split : int32_t {
  SPLIT_NONE = 0,
  SPLIT_CH = 1,   // parts along the channel (K) dim: dst channel c' = part*Cp + c
  SPLIT_IMG = 2,  // parts along the image dim (wgrad, K = pixels): dst image = part*n_img + img
};

struct PackGeom {
  int64_t s_img, s_c, s_h, s_w;  // source element strides
  int32_t C, Hin, Win;           // source extents
  int32_t Sh, Sw;                // phase counts (strides)
  int32_t lo_h, lo_w, Hp, Wp;    // padded plane grid
  int32_t n_img;                 // source images
  int32_t Cp;                    // channels-last pitch of one part (multiple of 8)
  int32_t split;                 // Split
  uint32_t lo_mask;              // bit k: part k holds lo(v), else hi(v)
  int64_t Fpitch;                // channel-major row pitch (multiple of 8)
  // pack blocks cover PK_PIX consecutive pixels of the flattened (image, h, w)
  // grid instead of whole rows: rows are contiguous (s_h = Win, s_w = 1), so
  // V-wide loads work whenever the image plane (Hin x Win) is a multiple of
  // V, also for rows that are not (14 x 14 maps).  2 = plane blocks: one
  // image x 64 channels per block (Hin x Win <= PK_PIX), read as one
  // contiguous run of 64 channel planes (s_c = Hin x Win) with 16-byte loads
  // whatever the plane size (7 x 7 maps)
  int32_t flat = 0;
  __host__ __device__ int32_t parts() const { return split == SPLIT_NONE ? 1 : 3; }
  __host__ __device__ int32_t n_img_out() const { return split == SPLIT_IMG ? 3 * n_img : n_img; }
  __host__ __device__ int32_t Ct() const { return split == SPLIT_CH ? 3 * Cp : Cp; }  // dst channel pitch
};

// dst[plane][img'][hp][wp][c'] (flat pixel f = ((plane*n_img' + img')*Hp + hp)*Wp + wp),
// zero outside the source.  A block moves 64 consecutive flat pixels x 64
// destination channels through shared memory: lanes walk pixels for the
// NCHW reads (coalesced along w), 8 threads per pixel write 16-byte
// channel chunks.
template <typename TI>
__global__ void __launch_bounds__(256) pack_cl_kernel(const TI* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                                      PackGeom g, int64_t total_pix) {
  pdl_trigger();
  pdl_wait();
  __shared__ __nv_bfloat16 tile[64][66];
  const int64_t f0 = (int64_t)blockIdx.x * 64;
  const int cb = blockIdx.y;
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const int n_out = g.n_img_out();
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int64_t f = f0 + lane + 32 * half;
    bool inb = f < total_pix;
    const TI* row = src;
    int part = 0;
    if (inb) {
      const int wp = (int)(f % g.Wp);
      int64_t q = f / g.Wp;
      const int hp = (int)(q % g.Hp);
      q /= g.Hp;
      int img = (int)(q % n_out);
      const int plane = (int)(q / n_out);
      if (g.split == SPLIT_IMG) {
        part = img / g.n_img;
        img -= part * g.n_img;
      }
      const int hi = g.Sh * (hp - g.lo_h) + plane / g.Sw;
      const int wi = g.Sw * (wp - g.lo_w) + plane % g.Sw;
      inb = hi >= 0 && hi < g.Hin && wi >= 0 && wi < g.Win;
      row = src + img * g.s_img + (int64_t)hi * g.s_h + (int64_t)wi * g.s_w;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int cl = warp * 8 + k;
      int c = cb * 64 + cl;
      int pt = part;
      if (g.split == SPLIT_CH) {
        pt = c / g.Cp;
        c -= pt * g.Cp;
      }
      float v = 0.f;
      if (inb && c < g.C && pt < g.parts()) v = (float)row[c * g.s_c];
      __nv_bfloat16 hv = __float2bfloat16(v);
      if (g.split != SPLIT_NONE && ((g.lo_mask >> pt) & 1u)) hv = __float2bfloat16(v - __bfloat162float(hv));
      tile[cl][lane + 32 * half] = hv;
    }
  }
  __syncthreads();
  const int Ct = g.Ct();
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int w = t / 8 + 32 * half, cc = (t % 8) * 8;
    const int64_t f = f0 + w;
    const int c0 = cb * 64 + cc;
    if (f < total_pix && c0 < Ct) {
      __align__(16) __nv_bfloat16 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = tile[cc + k][w];
      *reinterpret_cast<uint4*>(dst + f * Ct + c0) = *reinterpret_cast<const uint4*>(v);
    }
  }
}

// Folded fp32 weights [rows][Cp] -> bf16 split parts [rows][3*Cp] (pattern lo_mask).
__global__ void __launch_bounds__(256) split_rows_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                                         int64_t rows, int32_t Cp, uint32_t lo_mask) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = rows * 3 * (int64_t)Cp;
  if (i >= total) return;
  const int64_t r = i / (3 * (int64_t)Cp);
  const int cc = (int)(i - r * 3 * (int64_t)Cp);
  const int part = cc / Cp, c = cc - part * Cp;
  const float v = src[r * Cp + c];
  __nv_bfloat16 hv = __float2bfloat16(v);
  if ((lo_mask >> part) & 1u) hv = __float2bfloat16(v - __bfloat162float(hv));
  dst[i] = hv;
}

// Source-row packer: each block moves PK_PIX consecutive source pixels
// (whole rows of one image plane) x 64 destination channels.  Reads walk
// each channel's pixels contiguously (vectorised when the row allows),
// the tile is transposed in shared memory, and every destination pixel's
// 64 channels go out as 128 contiguous bytes.  Only data positions are
// written: the padding of the flat grid is zeroed once when the workspace
// is built and never changes.
#ifndef SYNO_PK_PIX
#define SYNO_PK_PIX 128
#endif
constexpr int PK_PIX = SYNO_PK_PIX;  // <= 256 (one thread per pixel in the index phase)
constexpr int PK_NQ = PK_PIX / 16;   // vector loads per thread of the bf16 read phase (cstep >= 1024 / PK_PIX)

template <typename TI, int V>
__device__ __forceinline__ void pack_rows_body(const TI* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                               const PackGeom& g, int32_t rows_per_block, int64_t total_rows,
                                               unsigned bx, unsigned by) {
  // channel-major tile: row cl holds the block's pixels; each group of 8
  // channel rows is rotated by 8 pixels so the transposed reads of the write
  // phase spread over all banks (the rotation keeps 16-byte alignment)
  __shared__ __align__(16) __nv_bfloat16 tile[64][PK_PIX + 8];
  __shared__ int64_t s_src[PK_PIX];    // per block row: source offset of (image, row, first pixel)
  __shared__ int64_t s_dst[PK_PIX];    // per block pixel: destination flat pixel index (-1: not stored)
  __shared__ int32_t s_part[PK_PIX];
  const int t = threadIdx.x;
  const int cb = (int)by;
  const int n_out = g.n_img_out();
  // rows of <= PK_PIX pixels: rows_per_block whole rows; wider rows: one PK_PIX segment per block
  int64_t row0 = 0;
  int nrows = 0, wbeg = 0, Win = g.Win;
  const int64_t HW = (int64_t)g.Hin * g.Win;
  const int64_t q0 = (int64_t)bx * PK_PIX;  // flat mode: first pixel of the block
  if (g.flat) {
    // (flat mode: SPLIT_NONE only, so output image = source image)
  } else if (g.Win <= PK_PIX) {
    row0 = (int64_t)bx * rows_per_block;
    nrows = (int)min((int64_t)rows_per_block, total_rows - row0);
    wbeg = 0;
    Win = g.Win;
  } else {
    const int nseg = (g.Win + PK_PIX - 1) / PK_PIX;
    row0 = bx / nseg;
    nrows = 1;
    wbeg = (int)(bx % nseg) * PK_PIX;
    Win = min(PK_PIX, g.Win - wbeg);
  }
  const int npix = g.flat == 2 ? (int)HW : g.flat ? (int)min((int64_t)PK_PIX, (int64_t)n_out * HW - q0) : nrows * Win;
  if (g.flat) {
    if (t < npix) {
      const int64_t q = g.flat == 2 ? (int64_t)bx * HW + t : q0 + t;
      const int imgo = (int)(q / HW);
      const int rem = (int)(q - (int64_t)imgo * HW);
      const int hi = rem / g.Win, wi = rem - hi * g.Win;
      const int ph = hi % g.Sh, hp = hi / g.Sh + g.lo_h;
      const int pw = wi % g.Sw, wp = wi / g.Sw + g.lo_w;
      s_dst[t] = (hp < g.Hp && wp < g.Wp)
                     ? (((int64_t)(ph * g.Sw + pw) * n_out + imgo) * g.Hp + hp) * g.Wp + wp
                     : -1;
    }
  } else if (t < nrows) {
    const int64_t row = row0 + t;  // (img', hi) flattened
    int img = (int)(row / g.Hin);
    const int hi = (int)(row - (int64_t)img * g.Hin);
    int part = 0;
    if (g.split == SPLIT_IMG) {
      part = img / g.n_img;
      img -= part * g.n_img;
    }
    s_part[t] = part;
    s_src[t] = img * g.s_img + (int64_t)hi * g.s_h + (int64_t)wbeg * g.s_w;
  }
  if (!g.flat && t < npix) {
    const int rr = t / Win, wi = wbeg + t - rr * Win;
    const int64_t row = row0 + rr;
    const int imgo = (int)(row / g.Hin);
    const int hi = (int)(row - (int64_t)imgo * g.Hin);
    const int ph = hi % g.Sh, hp = hi / g.Sh + g.lo_h;
    const int pw = wi % g.Sw, wp = wi / g.Sw + g.lo_w;
    s_dst[t] = (hp < g.Hp && wp < g.Wp)
                   ? (((int64_t)(ph * g.Sw + pw) * n_out + imgo) * g.Hp + hp) * g.Wp + wp
                   : -1;  // never read by any window
  }
  __syncthreads();
  if (g.flat == 2) {
    // plane blocks: the block's 64 channel planes of image bx are one
    // contiguous run; 16-byte loads walk it and scatter into the tile
    constexpr int VE = 16 / (int)sizeof(TI);
    const int nval = max(0, min(64, g.C - cb * 64));
    const TI* base = src + (int64_t)bx * g.s_img + (int64_t)cb * 64 * g.s_c;
    const int n_el = nval * npix;  // multiple of VE: host-checked (HW * 64 and the tail)
    for (int e = t * VE; e < n_el; e += 256 * VE) {
      __align__(16) TI q[VE];
      *reinterpret_cast<uint4*>(q) = __ldg(reinterpret_cast<const uint4*>(base + e));
#pragma unroll
      for (int j = 0; j < VE; ++j) {
        const int cl = (e + j) / npix, px = (e + j) - cl * npix;
        tile[cl][(px + 8 * (cl >> 3)) & (PK_PIX - 1)] = __float2bfloat16((float)q[j]);
      }
    }
    // channels past C: zero rows
    for (int e = nval * npix + t; e < 64 * npix; e += 256) {
      const int cl = e / npix, px = e - cl * npix;
      tile[cl][(px + 8 * (cl >> 3)) & (PK_PIX - 1)] = __float2bfloat16(0.f);
    }
  } else {
  // ---- read: each thread keeps one pixel vector and walks the channels
  const int vpr = g.flat ? 1 : Win / V;  // vectors per row
  const int nvec = g.flat ? npix / V : nrows * vpr;  // <= PK_PIX / V
  const int cstep = max(1, 256 / nvec);
  if (t < cstep * nvec) {
    const int vi = t % nvec;
    int px0;
    const TI* rowp;
    int part0 = 0;
    if (g.flat) {
      // a vector never straddles two images: HW and q0 are multiples of V
      px0 = vi * V;
      const int64_t q = q0 + px0;
      const int64_t img = q / HW;
      rowp = src + img * g.s_img + (q - img * HW);
    } else {
      const int rr = vi / vpr;
      const int w0 = (vi - rr * vpr) * V;
      px0 = rr * Win + w0;
      rowp = src + s_src[rr] + (int64_t)w0 * g.s_w;
      part0 = s_part[rr];
    }
    if constexpr (sizeof(TI) == 2 && V >= 4) {
      // bf16, vector rows: every load of the thread in flight before any
      // shared-memory store (<= PK_NQ per thread: nvec <= PK_PIX / 4 so
      // cstep >= 1024 / PK_PIX); the block's run is one latency round
      using VT = typename std::conditional<V == 8, uint4, uint2>::type;
      VT qv[PK_NQ];
      const int cl0 = t / nvec;
#pragma unroll
      for (int it = 0; it < PK_NQ; ++it) {
        const int cl = cl0 + it * cstep;
        const int c = cb * 64 + cl;
        qv[it] = VT{};
        if (cl < 64 && c < g.C) qv[it] = __ldg(reinterpret_cast<const VT*>(rowp + (int64_t)c * g.s_c));
      }
#pragma unroll
      for (int it = 0; it < PK_NQ; ++it) {
        const int cl = cl0 + it * cstep;
        if (cl >= 64) break;
        __nv_bfloat16* trow = &tile[cl][0];
        if constexpr (V == 8) {
          *reinterpret_cast<uint4*>(trow + ((px0 + 8 * (cl >> 3)) & (PK_PIX - 1))) = qv[it];
        } else {
          const __nv_bfloat16* hq = reinterpret_cast<const __nv_bfloat16*>(&qv[it]);
#pragma unroll
          for (int e = 0; e < 4; ++e) trow[(px0 + e + 8 * (cl >> 3)) & (PK_PIX - 1)] = hq[e];
        }
      }
    } else if constexpr (sizeof(TI) == 4 && V == 4) {
      // fp32, 4-pixel vectors (cfg1's split operands): as the bf16 form, every
      // load of the thread in flight before any conversion (<= PK_NQ: cstep
      // >= 1024 / PK_PIX); the serial two-at-a-time loop took 13 us for 2 MB
      float4 qf[PK_NQ];
      int partv[PK_NQ];
      const int cl0 = t / nvec;
#pragma unroll
      for (int it = 0; it < PK_NQ; ++it) {
        const int cl = cl0 + it * cstep;
        int c = cb * 64 + cl, part = part0;
        if (g.split == SPLIT_CH) {
          part = c / g.Cp;
          c -= part * g.Cp;
        }
        partv[it] = part;
        qf[it] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (cl < 64 && c < g.C && part < g.parts()) qf[it] = __ldg(reinterpret_cast<const float4*>(rowp + (int64_t)c * g.s_c));
      }
#pragma unroll
      for (int it = 0; it < PK_NQ; ++it) {
        const int cl = cl0 + it * cstep;
        if (cl >= 64) break;
        const float v[4] = {qf[it].x, qf[it].y, qf[it].z, qf[it].w};
        const bool lo = g.split != SPLIT_NONE && ((g.lo_mask >> partv[it]) & 1u);
        __nv_bfloat16* trow = &tile[cl][0];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat16 hv = __float2bfloat16(v[e]);
          if (lo) hv = __float2bfloat16(v[e] - __bfloat162float(hv));
          trow[(px0 + e + 8 * (cl >> 3)) & (PK_PIX - 1)] = hv;
        }
      }
    } else
#pragma unroll 2
    for (int cl = t / nvec; cl < 64; cl += cstep) {
      int c = cb * 64 + cl;
      int part = part0;
      if (g.split == SPLIT_CH) {
        part = c / g.Cp;
        c -= part * g.Cp;
      }
      const bool have = c < g.C && part < g.parts();
      __nv_bfloat16* trow = &tile[cl][0];
      const int col0 = (px0 + 8 * (cl >> 3)) & (PK_PIX - 1);
      if constexpr (sizeof(TI) == 2) {
        // bf16 sources are never split: move the bits untouched
        if constexpr (V == 8) {
          uint4 q = make_uint4(0, 0, 0, 0);
          if (have) q = __ldg(reinterpret_cast<const uint4*>(rowp + (int64_t)c * g.s_c));
          *reinterpret_cast<uint4*>(trow + col0) = q;
        } else if constexpr (V == 4) {
          uint2 q = make_uint2(0, 0);
          if (have) q = __ldg(reinterpret_cast<const uint2*>(rowp + (int64_t)c * g.s_c));
          const __nv_bfloat16* hq = reinterpret_cast<const __nv_bfloat16*>(&q);
#pragma unroll
          for (int e = 0; e < 4; ++e) trow[(px0 + e + 8 * (cl >> 3)) & (PK_PIX - 1)] = hq[e];
        } else {
          const __nv_bfloat16 z = __float2bfloat16(0.f);
          trow[(px0 + 8 * (cl >> 3)) & (PK_PIX - 1)] = have ? rowp[(int64_t)c * g.s_c] : z;
        }
        continue;
      } else {
      float v[V];
      if (have) {
        const TI* p = rowp + (int64_t)c * g.s_c;
        if (V == 8 && sizeof(TI) == 2) {
          const uint4 q = __ldg(reinterpret_cast<const uint4*>(p));
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f2 = __bfloat1622float2(h2[e]);
            v[2 * e] = f2.x;
            v[2 * e + 1] = f2.y;
          }
        } else if (V == 4 && sizeof(TI) == 2) {
          const uint2 q = __ldg(reinterpret_cast<const uint2*>(p));
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float2 f2 = __bfloat1622float2(h2[e]);
            v[2 * e] = f2.x;
            v[2 * e + 1] = f2.y;
          }
        } else if (V == 4 && sizeof(TI) == 4) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(p));
          v[0] = q.x;
          v[1] = q.y;
          v[2] = q.z;
          v[3] = q.w;
        } else {
#pragma unroll
          for (int e = 0; e < V; ++e) v[e] = (float)p[(int64_t)e * g.s_w];
        }
      } else {
#pragma unroll
        for (int e = 0; e < V; ++e) v[e] = 0.f;
      }
      const bool lo = g.split != SPLIT_NONE && ((g.lo_mask >> part) & 1u);
      __align__(16) __nv_bfloat16 hv[V];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        hv[e] = __float2bfloat16(v[e]);
        if (lo) hv[e] = __float2bfloat16(v[e] - __bfloat162float(hv[e]));
      }
      if (V == 8) {  // px0 and the rotation are multiples of 8: one 16-byte store
        *reinterpret_cast<uint4*>(trow + col0) = *reinterpret_cast<const uint4*>(hv);
      } else {
#pragma unroll
        for (int e = 0; e < V; ++e) trow[(px0 + e + 8 * (cl >> 3)) & (PK_PIX - 1)] = hv[e];
      }
      }
    }
  }
  }  // row / flat blocks
  __syncthreads();
  // ---- write: 8 threads per destination pixel, 16 bytes each
  const int Ct = g.Ct();
  const int chunk = t & 7;
  const int c0 = cb * 64 + chunk * 8;
  if (c0 >= Ct) return;
#pragma unroll 4
  for (int px = t >> 3; px < npix; px += 32) {
    const int64_t f = s_dst[px];
    if (f < 0) continue;
    __align__(16) __nv_bfloat16 q[8];
    const int col = (px + 8 * chunk) & (PK_PIX - 1);
#pragma unroll
    for (int k = 0; k < 8; ++k) q[k] = tile[chunk * 8 + k][col];
    *reinterpret_cast<uint4*>(dst + f * Ct + c0) = *reinterpret_cast<const uint4*>(q);
  }
}

template <typename TI, int V>
__global__ void __launch_bounds__(256) pack_rows_kernel(const TI* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                                        PackGeom g, int32_t rows_per_block, int64_t total_rows) {
  pdl_trigger();
  pdl_wait();
  pack_rows_body<TI, V>(src, dst, g, rows_per_block, total_rows, blockIdx.x, blockIdx.y);
}

// ---------------------------------------------------------------------------
// Weight transforms (fold into the B operand, chain rule out of dWf)
// ---------------------------------------------------------------------------

struct FoldArgs {
  const void* w[MAXFW];
  int64_t s[MAXFW][4];   // strides along fold slots (rh, rw, n, ci)
  int32_t nw, f32;       // weight dtype: f32 or bf16
  int32_t ext[4];        // Kh, Kw, A, B extents (A/B = rows/cols of the operand)
  int32_t sl_a, sl_b;    // fold slots of A and B (2 = n, 3 = ci)
  int32_t Bp;            // padded B pitch of one part
  int32_t split;         // 1: three bf16 parts (hi, lo, hi) at pitch 3*Bp
  __nv_bfloat16* out;
};

// out[rh][rw][a][b'] = prod_j w_j[...]; one block row per (rh, rw, a).
__global__ void __launch_bounds__(128) fold_kernel(const __grid_constant__ FoldArgs f) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.y;
  const int a = row % f.ext[2];
  const int rw = (row / f.ext[2]) % f.ext[1];
  const int rh = row / (f.ext[2] * f.ext[1]);
  const int parts = f.split ? 3 : 1;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < f.Bp; b += gridDim.x * blockDim.x) {
    float v = 0.f;
    if (b < f.ext[3]) {
      v = 1.f;
      for (int j = 0; j < f.nw; ++j) {
        const int64_t off = rh * f.s[j][0] + rw * f.s[j][1] + (int64_t)a * f.s[j][f.sl_a] + (int64_t)b * f.s[j][f.sl_b];
        v *= f.f32 ? __ldg(reinterpret_cast<const float*>(f.w[j]) + off)
                   : __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(f.w[j]) + off));
      }
    }
    __nv_bfloat16* o = f.out + (int64_t)row * parts * f.Bp + b;
    const __nv_bfloat16 hi = __float2bfloat16(v);
    o[0] = hi;
    if (parts == 3) {
      o[f.Bp] = __float2bfloat16(v - __bfloat162float(hi));
      o[2 * f.Bp] = hi;
    }
  }
}

// Tiled fold: a block covers TA operand rows x TB operand columns for every
// window k = (rh, rw).  Weights are read in an order that follows the
// dominant weight's memory layout (k fastest, then the loop with the smaller
// stride), staged in shared memory as fp32, and written back as coalesced
// bf16 rows (split into (hi, lo, hi) parts for fp32 operands).
// Direct fold: block = (operand row a, 64 operand columns); thread =
// (column, window phase).  Output rows are written coalesced along b; the
// weights are read through the read-only cache (neighbouring windows of the
// same weight element run in other iterations / threads of the block).
__device__ __forceinline__ void fold_direct_body(const FoldArgs& f, unsigned bx, unsigned by) {
  __shared__ int32_t koff[MAXFW][16];
  const int KK = f.ext[0] * f.ext[1];
  if ((int)threadIdx.x < KK) {
    const int rh = threadIdx.x / f.ext[1], rw = threadIdx.x - rh * f.ext[1];
#pragma unroll
    for (int j = 0; j < MAXFW; ++j)
      if (j < f.nw) koff[j][threadIdx.x] = (int32_t)(rh * f.s[j][0] + rw * f.s[j][1]);
  }
  __syncthreads();
  const int a = (int)bx;
  const int b = (int)by * 64 + (threadIdx.x & 63);
  if (b >= f.Bp) return;
  const bool inb = b < f.ext[3];
  int32_t base[MAXFW];
#pragma unroll
  for (int j = 0; j < MAXFW; ++j)
    base[j] = j < f.nw ? (int32_t)(a * f.s[j][f.sl_a] + (int64_t)b * f.s[j][f.sl_b]) : 0;
  const int parts = f.split ? 3 : 1;
#pragma unroll 4
  for (int k = threadIdx.x >> 6; k < KK; k += 4) {
    float v = 0.f;
    if (inb) {
      v = 1.f;
#pragma unroll
      for (int j = 0; j < MAXFW; ++j) {
        if (j >= f.nw) break;
        const int32_t off = base[j] + koff[j][k];
        v *= f.f32 ? __ldg(reinterpret_cast<const float*>(f.w[j]) + off)
                   : __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(f.w[j]) + off));
      }
    }
    __nv_bfloat16* o = f.out + ((int64_t)k * f.ext[2] + a) * parts * f.Bp + b;
    const __nv_bfloat16 hi = __float2bfloat16(v);
    o[0] = hi;
    if (parts == 3) {
      o[f.Bp] = __float2bfloat16(v - __bfloat162float(hi));
      o[2 * f.Bp] = hi;
    }
  }
}

__global__ void __launch_bounds__(256) fold_direct_kernel(const __grid_constant__ FoldArgs f) {
  pdl_trigger();
  pdl_wait();
  fold_direct_body(f, blockIdx.x, blockIdx.y);
}

// One launch for the two independent per-call operand preparations of a
// GEMM: blocks [0, n_pack) pack the activations, the rest fold the weights.
template <typename TI, int V>
__global__ void __launch_bounds__(256) prep_kernel(const TI* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                                   PackGeom g, int32_t rows_per_block, int64_t total_rows,
                                                   uint32_t pack_gx, uint32_t n_pack, const __grid_constant__ FoldArgs f,
                                                   uint32_t fold_gx) {
  pdl_trigger();
  pdl_wait();
  const uint32_t b = blockIdx.x;
  if (b < n_pack) pack_rows_body<TI, V>(src, dst, g, rows_per_block, total_rows, b % pack_gx, b / pack_gx);
  else fold_direct_body(f, (b - n_pack) % fold_gx, (b - n_pack) / fold_gx);
}

template <int TA, int TB>
__global__ void __launch_bounds__(256) fold_tile_kernel(const __grid_constant__ FoldArgs f, int a_inner) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sv[];  // [KK][TA][TB + 1]
  __shared__ int32_t koff[MAXFW][16];
  const int KK = f.ext[0] * f.ext[1];
  if ((int)threadIdx.x < KK) {
    const int rh = threadIdx.x / f.ext[1], rw = threadIdx.x - rh * f.ext[1];
#pragma unroll
    for (int j = 0; j < MAXFW; ++j)
      if (j < f.nw) koff[j][threadIdx.x] = (int32_t)(rh * f.s[j][0] + rw * f.s[j][1]);
  }
  int32_t sa[MAXFW], sb[MAXFW];
#pragma unroll
  for (int j = 0; j < MAXFW; ++j) {
    sa[j] = j < f.nw ? (int32_t)f.s[j][f.sl_a] : 0;
    sb[j] = j < f.nw ? (int32_t)f.s[j][f.sl_b] : 0;
  }
  __syncthreads();
  const int a0 = blockIdx.x * TA, b0 = blockIdx.y * TB;
  const int n_el = KK * TA * TB;
#pragma unroll 4
  for (int i = threadIdx.x; i < n_el; i += blockDim.x) {
    const int q = i / KK;
    const int k = i - q * KK;
    const int al = a_inner ? q % TA : q / TB;
    const int bl = a_inner ? q / TA : q % TB;
    const int a = a0 + al, b = b0 + bl;
    float v = 0.f;
    if (a < f.ext[2] && b < f.ext[3]) {
      v = 1.f;
#pragma unroll
      for (int j = 0; j < MAXFW; ++j) {
        if (j >= f.nw) break;
        const int32_t off = koff[j][k] + a * sa[j] + b * sb[j];
        v *= f.f32 ? __ldg(reinterpret_cast<const float*>(f.w[j]) + off)
                   : __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(f.w[j]) + off));
      }
    }
    sv[(k * TA + al) * (TB + 1) + bl] = v;
  }
  __syncthreads();
  const int parts = f.split ? 3 : 1;
#pragma unroll 4
  for (int i = threadIdx.x; i < n_el; i += blockDim.x) {
    const int bl = i % TB;
    const int al = (i / TB) % TA;
    const int k = i / (TA * TB);
    const int a = a0 + al, b = b0 + bl;
    if (a >= f.ext[2] || b >= f.Bp) continue;
    const float v = sv[(k * TA + al) * (TB + 1) + bl];
    __nv_bfloat16* o = f.out + ((int64_t)k * f.ext[2] + a) * parts * f.Bp + b;
    const __nv_bfloat16 hi = __float2bfloat16(v);
    o[0] = hi;
    if (parts == 3) {
      o[f.Bp] = __float2bfloat16(v - __bfloat162float(hi));
      o[2 * f.Bp] = hi;
    }
  }
}

// Both B operands in one pass: Wf[k][n][ci] (forward) and Wt[k][ci][n]
// (grad-input) from a 32 x 32 (n, ci) tile staged in shared memory for every
// window k; reads follow the weight's memory order (k fastest, then ci),
// both outputs are written as coalesced rows.
struct FoldDual {
  FoldArgs f;                 // f.out = Wf, f.Bp = Cp (ci pitch per part); ext = {Kh, Kw, N, C}
  __nv_bfloat16* out_t;       // Wt
  int32_t Np;                 // n pitch per part of Wt
};

__global__ void __launch_bounds__(256) fold_dual_kernel(const __grid_constant__ FoldDual d) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sv[];  // [KK][32][33]
  __shared__ int32_t koff[MAXFW][16];
  const FoldArgs& f = d.f;
  const int KK = f.ext[0] * f.ext[1];
  if ((int)threadIdx.x < KK) {
    const int rh = threadIdx.x / f.ext[1], rw = threadIdx.x - rh * f.ext[1];
    for (int j = 0; j < f.nw; ++j) koff[j][threadIdx.x] = (int32_t)(rh * f.s[j][0] + rw * f.s[j][1]);
  }
  __syncthreads();
  const int n0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int N = f.ext[2], C = f.ext[3];
#pragma unroll 1
  for (int i = threadIdx.x; i < 32 * 32 * KK; i += blockDim.x) {
    const int k = i % KK;
    const int q = i / KK;
    const int cl = q % 32, nl = q / 32;
    const int n = n0 + nl, ci = c0 + cl;
    float v = 0.f;
    if (n < N && ci < C) {
      v = 1.f;
      for (int j = 0; j < f.nw; ++j) {
        const int32_t off = koff[j][k] + n * (int32_t)f.s[j][2] + ci * (int32_t)f.s[j][3];
        v *= f.f32 ? __ldg(reinterpret_cast<const float*>(f.w[j]) + off)
                   : __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(f.w[j]) + off));
      }
    }
    sv[(k * 32 + nl) * 33 + cl] = v;
  }
  __syncthreads();
  const int parts = f.split ? 3 : 1;
  // Wf rows (k, n): ci contiguous
#pragma unroll 1
  for (int i = threadIdx.x; i < 32 * 32 * KK; i += blockDim.x) {
    const int cl = i % 32, nl = (i / 32) % 32, k = i / 1024;
    const int n = n0 + nl, ci = c0 + cl;
    if (n >= N || ci >= f.Bp) continue;
    const float v = sv[(k * 32 + nl) * 33 + cl];
    __nv_bfloat16* o = f.out + ((int64_t)k * N + n) * parts * f.Bp + ci;
    const __nv_bfloat16 hi = __float2bfloat16(v);
    o[0] = hi;
    if (parts == 3) {
      o[f.Bp] = __float2bfloat16(v - __bfloat162float(hi));
      o[2 * f.Bp] = hi;
    }
  }
  // Wt rows (k, ci): n contiguous
#pragma unroll 1
  for (int i = threadIdx.x; i < 32 * 32 * KK; i += blockDim.x) {
    const int nl = i % 32, cl = (i / 32) % 32, k = i / 1024;
    const int n = n0 + nl, ci = c0 + cl;
    if (ci >= C || n >= d.Np) continue;
    const float v = sv[(k * 32 + nl) * 33 + cl];
    __nv_bfloat16* o = d.out_t + ((int64_t)k * C + ci) * parts * d.Np + n;
    const __nv_bfloat16 hi = __float2bfloat16(v);
    o[0] = hi;
    if (parts == 3) {
      o[d.Np] = __float2bfloat16(v - __bfloat162float(hi));
      o[2 * d.Np] = hi;
    }
  }
}

struct ChainArgs {
  float* dwf;            // [Kh][Kw][N][C] fp32
  int32_t zero_dwf;      // last reader: leave dWf zeroed for the next grad-weight (no memset)
  const void* w[MAXFW];
  int64_t s[MAXFW][4];
  int32_t nw, j, f32;    // weights, the weight differentiated, dtype of w / out
  int32_t ext[4];        // Kh, Kw, N, C
  int32_t nout, nred;
  int32_t out_l[4], red_l[4];  // fold slots of the output / reduced loops (ascending)
  int64_t out_count, R, r_chunk;
  void* out;
  float* partial;        // [out_count][nsplit] (block mode)
  unsigned* counter;     // [out_count], zero between calls (block mode)
};

__device__ __forceinline__ float chain_term(const ChainArgs& c, const int* d) {
  const int64_t df = ((int64_t)(d[0] * c.ext[1] + d[1]) * c.ext[2] + d[2]) * c.ext[3] + d[3];
  float v = __ldg(c.dwf + df);
#pragma unroll 1
  for (int k = 0; k < c.nw; ++k) {
    if (k == c.j) continue;
    const int64_t off = d[0] * c.s[k][0] + d[1] * c.s[k][1] + (int64_t)d[2] * c.s[k][2] + (int64_t)d[3] * c.s[k][3];
    v *= c.f32 ? __ldg(reinterpret_cast<const float*>(c.w[k]) + off)
               : __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(c.w[k]) + off));
  }
  return v;
}

__device__ __forceinline__ void chain_decode(const ChainArgs& c, int64_t o64, int64_t r64, int* d) {
  // int32 digits: out_count and R are < 2^31 (checked on the host)
  int o = (int)o64, r = (int)r64;
  d[0] = d[1] = d[2] = d[3] = 0;
#pragma unroll 1
  for (int k = 3; k >= 0; --k) {
    if (k >= c.nout) continue;
    const int l = c.out_l[k];
    const int e = c.ext[l];
    d[l] = o % e;
    o /= e;
  }
#pragma unroll 1
  for (int k = 3; k >= 0; --k) {
    if (k >= c.nred) continue;
    const int l = c.red_l[k];
    const int e = c.ext[l];
    d[l] = r % e;
    r /= e;
  }
}

__device__ __forceinline__ void chain_store(const ChainArgs& c, const int* d, float v) {
  const int64_t off = d[0] * c.s[c.j][0] + d[1] * c.s[c.j][1] + (int64_t)d[2] * c.s[c.j][2] + (int64_t)d[3] * c.s[c.j][3];
  if (c.f32) reinterpret_cast<float*>(c.out)[off] = v;
  else reinterpret_cast<__nv_bfloat16*>(c.out)[off] = __float2bfloat16(v);
}

// dW_j = sum over the loops w_j does not use of dWf * prod_{k != j} w_k.
// Thread per output (short reductions), outputs ordered like dWf (ci fastest).
__global__ void __launch_bounds__(256) chain_thread_kernel(const __grid_constant__ ChainArgs c) {
  pdl_trigger();
  pdl_wait();
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= c.out_count) return;
  int d[4];
  float acc = 0.f;
  for (int64_t r = 0; r < c.R; ++r) {
    chain_decode(c, o, r, d);
    acc += chain_term(c, d);
    if (c.zero_dwf) c.dwf[((int64_t)(d[0] * c.ext[1] + d[1]) * c.ext[2] + d[2]) * c.ext[3] + d[3]] = 0.f;
  }
  chain_decode(c, o, 0, d);
  chain_store(c, d, acc);
}

// Chain rule for a weight that uses the n loop (every main weight): one
// block per (output channel n, chunk of input channels) stages
// dWf[:, :, n, chunk] (coalesced) in shared memory and produces those dW_j
// entries in dW_j's memory order, reducing over the loops the weight does
// not use (a window at most).  All index arithmetic is int32 with
// host-precomputed multipliers (digit -> smem / output / weight offsets).
struct ChainN {
  int32_t n_ol, n_rl;
  int32_t ol_ext[3], ol_sm[3], ol_out[3], ol_w[3][MAXFW];  // output loops in memory order (ci: chunk-local)
  int32_t rl_ext[3], rl_sm[3], rl_w[3][MAXFW];             // reduced loops
  int32_t n_out, n_w[MAXFW];                               // per-n offsets
  int32_t ci_q;                                            // position of ci among the output loops, -1 none
  int32_t ci_chunk;
  int32_t KK, C, Kw;
};

__global__ void __launch_bounds__(256) chain_n_kernel(const __grid_constant__ ChainArgs c, const __grid_constant__ ChainN h) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sd[];  // [KK][cw + 1]
  const int n = blockIdx.x;
  const int c_lo = h.ci_q >= 0 ? blockIdx.y * h.ci_chunk : 0;
  const int cw = h.ci_q >= 0 ? min(h.C - c_lo, h.ci_chunk) : h.C;
  const int P = cw + 1;
#pragma unroll 4
  for (int i = threadIdx.x; i < h.KK * cw; i += blockDim.x) {
    const int k = i / cw, ci = i - k * cw;
    float* src = c.dwf + ((int64_t)k * c.ext[2] + n) * h.C + c_lo + ci;
    sd[k * P + ci] = *src;
    if (c.zero_dwf) *src = 0.f;
  }
  __syncthreads();
  // per-block bases: n and the chunk start of ci
  int32_t base_out = n * h.n_out, base_w[MAXFW];
#pragma unroll
  for (int k = 0; k < MAXFW; ++k) base_w[k] = n * h.n_w[k];
  if (h.ci_q >= 0) {
    base_out += c_lo * h.ol_out[h.ci_q];
#pragma unroll
    for (int k = 0; k < MAXFW; ++k) base_w[k] += c_lo * h.ol_w[h.ci_q][k];
  }
  int ext[3];
  int m = 1;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    ext[q] = q < h.n_ol ? (q == h.ci_q ? cw : h.ol_ext[q]) : 1;
    m *= ext[q];
  }
  int R = 1;
#pragma unroll
  for (int q = 0; q < 3; ++q) R *= q < h.n_rl ? h.rl_ext[q] : 1;
#pragma unroll 2
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    int rem = i, o_out = base_out, o_sm = 0, o_w[MAXFW];
#pragma unroll
    for (int k = 0; k < MAXFW; ++k) o_w[k] = base_w[k];
#pragma unroll
    for (int q = 2; q >= 0; --q) {
      if (q >= h.n_ol) continue;
      const int dq = rem % ext[q];
      rem /= ext[q];
      o_out += dq * h.ol_out[q];
      o_sm += dq * h.ol_sm[q];
#pragma unroll
      for (int k = 0; k < MAXFW; ++k) o_w[k] += dq * h.ol_w[q][k];
    }
    float acc = 0.f;
    for (int r = 0; r < R; ++r) {
      int rr = r, r_sm = o_sm, r_w[MAXFW];
#pragma unroll
      for (int k = 0; k < MAXFW; ++k) r_w[k] = o_w[k];
#pragma unroll
      for (int q = 2; q >= 0; --q) {
        if (q >= h.n_rl) continue;
        const int dq = rr % h.rl_ext[q];
        rr /= h.rl_ext[q];
        r_sm += dq * h.rl_sm[q];
#pragma unroll
        for (int k = 0; k < MAXFW; ++k) r_w[k] += dq * h.rl_w[q][k];
      }
      float v = sd[r_sm];
#pragma unroll
      for (int k = 0; k < MAXFW; ++k) {
        if (k >= c.nw || k == c.j) continue;
        v *= c.f32 ? __ldg(reinterpret_cast<const float*>(c.w[k]) + r_w[k])
                   : __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(c.w[k]) + r_w[k]));
      }
      acc += v;
    }
    if (c.f32) reinterpret_cast<float*>(c.out)[o_out] = acc;
    else reinterpret_cast<__nv_bfloat16*>(c.out)[o_out] = __float2bfloat16(acc);
  }
}

// Chain rule for a weight that uses both channel loops (n, ci): one thread
// per (n, ci) walks the windows; dWf reads are coalesced along ci and each
// thread's outputs are contiguous in dW_j (window loops innermost in OIHW-
// style layouts).  Windows the weight does not use are reduced in-thread.
struct ChainNC {
  int32_t Kh, Kw, N, C;
  int32_t so_n, so_c, so_h, so_w;  // output strides (so_h / so_w = 0: reduced window loop)
  int32_t oh, ow;                  // rh / rw is an output loop
  int32_t sw[MAXFW][4];            // other weights' strides (0 for the differentiated one)
  int32_t dense;                   // dW_j is [n][ci][window outputs] dense: stage the block's outputs in smem
  // Side output: a second weight j2 that uses only window loops (sep_shared's
  // shared [K] weight) takes its gradient from the same pass over dWf:
  // dW_j2[win] = sum_{n, ci} dWf * prod_{q != j2} w_q, reduced per block into
  // `partial` and combined in block order by the last block (deterministic).
  int32_t side_j;                  // -1: none
  int32_t side_sw[MAXFW][4];       // strides of every weight except j2 (0 for j2)
  int32_t side_oh, side_ow, side_so_h, side_so_w;
  void* side_out;
  float* partial;                  // [gridDim.x][KK]
  unsigned* counter;               // zero between calls
};

// KH / KW: compile-time window extents (0: runtime).  With them known the
// per-thread window values stay in registers (the runtime-bounded version
// spilled them to local memory: a 512 x 512 x 3 x 3 chain took 16 us).
template <int KH, int KW>
__global__ void __launch_bounds__(256) chain_nc_kernel(const __grid_constant__ ChainArgs c, const __grid_constant__ ChainNC h) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float stage[];  // [blockDim.x][KKo]: each thread's window outputs
  const int i32 = blockIdx.x * blockDim.x + threadIdx.x;  // N * C < 2^31 (host-checked)
  const int64_t i = i32;
  const bool live = i < (int64_t)h.N * h.C;
  const int n = live ? i32 / h.C : 0, ci = live ? i32 - n * h.C : 0;
  const int64_t plane = (int64_t)h.N * h.C;
  constexpr int KKT = KH * KW;
  constexpr int VN = KKT ? KKT : 16;
  const int Kw = KW ? KW : h.Kw;
  const int KK = KKT ? KKT : h.Kh * h.Kw;  // <= 16 (host-checked)
  const int KKo_w = h.ow ? Kw : 1;
  const int KKo = (h.oh ? (KH ? KH : h.Kh) : 1) * KKo_w;
  float* my = stage + threadIdx.x * KKo;
  for (int q = 0; q < KKo; ++q) my[q] = 0.f;
  if (live) {
    // all windows' loads in flight together, then the zeroing stores
    float* __restrict__ src = c.dwf + i;
    float v[VN];
#pragma unroll
    for (int k = 0; k < VN; ++k)
      if (k < KK) v[k] = src[k * plane];
    if (c.zero_dwf) {
#pragma unroll
      for (int k = 0; k < VN; ++k)
        if (k < KK) src[k * plane] = 0.f;
    }
    // per-thread window values of the side output (odd stride); the smem
    // region exists only when h.side_j >= 0 (a small block leaves room to
    // co-reside with a concurrent persistent GEMM CTA)
    float* vs = stage + blockDim.x * KKo + threadIdx.x * 17;
    // every other weight's value per window, all loads in flight before the
    // products (a serial load per (window, weight) made a 64 x 64
    // sep_shared chain a 16 us latency chain); the products below keep the
    // original multiplication order, so results are unchanged bit for bit
    float wv[MAXFW][VN];
#pragma unroll
    for (int q = 0; q < MAXFW; ++q) {
#pragma unroll
      for (int k = 0; k < VN; ++k) {
        wv[q][k] = 1.f;
        if (q >= c.nw || k >= KK || (q == c.j && h.side_j < 0)) continue;
        const int kh = k / Kw, kw = k - kh * Kw;
        const int32_t* st = q == c.j ? h.side_sw[q] : h.sw[q];  // sw[j] is zeroed: w_j only feeds the side
        const int32_t off = kh * st[0] + kw * st[1] + n * st[2] + ci * st[3];
        wv[q][k] = c.f32 ? __ldg(reinterpret_cast<const float*>(c.w[q]) + off)
                         : __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(c.w[q]) + off));
      }
    }
#pragma unroll
    for (int k = 0; k < VN; ++k) {
      if (k >= KK) break;
      const int kh = k / Kw, kw = k - kh * Kw;
      const float d = v[k];
      float x = d;
#pragma unroll
      for (int q = 0; q < MAXFW; ++q)
        if (q < c.nw && q != c.j) x *= wv[q][k];
      // windows the weight does not use fold onto the same output
      my[(h.oh ? kh : 0) * KKo_w + (h.ow ? kw : 0)] += x;
      if (h.side_j >= 0) {
        float z = d;
#pragma unroll
        for (int q = 0; q < MAXFW; ++q)
          if (q < c.nw && q != h.side_j) z *= wv[q][k];
        vs[k] = z;
      }
    }
  } else if (h.side_j >= 0) {
    float* vs = stage + blockDim.x * KKo + threadIdx.x * 17;
    for (int k = 0; k < KK; ++k) vs[k] = 0.f;
  }
  if (h.side_j >= 0) {
    // block sums of the side products per window, then the last block combines
    __syncthreads();
    const float* vall = stage + blockDim.x * KKo;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ float wsum[8][16];
    for (int k = 0; k < KK; ++k) {
      float t = 0.f;
      t = vall[(warp * 32 + lane) * 17 + k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) wsum[warp][k] = t;
    }
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x < KK) {
      float t = 0.f;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += wsum[q][threadIdx.x];
      h.partial[(size_t)blockIdx.x * KK + threadIdx.x] = t;
      __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(h.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) {
      __threadfence();
      // every thread sums a strided set of the blocks' partials per window,
      // then a fixed-shape tree adds the 256 thread sums: the result depends
      // only on gridDim, not on which block finished last
      // (in the side-product region of the dynamic stage: 256 x 17 floats,
      // free again; no static buffer, so the block stays small enough to
      // co-reside with a persistent GEMM CTA)
      float* red = stage + blockDim.x * KKo;  // [KK][blockDim.x]
      __shared__ float tot[16];
      for (int k = 0; k < KK; ++k) {
        float t = 0.f;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
          t += *((volatile float*)h.partial + (size_t)b * KK + k);
        red[k * blockDim.x + threadIdx.x] = t;
      }
      __syncthreads();
      for (int width = (int)blockDim.x >> 1; width > 0; width >>= 1) {
        for (int e = threadIdx.x; e < KK * width; e += blockDim.x) {
          const int k = e / width, q = e - k * width;
          red[k * blockDim.x + q] += red[k * blockDim.x + q + width];
        }
        __syncthreads();
      }
      if (threadIdx.x < KK) tot[threadIdx.x] = red[threadIdx.x * blockDim.x];
      __syncthreads();
      if (threadIdx.x == 0) {
        const int ow2 = h.side_ow ? h.Kw : 1;
        const int no = (h.side_oh ? h.Kh : 1) * ow2;
        float acc[16];
        for (int q = 0; q < no; ++q) acc[q] = 0.f;
        for (int k = 0; k < KK; ++k) {
          const int kh = k / h.Kw, kw = k - kh * h.Kw;
          acc[(h.side_oh ? kh : 0) * ow2 + (h.side_ow ? kw : 0)] += tot[k];
        }
        for (int q = 0; q < no; ++q) {
          const int ah = q / ow2, aw = q - ah * ow2;
          const int64_t o = (int64_t)ah * h.side_so_h + (int64_t)aw * h.side_so_w;
          if (c.f32) reinterpret_cast<float*>(h.side_out)[o] = acc[q];
          else reinterpret_cast<__nv_bfloat16*>(h.side_out)[o] = __float2bfloat16(acc[q]);
        }
        *h.counter = 0;  // ready for the next call (stream order)
      }
    }
  }
  if (!h.dense) {
    if (!live) return;
    const int64_t obase = (int64_t)n * h.so_n + (int64_t)ci * h.so_c;
    for (int q = 0; q < KKo; ++q) {
      const int ah = q / KKo_w, aw = q - ah * KKo_w;
      const int64_t o = obase + (int64_t)ah * h.so_h + (int64_t)aw * h.so_w;
      if (c.f32) reinterpret_cast<float*>(c.out)[o] = my[q];
      else reinterpret_cast<__nv_bfloat16*>(c.out)[o] = __float2bfloat16(my[q]);
    }
    return;
  }
  // dense [n][ci][windows] layout: the block's outputs are one contiguous run
  __syncthreads();
  const int64_t blk_base = (int64_t)blockIdx.x * blockDim.x * KKo;
  const int64_t total = plane * KKo;
  const int run = (int)min((int64_t)blockDim.x * KKo, total - blk_base);
  for (int e = threadIdx.x; e < run; e += blockDim.x) {
    if (c.f32) reinterpret_cast<float*>(c.out)[blk_base + e] = stage[e];
    else reinterpret_cast<__nv_bfloat16*>(c.out)[blk_base + e] = __float2bfloat16(stage[e]);
  }
}

// Single weight whose every window is an output (conv3x3, strided and 1x1
// convolutions): dW_j[n][ci][kh][kw] = dWf[k][n][ci], one thread per dWf
// element (coalesced reads and re-zeroing), grid.y over the windows, so even
// a 64 x 64 layer launches 16 x 9 blocks instead of 16 latency-bound ones.
__global__ void __launch_bounds__(256) chain_win_kernel(const __grid_constant__ ChainArgs c,
                                                        const __grid_constant__ ChainNC h) {
  pdl_trigger();
  pdl_wait();
  const int64_t plane = (int64_t)h.N * h.C;  // < 2^31 (host-checked)
  const int i32 = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = i32;
  if (i >= plane) return;
  const int k = blockIdx.y;
  const int kh = k / h.Kw, kw = k - kh * h.Kw;
  const int n = i32 / h.C, ci = i32 - n * h.C;  // 32-bit: a 64-bit divide is a subroutine call
  float* src = c.dwf + (int64_t)k * plane + i;
  const float v = *src;
  if (c.zero_dwf) *src = 0.f;
  const int64_t o = (int64_t)n * h.so_n + (int64_t)ci * h.so_c + (int64_t)kh * h.so_h + (int64_t)kw * h.so_w;
  if (c.f32) reinterpret_cast<float*>(c.out)[o] = v;
  else reinterpret_cast<__nv_bfloat16*>(c.out)[o] = __float2bfloat16(v);
}

// Vectorised chain rule for a weight dW_j dense as [n][ci][window outputs]
// (OIHW-like: conv3x3 / strided convolutions, sep_shared's [C_out][C_in][K])
// with at most one other weight, which then uses window loops only (the
// side output, sep_shared's shared [K] weight).  One thread per (n, four
// consecutive ci): the KK window planes of dWf are read as 16-byte vectors,
// all in flight before any use, and the thread's 4 * KKo outputs are one
// contiguous run written with 8- / 16-byte stores (chain_nc / chain_win did
// one ci per thread with serial weight loads and 2-byte strided stores:
// 6.5-30 us per launch on ResNet-18 layers, latency-bound).  Products keep
// chain_nc's multiplication order; the side output reduces per window in
// blocks and the last block combines the block partials in a fixed tree
// (deterministic: the result depends on gridDim only).
template <int KH, int KW, bool OH, bool OW, bool SIDE, bool WRED = false>
__global__ void __launch_bounds__(256) chain_v4_kernel(const __grid_constant__ ChainArgs c,
                                                       const __grid_constant__ ChainNC h) {
  pdl_trigger();
  pdl_wait();
  constexpr int KK = KH * KW;
  const int plane4 = h.N * h.C / 4;  // N * C < 2^31, C % 4 == 0 (host-checked)
  const int other = h.side_j >= 0 ? h.side_j : -1;
  float vs[KK];  // side products per window, summed over the thread's (n, ci) elements
#pragma unroll
  for (int k = 0; k < KK; ++k) vs[k] = 0.f;
  // grid-stride: one block may walk a small problem (SYNO_TC_V4_ONE)
#pragma unroll 1
  for (int i4 = blockIdx.x * blockDim.x + threadIdx.x, it = 0; it == 0 || i4 < plane4;
       i4 += gridDim.x * blockDim.x, ++it) {
    const bool live = i4 < plane4;
    const int q0 = live ? i4 * 4 : 0;  // flat (n, ci) of the thread's first element
    const int n = q0 / h.C, ci = q0 - n * h.C;
    float4 v[KK];
    float wj[KK][4], wo[KK];
    if (live) {
      float4* src = reinterpret_cast<float4*>(c.dwf) + i4;
  #pragma unroll
      for (int k = 0; k < KK; ++k) v[k] = __ldcg(src + (int64_t)k * plane4);
  #pragma unroll
      for (int k = 0; k < KK; ++k) {
        const int kh = k / KW, kw = k - kh * KW;
        wo[k] = 1.f;
        if (other >= 0) {
          // the side weight's value at this window (window loops only)
          const int32_t off = kh * h.sw[other][0] + kw * h.sw[other][1];
          wo[k] = c.f32 ? __ldg(reinterpret_cast<const float*>(c.w[other]) + off)
                        : __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(c.w[other]) + off));
  #pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int32_t offj = kh * h.side_sw[c.j][0] + kw * h.side_sw[c.j][1] + n * h.side_sw[c.j][2] +
                                 (ci + e) * h.side_sw[c.j][3];
            wj[k][e] = c.f32 ? __ldg(reinterpret_cast<const float*>(c.w[c.j]) + offj)
                             : __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(c.w[c.j]) + offj));
          }
        }
      }
      if (c.zero_dwf) {
  #pragma unroll
        for (int k = 0; k < KK; ++k) src[(int64_t)k * plane4] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    // main output: o[e][a] over the weight's window outputs (windows it does not use fold in)
    constexpr int KKo_w = OW ? KW : 1;
    constexpr int KKo = (OH ? KH : 1) * KKo_w;  // the weight's window outputs (compile-time: register arrays)
    float o[4][KKo];
  #pragma unroll
    for (int e = 0; e < 4; ++e)
  #pragma unroll
      for (int a = 0; a < KKo; ++a) o[e][a] = 0.f;
  #pragma unroll
    for (int k = 0; k < KK; ++k) {
      const int kh = k / KW, kw = k - kh * KW;
      const int a = (OH ? kh : 0) * KKo_w + (OW ? kw : 0);
      const float d[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
  #pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (!live) break;
        o[e][a] += other >= 0 ? d[e] * wo[k] : d[e];
        if (other >= 0) vs[k] += d[e] * wj[k][e];
      }
    }
    if (live) {
      // the thread's outputs: 4 * KKo contiguous elements at flat (n, ci) * KKo
      const int64_t base = (int64_t)q0 * KKo;
      if (c.f32) {
        float* ob = reinterpret_cast<float*>(c.out) + base;
  #pragma unroll
        for (int e = 0; e < 4; ++e)
  #pragma unroll
          for (int a = 0; a < KKo; ++a) ob[e * KKo + a] = o[e][a];
      } else {
        // 8 * KKo bytes per thread at an 8-byte aligned offset: 2 * KKo 4-byte words
        uint32_t* ob = reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(c.out) + base);
  #pragma unroll
        for (int t = 0; t < 2 * KKo; ++t) {
          const int i0 = 2 * t, i1 = 2 * t + 1;
          const float f0 = o[i0 / KKo][i0 % KKo];
          const float f1 = o[i1 / KKo][i1 % KKo];
          const __nv_bfloat162 p2 = __floats2bfloat162_rn(f0, f1);
          ob[t] = *reinterpret_cast<const uint32_t*>(&p2);
        }
      }
    }
  }
  if constexpr (SIDE && WRED) {
    // side output without shared memory (a block that needs none can start
    // beside the concurrent grad-input GEMM's CTAs): warp sums per window to
    // global partials, then the last warp to arrive reduces all of them in a
    // fixed order (lane-strided sums + a fixed xor tree: deterministic)
    const int lane = threadIdx.x & 31;
    const unsigned gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // global warp
    const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
#pragma unroll
    for (int k = 0; k < KK; ++k) {
      float t = vs[k];
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) t += __shfl_xor_sync(0xffffffffu, t, s);
      vs[k] = t;
    }
    unsigned prev = 0;
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < KK; ++k) h.partial[(size_t)gw * KK + k] = vs[k];
      __threadfence();
      prev = atomicAdd(h.counter, 1u);
    }
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != nwarps - 1) return;
    __threadfence();
    float tot[KK];
#pragma unroll
    for (int k = 0; k < KK; ++k) tot[k] = 0.f;
    for (unsigned w = lane; w < nwarps; w += 32) {
      float pv[KK];
#pragma unroll
      for (int k = 0; k < KK; ++k) pv[k] = __ldcg(h.partial + (size_t)w * KK + k);
#pragma unroll
      for (int k = 0; k < KK; ++k) tot[k] += pv[k];
    }
#pragma unroll
    for (int k = 0; k < KK; ++k) {
      float t = tot[k];
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) t += __shfl_xor_sync(0xffffffffu, t, s);
      tot[k] = t;
    }
    if (lane == 0) {
      const int ow2 = h.side_ow ? KW : 1;
      const int no = (h.side_oh ? KH : 1) * ow2;
      for (int q = 0; q < no; ++q) {
        const int ah = q / ow2, aw = q - ah * ow2;
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < KK; ++k) {
          const int kh = k / KW, kw = k - kh * KW;
          if ((h.side_oh ? kh : 0) == ah && (h.side_ow ? kw : 0) == aw) acc += tot[k];
        }
        const int64_t off = (int64_t)ah * h.side_so_h + (int64_t)aw * h.side_so_w;
        if (c.f32) reinterpret_cast<float*>(h.side_out)[off] = acc;
        else reinterpret_cast<__nv_bfloat16*>(h.side_out)[off] = __float2bfloat16(acc);
      }
      *h.counter = 0;  // ready for the next call (stream order)
    }
  } else if constexpr (SIDE) {
  if (other < 0) return;
  // side output: block sums per window, then the last block combines
  __shared__ float wsum[8][KK];
  __shared__ float red[KK][256];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < KK; ++k) {
    float t = vs[k];
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) t += __shfl_xor_sync(0xffffffffu, t, s);
    if (lane == 0) wsum[warp][k] = t;
  }
  __syncthreads();
  if (gridDim.x == 1) {
    // one block: its warp sums are the totals (fixed order)
    if (threadIdx.x < KK) {
      float t = 0.f;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += wsum[q][threadIdx.x];
      red[threadIdx.x][0] = t;
    }
    __syncthreads();
  } else {
    if (threadIdx.x < KK) {
      float t = 0.f;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += wsum[q][threadIdx.x];
      h.partial[(size_t)blockIdx.x * KK + threadIdx.x] = t;
      __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(h.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // each thread sums a strided set of the blocks' partials, every window's
    // load of one block in flight together (a loop per window serialised
    // KK L2 round trips: ~6 us of a 64 x 64 layer's chain)
    float tk[KK];
#pragma unroll
    for (int k = 0; k < KK; ++k) tk[k] = 0.f;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
      float pv[KK];
#pragma unroll
      for (int k = 0; k < KK; ++k) pv[k] = __ldcg(h.partial + (size_t)b * KK + k);
#pragma unroll
      for (int k = 0; k < KK; ++k) tk[k] += pv[k];
    }
#pragma unroll
    for (int k = 0; k < KK; ++k) red[k][threadIdx.x] = tk[k];
    __syncthreads();
    for (int width = (int)blockDim.x >> 1; width > 0; width >>= 1) {
      if ((int)threadIdx.x < width) {
#pragma unroll
        for (int k = 0; k < KK; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + width];
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    const int ow2 = h.side_ow ? KW : 1;
    const int no = (h.side_oh ? KH : 1) * ow2;
    float acc[KK];
    for (int q = 0; q < no; ++q) acc[q] = 0.f;
    for (int k = 0; k < KK; ++k) {
      const int kh = k / KW, kw = k - kh * KW;
      acc[(h.side_oh ? kh : 0) * ow2 + (h.side_ow ? kw : 0)] += red[k][0];
    }
    for (int q = 0; q < no; ++q) {
      const int ah = q / ow2, aw = q - ah * ow2;
      const int64_t off = (int64_t)ah * h.side_so_h + (int64_t)aw * h.side_so_w;
      if (c.f32) reinterpret_cast<float*>(h.side_out)[off] = acc[q];
      else reinterpret_cast<__nv_bfloat16*>(h.side_out)[off] = __float2bfloat16(acc[q]);
    }
    if (gridDim.x > 1) *h.counter = 0;  // ready for the next call (stream order)
  }
  }  // SIDE: no shared memory in the single-weight instances
}

// Single weight, single window, dense [N][C] gradient (QKV-like): dW = dWf
// cast, dWf re-zeroed; four elements per thread with 16-byte accesses.
__global__ void __launch_bounds__(256) chain_cast_kernel(float* __restrict__ dwf, void* __restrict__ out, int64_t n,
                                                         int f32, int zero) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    const float4 v = *reinterpret_cast<const float4*>(dwf + i);
    if (zero) *reinterpret_cast<float4*>(dwf + i) = make_float4(0.f, 0.f, 0.f, 0.f);
    if (f32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + i) = v;
    } else {
      __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(out) + i);
      o[0] = __floats2bfloat162_rn(v.x, v.y);
      o[1] = __floats2bfloat162_rn(v.z, v.w);
    }
  } else {
    for (int64_t k = i; k < n; ++k) {
      const float v = dwf[k];
      if (zero) dwf[k] = 0.f;
      if (f32) reinterpret_cast<float*>(out)[k] = v;
      else reinterpret_cast<__nv_bfloat16*>(out)[k] = __float2bfloat16(v);
    }
  }
}

// Long reductions: block (o, split) reduces one chunk; the last block of an
// output sums the partials in split order (deterministic) and stores.
__global__ void __launch_bounds__(256) chain_block_kernel(const __grid_constant__ ChainArgs c) {
  pdl_trigger();
  pdl_wait();
  const int64_t o = blockIdx.x;
  const int nsplit = gridDim.y;
  const int64_t r0 = (int64_t)blockIdx.y * c.r_chunk;
  const int64_t r1 = min(c.R, r0 + c.r_chunk);
  int d[4];
  float acc = 0.f;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    chain_decode(c, o, r, d);
    acc += chain_term(c, d);
    if (c.zero_dwf) c.dwf[((int64_t)(d[0] * c.ext[1] + d[1]) * c.ext[2] + d[2]) * c.ext[3] + d[3]] = 0.f;
  }
#pragma unroll
  for (int k = 16; k > 0; k >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, k);
  __shared__ float part[8];
  __shared__ bool last;
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += part[k];
    c.partial[o * nsplit + blockIdx.y] = t;
    __threadfence();
    last = atomicAdd(c.counter + o, 1u) == (unsigned)nsplit - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    float t = 0.f;
    for (int k = 0; k < nsplit; ++k) t += *((volatile float*)c.partial + o * nsplit + k);
    chain_decode(c, o, 0, d);
    chain_store(c, d, t);
    c.counter[o] = 0;  // ready for the next call (stream order)
  }
}

// ---------------------------------------------------------------------------
// Plan
// ---------------------------------------------------------------------------

struct PixDim {
  int axis = -1;       // stage loop (output axis)
  int win = -1;        // window reduce loop, -1 none
  int S = 1, K = 1;
  int64_t c = 0;       // offset constant
  int64_t E = 1;       // output extent
  int64_t Ein = 1;     // input extent
  int64_t xs = 0, ys = 0;  // element strides of the coordinate in x and y
  int lo = 0, hi = 0;  // forward padding of the phase planes
  int dlo = 0, dhi = 0;  // grad-input padding of dy
  bool share = false;   // pad rows may be shared between neighbours (all pads read zero)
  // Padded extent of the flat grid.  When every out-of-footprint read is a
  // zero (x has exactly S*E rows), the trailing pad of one row / image is
  // the leading pad of the next, so max(lo, hi) pad rows suffice instead of
  // lo + hi (a 4x4 map: 25 instead of 36 rows per image).
  int64_t Ep() const { return E + (share ? std::max(lo, hi) : lo + hi); }
  int64_t dEp() const { return E + std::max(dlo, dhi); }
  int delta(int r) const { return (int)std::floor((double)(r - c) / S); }
  int phi(int r) const { return (int)(((r - c) % S + S) % S); }
};

struct TcPlan {
  int n_img = 1;
  int64_t x_img = 0, y_img = 0;   // element strides of the flattened image index
  int64_t x_c = 0, y_n = 0;       // channel / output-channel strides
  int C = 0, N = 0, Cp = 0, Np = 0;
  PixDim dh, dw;
  double scale = 1;
  double flops = 0;  // algorithmic FLOPs of one GEMM (= codegen.flops(staged=True), batch included)
  bool dgrad_ok = false;
  DevStage fold_fwd, fold_dgrad;
  std::vector<DevStage> chain;    // dW_j from the folded gradient
  std::vector<int64_t> w_numel;
  // Direct weight transforms: every weight coordinate is a bare fold loop
  // (rh, rw, n, ci) with the loop's full extent and there are no weight-only
  // reduces, so a weight offset is affine in the fold loops.
  bool fast_fold = false;
  int nw = 0;
  int64_t wstr[MAXFW][4] = {};  // element strides of w_j along (rh, rw, n, ci)
  std::mutex mu;                  // guards ws
  std::map<std::tuple<int, void*, int>, std::unique_ptr<struct TcWs>> ws;  // per (device, stream, dtype)
  int nwin() const { return dh.K * dw.K; }
  int64_t y_numel() const { return (int64_t)n_img * dh.E * dw.E * N; }
  int64_t x_numel() const { return (int64_t)n_img * dh.Ein * dw.Ein * C; }
};

static std::vector<int64_t> rm_strides(const std::vector<int64_t>& ext) {
  std::vector<int64_t> s(ext.size(), 1);
  for (int k = (int)ext.size() - 2; k >= 0; --k) s[k] = s[k + 1] * ext[k + 1];
  return s;
}

// S*i + r - c  /  i + r - c  (unfold over a [strided] data dim)
static bool match_window(const CE& e, int A, int* axis, int* red, int* S, int64_t* c) {
  if (e->op != COp::Sub || e->rhs->op != COp::Const) return false;
  const CE& add = e->lhs;
  if (add->op != COp::Add || add->rhs->op != COp::Loop || add->rhs->loop < A) return false;
  const CE& data = add->lhs;
  if (data->op == COp::Loop && data->loop < A) {
    *S = 1;
    *axis = data->loop;
  } else if (data->op == COp::Mul && data->lhs->op == COp::Const && data->rhs->op == COp::Loop &&
             data->rhs->loop < A) {
    *S = (int)data->lhs->value;
    *axis = data->rhs->loop;
  } else {
    return false;
  }
  *red = add->rhs->loop;
  *c = e->rhs->value;
  return *S >= 1;
}

static TcPlan* try_match(const Plan& plan) {
  const CStage& S = plan.unstaged;
  const int A = (int)S.axis_ext.size();
  const int L = S.nloops();
  if (S.terms.empty() || S.terms[0].t.kind != TK_X || S.terms.size() < 2) return nullptr;
  const CTerm& x = S.terms[0];
  for (size_t t = 1; t < S.terms.size(); ++t)
    if (S.terms[t].t.kind != TK_W) return nullptr;
  auto xs = rm_strides(x.t.extents);
  auto ys = rm_strides(S.axis_ext);  // y is row-major over the stage axes
  int chan = -1, chan_coord = -1;
  std::vector<PixDim> pix;
  std::set<int> used_axes, used_red;
  for (size_t d = 0; d < x.coords.size(); ++d) {
    const CE& e = x.coords[d];
    PixDim p;
    if (e->op == COp::Loop) {
      if (e->loop >= A) {
        if (chan >= 0) return nullptr;
        chan = e->loop;
        chan_coord = (int)d;
        if (x.t.extents[d] != S.ext(chan)) return nullptr;
        continue;
      }
      p.axis = e->loop;
      p.E = S.ext(p.axis);
      p.Ein = x.t.extents[d];
      if (p.Ein != p.E) return nullptr;
    } else {
      int axis, red, st;
      int64_t c;
      if (!match_window(e, A, &axis, &red, &st, &c)) return nullptr;
      p.axis = axis;
      p.win = red;
      p.S = st;
      p.K = (int)S.ext(red);
      p.c = c;
      p.E = S.ext(axis);
      p.Ein = x.t.extents[d];
      if (!used_red.insert(red).second) return nullptr;
    }
    if (!used_axes.insert(p.axis).second) return nullptr;
    p.xs = xs[d];
    p.ys = ys[p.axis];
    pix.push_back(p);
  }
  if (chan < 0) return nullptr;
  used_red.insert(chan);
  // exactly one axis is read only by weights
  int naxis = -1;
  for (int a = 0; a < A; ++a)
    if (!used_axes.count(a)) {
      if (naxis >= 0) return nullptr;
      naxis = a;
    }
  if (naxis < 0) return nullptr;
  // weights: bare loops only
  bool n_in_w = false;
  for (size_t t = 1; t < S.terms.size(); ++t)
    for (auto& e : S.terms[t].coords) {
      if (e->op != COp::Loop) return nullptr;
      if (e->loop == naxis) n_in_w = true;
      if (e->loop < A && e->loop != naxis) return nullptr;
    }
  if (!n_in_w) return nullptr;
  // image dims: all pixel dims but the last two, window-free and row-major-contiguous
  auto tp = std::make_unique<TcPlan>();
  while (pix.size() < 2) pix.insert(pix.begin(), PixDim());  // unit dims
  const size_t nimg = pix.size() - 2;
  for (size_t k = 0; k < nimg; ++k) {
    if (pix[k].win >= 0) return nullptr;
    if (k + 1 < nimg && (pix[k].xs != pix[k + 1].xs * pix[k + 1].E || pix[k].ys != pix[k + 1].ys * pix[k + 1].E))
      return nullptr;
  }
  tp->n_img = 1;
  for (size_t k = 0; k < nimg; ++k) tp->n_img *= (int)pix[k].E;
  tp->x_img = nimg ? pix[nimg - 1].xs : 0;
  tp->y_img = nimg ? pix[nimg - 1].ys : 0;
  tp->dh = pix[nimg];
  tp->dw = pix[nimg + 1];
  tp->x_c = xs[chan_coord];
  tp->y_n = ys[naxis];
  tp->C = (int)S.ext(chan);
  tp->N = (int)S.ext(naxis);
  tp->Cp = (tp->C + 7) / 8 * 8;
  {
    // narrow inputs (a 3-channel stem) padded to a whole 64-channel block:
    // full 128-byte rows keep the TMA loads of the forward / grad-weight A
    // operands efficient (8-channel rows with 112 bytes of out-of-bounds fill
    // each made the stem's GEMMs the slowest of the step: ResNet-18 step
    // 1.451 -> 1.413 ms, stem fwd 32 -> 19 us, grad-weight 49 -> 21 us);
    // the MMA K steps stop at the real channels (kq_last): no extra MMAs
    static const int cp_min = getenv("SYNO_TC_CP_MIN") ? atoi(getenv("SYNO_TC_CP_MIN")) : 64;  // A/B: 0 = off
    if (tp->C < cp_min) tp->Cp = (cp_min + 7) / 8 * 8;
  }
  tp->Np = (tp->N + 7) / 8 * 8;
  tp->scale = S.scale;
  for (PixDim* p : {&tp->dh, &tp->dw}) {
    int dmin = 0, dmax = 0;
    for (int r = 0; r < p->K; ++r) {
      dmin = std::min(dmin, p->delta(r));
      dmax = std::max(dmax, p->delta(r));
    }
    p->lo = -dmin;
    p->hi = dmax;
    // grad-input reads dy at u - delta(r)
    p->dlo = dmax;
    p->dhi = -dmin;
    p->share = p->Ein <= (int64_t)p->S * p->E;
    if (p->S > 2 || p->E * p->S < 1) return nullptr;
  }
  if (tp->nwin() > MAXWIN) return nullptr;
  if (tp->dh.S * tp->dw.S > 8) return nullptr;
  tp->dgrad_ok = tp->dh.Ein == (int64_t)tp->dh.S * tp->dh.E && tp->dw.Ein == (int64_t)tp->dw.S * tp->dw.E;
  // loop ids of the fold stages: rh, rw, then two channel axes, then weight-only reduces
  std::vector<int> wonly;
  for (int l = A; l < L; ++l)
    if (!used_red.count(l)) wonly.push_back(l);
  (void)wonly;
  return tp.release();
}

// Fold stage: Wf[rh][rw][a][b] = sum_{weight-only reduces} prod_j w_j, with (a, b) = (n, ci)
// for the forward operand and (ci, n) for the grad-input operand.  Channel extents
// are padded (the weight's own range check zero-fills the pad).
static CStage fold_stage(const Plan& plan, const TcPlan& tp, bool dgrad, bool padded) {
  const CStage& S = plan.unstaged;
  const int A = (int)S.axis_ext.size();
  int naxis = -1, chan = -1;
  for (int a = 0; a < A; ++a) {
    bool in_x = false;
    for (auto& e : S.terms[0].coords) {
      std::vector<int> ls;
      c_loops(e, &ls);
      in_x = in_x || std::count(ls.begin(), ls.end(), a);
    }
    if (!in_x) naxis = a;
  }
  for (auto& e : S.terms[0].coords)
    if (e->op == COp::Loop && e->loop >= A) chan = e->loop;
  std::map<int, int> m;
  CStage f;
  f.axis_ext = {tp.dh.K, tp.dw.K};
  if (tp.dh.win >= 0) m[tp.dh.win] = 0;
  if (tp.dw.win >= 0) m[tp.dw.win] = 1;
  if (!dgrad) {
    m[naxis] = 2;
    m[chan] = 3;
    f.axis_ext.push_back(tp.N);
    f.axis_ext.push_back(padded ? tp.Cp : tp.C);
  } else {
    m[chan] = 2;
    m[naxis] = 3;
    f.axis_ext.push_back(tp.C);
    f.axis_ext.push_back(padded ? tp.Np : tp.N);
  }
  for (int l = A; l < S.nloops(); ++l)
    if (!m.count(l)) {
      m[l] = 4 + (int)f.red_ext.size();
      f.red_ext.push_back(S.ext(l));
    }
  std::function<CE(const CE&)> rn = [&](const CE& e) -> CE {
    if (e->op == COp::Loop) return c_loop(m.at(e->loop));
    if (e->op == COp::Const) return e;
    return c_bin(e->op, rn(e->lhs), rn(e->rhs));
  };
  for (size_t t = 1; t < S.terms.size(); ++t) {
    CTerm ct = S.terms[t];
    for (auto& c : ct.coords) c = rn(c);
    f.terms.push_back(ct);
  }
  f.out.kind = TK_STAGE;
  f.out.index = 0;
  f.out.extents = f.axis_ext;
  return f;
}

bool tc_matches(const Plan& plan) {
  TcPlan* raw = try_match(plan);
  delete raw;
  if (!raw) return false;
  // the chain rule through the fold must invert (bare weight coordinates always do)
  return true;
}

// Fast weight transforms apply when each weight coordinate is a bare fold
// loop (rh, rw, n, ci) of full extent: no weight-only reduces, no range checks.
static void setup_fast_fold(const Plan& plan, TcPlan& tp) {
  const CStage& S = plan.unstaged;
  const int A = (int)S.axis_ext.size();
  int naxis = -1, chan = -1;
  for (int a = 0; a < A; ++a) {
    bool in_x = false;
    for (auto& e : S.terms[0].coords) {
      std::vector<int> ls;
      c_loops(e, &ls);
      in_x = in_x || std::count(ls.begin(), ls.end(), a);
    }
    if (!in_x) naxis = a;
  }
  for (auto& e : S.terms[0].coords)
    if (e->op == COp::Loop && e->loop >= A) chan = e->loop;
  std::map<int, int> slot;
  if (tp.dh.win >= 0) slot[tp.dh.win] = 0;
  if (tp.dw.win >= 0) slot[tp.dw.win] = 1;
  slot[naxis] = 2;
  slot[chan] = 3;
  const int nw = (int)S.terms.size() - 1;
  if (nw < 1 || nw > MAXFW) return;
  for (int j = 0; j < nw; ++j) {
    const CTerm& t = S.terms[j + 1];
    auto st = rm_strides(t.t.extents);
    for (size_t d = 0; d < t.coords.size(); ++d) {
      const CE& e = t.coords[d];
      if (e->op != COp::Loop) return;
      auto it = slot.find(e->loop);
      if (it == slot.end()) return;  // weight-only reduce: the general fold stage handles it
      if (t.t.extents[d] != S.ext(e->loop)) return;
      if (tp.wstr[j][it->second] != 0) return;
      tp.wstr[j][it->second] = st[d];
    }
  }
  tp.nw = nw;
  tp.fast_fold = getenv("SYNO_TC_SLOW_FOLD") == nullptr;
}

TcPlanPtr tc_build(const Plan& plan, cudaStream_t stream) {
  TcPlan* raw = try_match(plan);
  if (!raw) return TcPlanPtr();
  TcPlanPtr tp(raw);
  // algorithmic FLOPs per GEMM = codegen.flops(staged=True):
  // a folded sep_shared GEMM is credited only with the staged volume
  tp->flops = (double)(plan.flops_staged ? plan.flops_staged : plan.flops_unstaged);
  setup_fast_fold(plan, *tp);
  build_dev_stage(fold_stage(plan, *tp, false, true), &tp->fold_fwd, stream);
  if (tp->dgrad_ok) build_dev_stage(fold_stage(plan, *tp, true, true), &tp->fold_dgrad, stream);
  // chain rule through the fold: dW_j from dWf[rh][rw][n][ci] (fp32)
  CStage ref = fold_stage(plan, *tp, false, false);
  for (size_t j = 0; j < plan.w_ext.size(); ++j) {
    CTensor gw;
    gw.kind = TK_DW;
    gw.index = (int)j;
    gw.extents = plan.w_ext[j];
    CStage g = derive_gradient(ref, (int)j, gw);
    if (g.scatter) return TcPlanPtr();
    for (auto& t : g.terms)
      if (t.t.kind == TK_DY) {
        t.t.kind = TK_STAGE;  // dWf is fp32: read in accumulator precision
        t.t.index = 0;
      }
    tp->chain.emplace_back();
    build_dev_stage(g, &tp->chain.back(), stream);
    int64_t n = 1;
    for (auto e : plan.w_ext[j]) n *= e;
    tp->w_numel.push_back(n);
  }
  return tp;
}

std::string tc_describe(const TcPlan* tp) {
  if (!tp) return "tc: none\n";
  std::ostringstream o;
  o << "tc: img=" << tp->n_img << " C=" << tp->C << " N=" << tp->N << " H=" << tp->dh.E << "(S" << tp->dh.S << ",K"
    << tp->dh.K << ",lo" << tp->dh.lo << ",hi" << tp->dh.hi << ") W=" << tp->dw.E << "(S" << tp->dw.S << ",K"
    << tp->dw.K << ",lo" << tp->dw.lo << ",hi" << tp->dw.hi << ") dgrad=" << tp->dgrad_ok << "\n";
  return o.str();
}

// ---------------------------------------------------------------------------
// Launch helpers
// ---------------------------------------------------------------------------

// PDL launch of a GEMM kernel; `pair`: clusters of two CTAs (one TPC) for
// the cta_group::2 configuration.
static void launch_tc(void (*kernel)(TcGemmParams), bool pair, unsigned grid, int smem, cudaStream_t stream,
                      const TcGemmParams& p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = pair ? 2 : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pair ? 2 : 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kernel, p), "cudaLaunchKernelEx(tc_gemm)");
}

template <int BN, int MODE, int CFG>
static void launch_gemm(const TcGemmParams& p, unsigned grid, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};  // per-device bit
  constexpr int smem = smem_bytes<BN, CFG>();
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cuda_check(cudaFuncSetAttribute(tc_gemm_kernel<BN, MODE, CFG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
               "cudaFuncSetAttribute(tc_gemm)");
    configured.fetch_or(bit);
  }
  note_launch();
  // SYNO_TC_TRACE=<file>: append the SM-0 event log of every launch to <file>
  static const char* trace_path = getenv("SYNO_TC_TRACE");
  static unsigned long long* trace_buf = nullptr;
  if (trace_path && !trace_buf) cuda_check(cudaMalloc(&trace_buf, 8192 * sizeof(unsigned long long)), "trace");
  if (!trace_path) {
    launch_tc(tc_gemm_kernel<BN, MODE, CFG>, CFG == CFG_PAIR, grid, smem, stream, p);
  } else {
    TcGemmParams q = p;
    q.trace = trace_buf;
    cuda_check(cudaMemsetAsync(trace_buf, 0, 8192 * sizeof(unsigned long long), stream), "trace memset");
    launch_tc(tc_gemm_kernel<BN, MODE, CFG>, CFG == CFG_PAIR, grid, smem, stream, q);
    std::vector<unsigned long long> h(8192);
    cuda_check(cudaMemcpyAsync(h.data(), trace_buf, 8192 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream),
               "trace copy");
    cuda_check(cudaStreamSynchronize(stream), "trace sync");
    if (FILE* f = fopen(trace_path, "a")) {
      fprintf(f, "launch BN=%d mode=%d cfg=%d tiles=%d grid=%u G=%d\n", BN, p.mode, CFG, p.m_tiles * p.n_tiles * p.z_tiles,
              grid, p.G);
      const unsigned long long nc = std::min<unsigned long long>(h[0], 7);
      for (unsigned long long c = 0; c < nc; ++c)
        for (int i = 0; i < 512; ++i) {
          const unsigned long long t = h[64 + c * 1024 + 2 * i], v = h[64 + c * 1024 + 2 * i + 1];
          if (t) fprintf(f, "%llu %llu %llu %llu %llu\n", t, v & 0xFF, (v >> 8) & 0xFFFF, (v >> 24) & 0xFFFF, v >> 40);
        }
      fclose(f);
    }
  }
  cuda_check(cudaGetLastError(), "tc_gemm_kernel");
}

static int sm_count() {
  int dev = 0, n = 148;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
  return n;
}

static bool tc_log();

// Persistent launch: one CTA per SM walks the (n fastest, m, z) tile grid.
static void gemm(TcGemmParams& p, int bn, int m_tiles, int n_tiles, int z_tiles, cudaStream_t stream,
                 const char* name, double flops) {
  if (skip_class("gemm")) return;
  {
    const int split = p.mode == MODE_ROWS ? std::max(1, p.rsplit) : std::max(1, p.ksplit);
    p.k_per = (p.n_cblocks + split - 1) / split;
    // pair grad-weight stages two K blocks: every split but the last covers an even count
    if (p.mode == MODE_WGRAD && p.cfg == CFG_PAIR) p.k_per += p.k_per & 1;
  }
  if (p.mode == MODE_ROWS && (int64_t)m_tiles * std::max(1, p.G) * BM >= INT32_MAX)
    fail(SYNO_E_UNSUPPORTED, "tc: 2^31 or more rows in one operand plane");
  const bool pair = p.cfg == CFG_PAIR;
  // pair: the kernel's M tiles are pairs of 128-row tiles
  p.m_tiles = pair ? (m_tiles + 1) / 2 : m_tiles;
  p.n_tiles = n_tiles;
  p.z_tiles = z_tiles;
  const bool small = p.cfg == 1 && bn <= 128;
  const int a_region = pair ? (bn == 128 ? a_region_bytes<128, CFG_PAIR>() : a_region_bytes<256, CFG_PAIR>())
                       : small ? (bn == 64 ? a_region_bytes<64, 1>() : a_region_bytes<128, 1>())
                               : (bn == 64 ? a_region_bytes<64>() : bn == 128 ? a_region_bytes<128>() : a_region_bytes<256>());
  const int ring = small ? ring_bytes<1>() : ring_bytes<0>();
  p.a_stages = std::max(1, std::min(8, (p.mode == MODE_ROWS && p.b_res ? ring - p.b_res * bn * BK * 2 : a_region) /
                                           p.a_stage_bytes));
  const int64_t tiles = (int64_t)p.m_tiles * n_tiles * z_tiles;
  if (tiles <= 0) return;
  const unsigned grid = pair ? (unsigned)std::min<int64_t>(tiles, sm_count() / 2) * 2
                             : (unsigned)std::min<int64_t>(tiles, (int64_t)sm_count() * (small ? 2 : 1));
  if (tc_log())
    fprintf(stderr, "[tc] gemm %s bn=%d cfg=%d tiles=%lld grid=%u G=%d rsplit=%d a_stages=%d\n", name, bn, p.cfg,
            (long long)tiles, grid, p.G, p.rsplit, p.a_stages);
  const int id = prof_begin(name, flops, 0.0, stream);
  if (p.mode == MODE_ROWS) {
    if (pair) {
      if (bn == 128) launch_gemm<128, MODE_ROWS, CFG_PAIR>(p, grid, stream);
      else launch_gemm<256, MODE_ROWS, CFG_PAIR>(p, grid, stream);
    } else if (small) {
      if (bn == 64) launch_gemm<64, MODE_ROWS, 1>(p, grid, stream);
      else launch_gemm<128, MODE_ROWS, 1>(p, grid, stream);
    } else if (bn == 64) launch_gemm<64, MODE_ROWS, 0>(p, grid, stream);
    else if (bn == 128) launch_gemm<128, MODE_ROWS, 0>(p, grid, stream);
    else launch_gemm<256, MODE_ROWS, 0>(p, grid, stream);
  } else {
    if (small) {
      if (bn == 64) launch_gemm<64, MODE_WGRAD, 1>(p, grid, stream);
      else launch_gemm<128, MODE_WGRAD, 1>(p, grid, stream);
    } else if (pair) {
      launch_gemm<256, MODE_WGRAD, CFG_PAIR>(p, grid, stream);
    } else if (bn == 64) launch_gemm<64, MODE_WGRAD, 0>(p, grid, stream);
    else if (bn == 128) launch_gemm<128, MODE_WGRAD, 0>(p, grid, stream);
    else launch_gemm<256, MODE_WGRAD, 0>(p, grid, stream);
  }
  prof_end(id, stream);
}

static int mgroup_of(int bn) { return bn == 64 ? mgroup<64>() : bn == 128 ? mgroup<128>() : mgroup<256>(); }

// MODE_ROWS work split for small problems: fewer M tiles per step (G) and
// then a split of the channel blocks across CTAs (fp32 atomic output), until
// the persistent grid has at least one tile per SM.
struct RowsTiling {
  int G, rs;
  int64_t m_tiles;
};

// Two-CTA-per-SM configuration for BN <= 128 (SYNO_TC_SMALL=0 disables).
static bool use_small_cfg(int bn) {
  static const bool on = !(getenv("SYNO_TC_SMALL") && atoi(getenv("SYNO_TC_SMALL")) == 0);
  return on && bn <= 128;
}

// Resident B (TcGemmParams::b_res) when the whole weight operand of the
// launch (one N tile, one channel block) fits beside one A stage.
static void set_b_res(TcGemmParams& p, int bn, int n_tiles) {
  static const bool off = getenv("SYNO_TC_NO_BRES") != nullptr;
  p.b_res = 0;
  if (off || n_tiles != 1 || p.n_cblocks != 1 || p.rsplit > 1) return;
  const int ring = (p.cfg == 1 && bn <= 128) ? ring_bytes<1>() : ring_bytes<0>();
  if (p.n_win * bn * BK * 2 + p.a_stage_bytes <= ring) p.b_res = p.n_win;
}

// CTA-pair configuration (CFG_PAIR, SYNO_TC_PAIR=0 disables): BN = 256
// launches without a channel split or resident B and with two or more M
// tiles.  Returns the B box rows of one CTA.
static int set_pair(TcGemmParams& p, int bn, const RowsTiling& rt) {
  static const bool on = !(getenv("SYNO_TC_PAIR") && atoi(getenv("SYNO_TC_PAIR")) == 0);
  // BN = 128 in CTA pairs (M = 256 x N = 128 per MMA, 64 B rows per CTA):
  // experiment switch SYNO_TC_PAIR128=1
  static const bool on128 = getenv("SYNO_TC_PAIR128") && atoi(getenv("SYNO_TC_PAIR128")) == 1;
  if (!on || !(bn == 256 || (bn == 128 && on128)) || rt.G != 1 || rt.rs != 1 || p.b_res || rt.m_tiles < 2)
    return bn;
  p.cfg = CFG_PAIR;
  p.b_tx = (uint32_t)(bn / 2) * BK * 2;
  return bn / 2;
}

static RowsTiling rows_tiling(int64_t F, int n_tiles, int groups, int bn, int n_cblocks, int nwin) {
  // Cost model (measured on B200, profiles/r01_gemm_trace_dbg.txt): a
  // 128 x BN x 16 MMA from shared memory takes ~80 cycles for BN <= 128 and
  // ~160 for BN = 256; the epilogue of a 128-row sub-tile costs about as
  // much as 16 such MMAs (more with split-K atomics).  A CTA's time is the
  // number of waves times one tile; pick the (G, split) with the least.
  const bool small = use_small_cfg(bn);
  const int sms = sm_count() * (small ? 2 : 1);
  const int gm = small ? 1 : mgroup_of(bn);
  auto mt = [&](int g) { return (F + (int64_t)g * BM - 1) / ((int64_t)g * BM); };
  const double mma = bn >= 256 ? 2.0 : 1.0;
  const bool no_split = getenv("SYNO_TC_NO_RSPLIT") != nullptr;
  RowsTiling best{gm, 1, mt(gm)};
  double best_cost = 1e300;
  static const int force_g = getenv("SYNO_TC_G") ? atoi(getenv("SYNO_TC_G")) : 0;  // experiments
  for (int G = gm; G >= 1; G /= 2) {
    if (force_g && G != force_g && force_g <= gm) continue;
    for (int rs = 1; rs <= (no_split ? 1 : n_cblocks); ++rs) {
      const int per = (n_cblocks + rs - 1) / rs;
      if (rs > 1 && (n_cblocks + per - 1) / per != rs) continue;  // an empty split: same as fewer splits
      const int64_t tiles = mt(G) * n_tiles * groups * rs;
      const int64_t waves = (tiles + sms - 1) / sms;
      const double tile = G * (nwin * per * 4.0 * mma + 16.0 * mma * (rs > 1 ? 2.0 : 1.0));
      const double cost = waves * tile + (rs > 1 ? 8.0 * mma : 0.0);  // + the cast / zero fill
      if (cost < best_cost * 0.98) {
        best_cost = cost;
        best = {G, rs, mt(G)};
      }
    }
  }
  return best;
}

// Split-K accumulator -> bf16 output; the accumulator is left zeroed for
// the next call (it starts zeroed), so no memset precedes the GEMM.
__global__ void cast_f32_bf16_kernel(float* __restrict__ in, __nv_bfloat16* __restrict__ out, int64_t n) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    const float4 v = *reinterpret_cast<const float4*>(in + i);
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    *reinterpret_cast<__nv_bfloat162*>(out + i) = a;
    *reinterpret_cast<__nv_bfloat162*>(out + i + 2) = b;
    *reinterpret_cast<float4*>(in + i) = make_float4(0.f, 0.f, 0.f, 0.f);
  } else {
    for (int64_t k = i; k < n; ++k) {
      out[k] = __float2bfloat16(in[k]);
      in[k] = 0.f;
    }
  }
}

static void cast_to_bf16(float* in, void* out, int64_t n, cudaStream_t stream) {
  if (skip_class("cast")) return;
  const int id = prof_begin("cast_f32_bf16", 0.0, (double)n * 10, stream);
  note_launch();
  launch_k(cast_f32_bf16_kernel, (unsigned)((n / 4 + 256) / 256), 256, 0, stream, in, static_cast<__nv_bfloat16*>(out), n);
  cuda_check(cudaGetLastError(), "cast_f32_bf16_kernel");
  prof_end(id, stream);
}

static int pick_bn(int n, int64_t m_rows = -1) {
  // BN = 128 costs the same cycles per 128x128x16 as BN = 256 does per half of
  // its tile (shared-memory bound), and it allows two CTAs per SM
  static const int cap = getenv("SYNO_TC_MAXBN") ? atoi(getenv("SYNO_TC_MAXBN")) : 256;
  int bn = n <= 64 ? 64 : n <= 128 ? 128 : 256;
  // a row GEMM whose 256-wide tiles would not cover the SMs once (ResNet-18's
  // 8 x 8 and 4 x 4 maps: 50-81 tiles) takes 128-wide tiles, twice as many:
  // forward / grad-input 1.368 -> 1.356 ms on the ResNet-18 step
  // (profiles/r02_tiling.txt); SYNO_TC_BN_FILL=0 disables
  static const bool fill = !(getenv("SYNO_TC_BN_FILL") && atoi(getenv("SYNO_TC_BN_FILL")) == 0);
  static const int fill_waves = getenv("SYNO_TC_BN_FILL_WAVES") ? atoi(getenv("SYNO_TC_BN_FILL_WAVES")) : 1;
  if (fill && bn == 256 && m_rows >= 0 && (m_rows + BM - 1) / BM * ((n + 255) / 256) < fill_waves * sm_count())
    bn = 128;
  return std::min(bn, std::max(64, cap));
}

template <typename TI, int V>
static void launch_pack_rows(const void* src, const PackGeom& g, __nv_bfloat16* dst, dim3 grid, int rpb,
                             int64_t rows, cudaStream_t stream) {
  launch_k(pack_rows_kernel<TI, V>, grid, 256, 0, stream, static_cast<const TI*>(src), dst, g, rpb, rows);
}

// Launch geometry of a pack and its vector width (0: scalar).
struct PackPlan {
  dim3 grid;
  int rpb = 1;
  int64_t rows = 0;
  int V = 1;
  int flat = 0;  // PackGeom::flat blocks
};

static PackPlan pack_plan(const void* src, DType dt, const PackGeom& g) {
  PackPlan pp;
  pp.rpb = std::max(1, PK_PIX / g.Win);
  pp.rows = (int64_t)g.n_img_out() * g.Hin;
  const int64_t blocks = g.Win <= PK_PIX ? (pp.rows + pp.rpb - 1) / pp.rpb : pp.rows * ((g.Win + PK_PIX - 1) / PK_PIX);
  pp.grid = dim3((unsigned)blocks, (unsigned)((g.Ct() + 63) / 64));
  const uintptr_t base = reinterpret_cast<uintptr_t>(src);
  auto aligned = [&](int v, int es) {
    return g.s_w == 1 && g.Win % v == 0 && (g.Win <= PK_PIX || PK_PIX % v == 0) && g.s_h % v == 0 &&
           g.s_c % v == 0 && g.s_img % v == 0 && base % (v * es) == 0;
  };
  if (dt == DT_BF16) pp.V = aligned(8, 2) ? 8 : aligned(4, 2) ? 4 : 1;
  else pp.V = aligned(4, 4) ? 4 : 1;
  // flat pixel blocks when rows are contiguous and the row width defeats the
  // vector loads (SYNO_TC_NO_FLAT_PACK=1: row blocks, A/B switch)
  static const bool no_flat = getenv("SYNO_TC_NO_FLAT_PACK") != nullptr;
  const int64_t HW = (int64_t)g.Hin * g.Win;
  auto flat_ok = [&](int v, int es) {
    return g.split == SPLIT_NONE && g.s_w == 1 && g.s_h == g.Win && HW % v == 0 && g.s_c % v == 0 &&
           g.s_img % v == 0 && base % (v * es) == 0;
  };
  const int vmax = dt == DT_BF16 ? 8 : 4, es = dt == DT_BF16 ? 2 : 4;
  int vf = 0;
  for (int v = vmax; v >= 4 && !vf; v /= 2)
    if (flat_ok(v, es)) vf = v;
  if (!no_flat && vf > pp.V) {
    pp.V = vf;
    pp.flat = 1;
    pp.rows = 0;
    pp.grid = dim3((unsigned)(((int64_t)g.n_img_out() * HW + PK_PIX - 1) / PK_PIX), (unsigned)((g.Ct() + 63) / 64));
  }
  // plane blocks: planes of <= PK_PIX pixels whose rows defeat both vector forms
  const int ve = 16 / es;
  const int tail = g.C % 64;
  if (!no_flat && pp.V == 1 && g.split == SPLIT_NONE && HW <= PK_PIX && g.s_w == 1 && g.s_h == g.Win &&
      g.s_c == HW && g.s_img % ve == 0 && (64 * HW) % ve == 0 && (tail * HW) % ve == 0 && base % 16 == 0) {
    pp.flat = 2;
    pp.V = 1;
    pp.rows = 0;
    pp.grid = dim3((unsigned)g.n_img_out(), (unsigned)((g.Ct() + 63) / 64));
  }
  return pp;
}

static double pack_bytes(DType dt, const PackGeom& g) {
  const double src_elems = (double)g.n_img_out() * g.C * g.Hin * g.Win;
  return src_elems * (dt == DT_BF16 ? 2 : 4) + src_elems * (g.split == SPLIT_CH ? 3 : 1) * 2;
}

static bool tc_log() {
  static const bool on = getenv("SYNO_TC_LOG") != nullptr;
  return on;
}

static void log_pack(const char* what, const void* src, const PackGeom& g) {
  if (tc_log())
    fprintf(stderr, "[tc] %s src=%p C=%d in=%dx%d S=%dx%d lo=%d,%d grid=%dx%d split=%d imgs=%d\n", what, src, g.C, g.Hin,
            g.Win, g.Sh, g.Sw, g.lo_h, g.lo_w, g.Hp, g.Wp, g.split, g.n_img);
}

static void pack_cl(const void* src, DType dt, const PackGeom& g, __nv_bfloat16* dst, cudaStream_t stream) {
  if (skip_class("pack")) return;
  log_pack("pack", src, g);
  // one block = whole source rows (<= PK_PIX pixels), one PK_PIX segment of a
  // wider row, or PK_PIX consecutive pixels of contiguous rows (flat)
  const PackPlan pp = pack_plan(src, dt, g);
  PackGeom gf = g;
  gf.flat = pp.flat;
  const int rpb = pp.rpb;
  const int64_t rows = pp.rows;
  const dim3 grid = pp.grid;
  const double src_elems = (double)g.n_img_out() * g.C * g.Hin * g.Win;
  const int id = prof_begin("pack_cl", 0.0, src_elems * (dt == DT_BF16 ? 2 : 4) * (g.split == SPLIT_CH ? 1 : 1) +
                                                src_elems * (g.split == SPLIT_CH ? 3 : 1) * 2, stream);
  note_launch();
  if (dt == DT_BF16) {
    if (pp.V == 8) launch_pack_rows<__nv_bfloat16, 8>(src, gf, dst, grid, rpb, rows, stream);
    else if (pp.V == 4) launch_pack_rows<__nv_bfloat16, 4>(src, gf, dst, grid, rpb, rows, stream);
    else launch_pack_rows<__nv_bfloat16, 1>(src, gf, dst, grid, rpb, rows, stream);
  } else {
    if (pp.V == 4) launch_pack_rows<float, 4>(src, gf, dst, grid, rpb, rows, stream);
    else launch_pack_rows<float, 1>(src, gf, dst, grid, rpb, rows, stream);
  }
  cuda_check(cudaGetLastError(), "pack_rows_kernel");
  prof_end(id, stream);
}

static void split_rows(const float* src, __nv_bfloat16* dst, int64_t rows, int Cp, uint32_t lo_mask,
                       cudaStream_t stream) {
  const int64_t total = rows * 3 * (int64_t)Cp;
  const int id = prof_begin("split_weights", 0.0, (double)rows * Cp * 4 + (double)total * 2, stream);
  note_launch();
  launch_k(split_rows_kernel, (unsigned)((total + 255) / 256), 256, 0, stream, src, dst, rows, Cp, lo_mask);
  cuda_check(cudaGetLastError(), "split_rows_kernel");
  prof_end(id, stream);
}

static PackGeom geom(const TcPlan& tp, bool dy_side, bool grad_pad, int split = SPLIT_NONE, uint32_t lo_mask = 0) {
  PackGeom g{};
  g.n_img = tp.n_img;
  g.split = split;
  g.lo_mask = lo_mask;
  if (!dy_side) {
    g.s_img = tp.x_img;
    g.s_c = tp.x_c;
    g.s_h = tp.dh.xs;
    g.s_w = tp.dw.xs;
    g.C = tp.C;
    g.Hin = (int)tp.dh.Ein;
    g.Win = (int)tp.dw.Ein;
    g.Sh = tp.dh.S;
    g.Sw = tp.dw.S;
    g.Cp = tp.Cp;
  } else {
    g.s_img = tp.y_img;
    g.s_c = tp.y_n;
    g.s_h = tp.dh.ys;
    g.s_w = tp.dw.ys;
    g.C = tp.N;
    g.Hin = (int)tp.dh.E;
    g.Win = (int)tp.dw.E;
    g.Sh = g.Sw = 1;
    g.Cp = tp.Np;
  }
  g.lo_h = grad_pad ? tp.dh.dlo : tp.dh.lo;
  g.lo_w = grad_pad ? tp.dw.dlo : tp.dw.lo;
  g.Hp = (int)(grad_pad ? tp.dh.dEp() : tp.dh.Ep());
  g.Wp = (int)(grad_pad ? tp.dw.dEp() : tp.dw.Ep());
  const int64_t F = (int64_t)g.n_img_out() * g.Hp * g.Wp;
  g.Fpitch = (F + 7) / 8 * 8;
  return g;
}

// MODE_ROWS schedule.  Windows of each group are sorted by (plane, row
// shift) and cut into chunks whose shift span fits one TMA box (<= 128 extra
// rows): one A halo tile serves every window of a chunk.
struct Win {
  int shift, plane, bplane;
};

static int base_mode() {
  static int m = [] {
    // measured on B200: the swizzle follows absolute smem address bits, so a
    // row-shifted view needs base offset 0 (mode 1 fails the parity tests)
    const char* e = getenv("SYNO_TC_BASEMODE");
    return e ? atoi(e) : 0;
  }();
  return m;
}

static void rows_schedule(TcGemmParams& p, std::vector<std::vector<Win>> groups, int bn, int G) {
  int n = 0, nc = 0, span = 0;
  if (groups.size() > 8) fail(SYNO_E_UNSUPPORTED, "too many window groups");
  for (size_t g = 0; g < groups.size(); ++g) {
    auto& ws = groups[g];
    std::sort(ws.begin(), ws.end(), [](const Win& a, const Win& b) {
      return a.plane != b.plane ? a.plane < b.plane : a.shift < b.shift;
    });
    p.g_chunk0[g] = nc;
    for (size_t i = 0; i < ws.size(); ++i) {
      const bool fresh = i == 0 || ws[i].plane != ws[i - 1].plane || ws[i].shift - p.chunk_pmin[nc - 1] > 128;
      if (fresh) {
        if (nc >= MAXCHUNK) fail(SYNO_E_UNSUPPORTED, "too many window chunks");
        p.chunk_plane[nc] = ws[i].plane;
        p.chunk_pmin[nc] = ws[i].shift;
        p.chunk_w0[nc] = n;
        ++nc;
      }
      if (n >= MAXWIN) fail(SYNO_E_UNSUPPORTED, "too many windows");
      p.a_shift[n] = ws[i].shift;
      p.b_plane[n] = ws[i].bplane;
      span = std::max(span, ws[i].shift - p.chunk_pmin[nc - 1]);
      ++n;
      p.chunk_w1[nc - 1] = n;
    }
    p.g_chunk1[g] = nc;
    p.g_nwin[g] = (int32_t)ws.size();
  }
  p.n_win = n;
  p.G = G;
  p.a_rows = (G * BM + span + 63) / 64 * 64;
  p.a_tx = (uint32_t)p.a_rows * BK * 2;
  p.a_stage_bytes = (int)p.a_tx;
  p.b_tx = (uint32_t)bn * BK * 2;
  p.base_mode = base_mode();
  p.dbg = getenv("SYNO_TC_DEBUG") ? atoi(getenv("SYNO_TC_DEBUG")) : 0;
}

// Per (device, stream, dtype) workspace of an operator: packed operands,
// folded weights, the fp32 grad-weight accumulator and the fully built GEMM
// parameters (their TMA maps point into the workspace, so they are encoded
// once).  Steady-state calls only launch kernels: no allocation, no host
// synchronisation, CUDA-graph capturable.
//
// bf16: operands are packed once.  fp32: every operand is packed as three
// bf16 parts along the GEMM's contraction dim (channels for fwd / dgrad,
// images for wgrad), A = (hi, hi, lo) and B = (hi, lo, hi), so the same
// tcgen05 kernel accumulates xh*wh + xh*wl + xl*wh in fp32 (see Split).
struct TcWs {
  bool f32 = false;
  __nv_bfloat16 *xcl = nullptr, *xclw = nullptr, *wf = nullptr, *dycl_g = nullptr, *dycl_w = nullptr, *wt = nullptr;
  float *dwf = nullptr, *wf32 = nullptr, *wt32 = nullptr;
  float *ysc = nullptr, *dxsc = nullptr;  // fp32 accumulators of split-K (bf16 outputs)
  float* chain_partial = nullptr;     // fast chain rule, block mode
  unsigned* chain_counter = nullptr;
  int chain_nsplit[MAXFW] = {};       // 0: thread mode
  bool wg_fixup = false;              // grad-weight epilogue writes dW directly (no chain launch)
  // grad-weight runs on a side stream concurrently with grad-input (fork /
  // join by events; graph-capturable), so one GEMM's tail overlaps the other
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // zero-copy operands: a source already in the packed layout (channels-last,
  // unpadded, e.g. QKV activations) is read by TMA in place
  bool x_ident = false, xw_ident = false, dyg_ident = false, dyw_ident = false;
  // the forward B operand IS the weight (one bf16 [N][C] weight, one window,
  // no channel padding, QKV-like): TMA reads it in place, no fold launch
  bool wf_ident = false;
  MapSpec ms_fwd_b;
  // the same weight as the grad-input B operand, read MN-major in place
  bool wt_ident = false;
  MapSpec ms_dg_b_mn;
  const void* packed_x_src = nullptr;  // x whose packed operand xcl currently holds (last forward)
  std::vector<const void*> wt_src;      // weights the grad-input operand wt was folded from (last forward)
  MapSpec ms_fwd_a, ms_dg_a, ms_wg_a, ms_wg_b;
  PackGeom gx{}, gxw{}, gdy_g{}, gdy_w{};
  bool share_dy = false, share_x = false;
  TcGemmParams fwd, dg, wg;
  int bn_fwd = 0, bn_dg = 0, bn_wg = 0;
  int t_fwd[3] = {0, 0, 0}, t_dg[3] = {0, 0, 0}, t_wg[3] = {0, 0, 0};
  std::vector<void*> owned;
  bool pooled = false;  // owned blocks come from the stream-ordered pool (cudaMallocAsync)
  ~TcWs() {
    if (pooled && !owned.empty()) {
      // every use of a workspace is ordered on the stream it was built for
      // (and its joined side stream); after a device-wide wait the blocks go
      // back to the pool, which keeps them mapped for the next operator
      cudaDeviceSynchronize();
      for (void* q : owned) cudaFreeAsync(q, 0);
    } else {
      for (void* q : owned) cudaFree(q);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
  }
};

void TcPlanDeleter::operator()(TcPlan* p) const {
  if (!p) return;
  release_dev_stage(p->fold_fwd);
  release_dev_stage(p->fold_dgrad);
  for (auto& s : p->chain) release_dev_stage(s);
  delete p;
}

static bool same_grid(const PackGeom& a, const PackGeom& b) {
  return a.lo_h == b.lo_h && a.lo_w == b.lo_w && a.Hp == b.Hp && a.Wp == b.Wp && a.split == b.split &&
         (a.split == SPLIT_NONE || a.lo_mask == b.lo_mask);
}

// The stream a workspace is being built for (workspace() sets it): the zero
// fills are ordered on it, ahead of the caller's first kernel.
static thread_local cudaStream_t g_ws_stream = nullptr;

// Workspaces come from the device's stream-ordered pool (kept mapped by its
// release threshold, engine.cu build_dev_plan): a fresh operator -- every
// candidate of a sweep -- then costs no driver-level allocation, where
// cudaMalloc mapped new memory with the device idle behind the host.
// SYNO_TC_SYNC_ALLOC=1 restores cudaMalloc (A/B switch).
template <typename T>
static T* ws_alloc(TcWs& w, size_t count) {
  static const bool sync_alloc = getenv("SYNO_TC_SYNC_ALLOC") != nullptr;
  void* p = nullptr;
  const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  if (sync_alloc) {
    cuda_check(cudaMalloc(&p, bytes), "cudaMalloc(tc workspace)");
  } else {
    cuda_check(cudaMallocAsync(&p, bytes, g_ws_stream), "cudaMallocAsync(tc workspace)");
    w.pooled = true;
  }
  w.owned.push_back(p);
  // packed operands rely on this: their padding is written once, here
  cuda_check(cudaMemsetAsync(p, 0, std::max<size_t>(count, 1) * sizeof(T), g_ws_stream), "cudaMemset(tc workspace)");
  return static_cast<T*>(p);
}

// The packed layout of g equals the source's own memory layout.
static bool pack_identity(const PackGeom& g, DType dt) {
  return dt == DT_BF16 && g.split == SPLIT_NONE && g.Sh == 1 && g.Sw == 1 && g.lo_h == 0 && g.lo_w == 0 &&
         g.Hp == g.Hin && g.Wp == g.Win && g.Cp == g.C && g.s_c == 1 && g.s_w == g.C &&
         g.s_h == (int64_t)g.Win * g.C && (g.n_img == 1 || g.s_img == (int64_t)g.Hin * g.Win * g.C) &&
         getenv("SYNO_TC_NO_ZEROCOPY") == nullptr;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

constexpr uint32_t LO_A = 0b100;  // A parts (hi, hi, lo)
constexpr uint32_t LO_B = 0b010;  // B parts (hi, lo, hi)

static void build_ws(TcPlan& tp, TcWs& w, DType dt) {
  w.f32 = dt == DT_F32;
  const int chs = w.f32 ? SPLIT_CH : SPLIT_NONE;
  w.gx = geom(tp, false, false, chs, LO_A);
  const int planes = w.gx.Sh * w.gx.Sw;
  const int64_t F = (int64_t)w.gx.n_img * w.gx.Hp * w.gx.Wp;
  const int Ck = w.gx.Ct();  // contraction channels of the forward A / B operands
  w.xcl = ws_alloc<__nv_bfloat16>(w, (size_t)planes * F * Ck);
  w.wf = ws_alloc<__nv_bfloat16>(w, (size_t)tp.nwin() * tp.N * Ck);
  if (w.f32) w.wf32 = ws_alloc<float>(w, (size_t)tp.nwin() * tp.N * tp.Cp);

  // ---- forward: y = sum_win sum_ci Xcl[plane][flat + shift] Wf[win][n][ci]
  {
    const int bn = pick_bn(tp.N, F);
    TcGemmParams& p = w.fwd;
    memset(&p, 0, sizeof(p));
    p.mode = MODE_ROWS;
    p.n_cblocks = (Ck + BK - 1) / BK;
    // 16-wide MMA K steps of the last channel block (bf16: up to the real channels; the padding is zero)
    p.kq_last = ((w.f32 ? Ck : std::min(Ck, tp.C)) - (p.n_cblocks - 1) * BK + 15) / 16;
    std::vector<std::vector<Win>> groups(1);
    for (int rh = 0; rh < tp.dh.K; ++rh)
      for (int rw = 0; rw < tp.dw.K; ++rw)
        groups[0].push_back({tp.dh.delta(rh) * w.gx.Wp + tp.dw.delta(rw), tp.dh.phi(rh) * w.gx.Sw + tp.dw.phi(rw),
                             rh * tp.dw.K + rw});
    const RowsTiling rt = rows_tiling(F, (tp.N + bn - 1) / bn, 1, bn, p.n_cblocks, tp.nwin());
    p.cfg = use_small_cfg(bn) ? 1 : 0;
    rows_schedule(p, groups, bn, rt.G);
    p.rsplit = rt.rs;
    set_b_res(p, bn, (tp.N + bn - 1) / bn);
    const int b_box = set_pair(p, bn, rt);
    w.ms_fwd_a = map_spec(Ck, F, planes, Ck, F * Ck, 64);
    p.tma_a = make_map(w.xcl, w.ms_fwd_a);
    w.ms_fwd_b = map_spec(Ck, tp.N, tp.nwin(), Ck, (int64_t)tp.N * Ck, b_box);
    p.tma_b = make_map(w.wf, w.ms_fwd_b);
    w.wf_ident = !w.f32 && tp.fast_fold && tp.nw == 1 && tp.nwin() == 1 && tp.wstr[0][2] == tp.C &&
                 tp.wstr[0][3] == 1 && Ck == tp.C && tp.C % 8 == 0 && getenv("SYNO_TC_NO_WZC") == nullptr;
    p.Hp = w.gx.Hp;
    p.Wp = w.gx.Wp;
    p.lo_h = w.gx.lo_h;
    p.lo_w = w.gx.lo_w;
    p.H = (int)tp.dh.E;
    p.W = (int)tp.dw.E;
    p.n_img = tp.n_img;
    p.o_img = tp.y_img;
    p.o_h = tp.dh.ys;
    p.o_w = tp.dw.ys;
    p.o_n = tp.y_n;
    p.n_ext = tp.N;
    p.out_kind = rt.rs > 1 ? OUT_F32_ATOMIC : w.f32 ? OUT_F32 : OUT_BF16;
    p.scale = (float)tp.scale;
    w.bn_fwd = bn;
    w.t_fwd[0] = (int)rt.m_tiles;
    w.t_fwd[1] = (tp.N + bn - 1) / bn;
    w.t_fwd[2] = rt.rs;
    if (rt.rs > 1 && !w.f32) w.ysc = ws_alloc<float>(w, (size_t)tp.y_numel());
  }

  // ---- backward operands
  w.gdy_g = geom(tp, true, true, chs, LO_A);
  const int64_t Fg = (int64_t)w.gdy_g.n_img * w.gdy_g.Hp * w.gdy_g.Wp;
  const int Nk = w.gdy_g.Ct();
  if (w.f32) {
    // wgrad operands split along the images (its contraction dim)
    w.gxw = geom(tp, false, false, SPLIT_IMG, LO_A);
    w.gdy_w = geom(tp, true, false, SPLIT_IMG, LO_B);
  } else {
    w.gxw = w.gx;
    w.gdy_w = geom(tp, true, false);
  }
  w.share_x = !w.f32;
  w.share_dy = same_grid(w.gdy_g, w.gdy_w);
  const int64_t Fw = (int64_t)w.gxw.n_img_out() * w.gxw.Hp * w.gxw.Wp;  // wgrad K rows per plane
  if (tp.dgrad_ok) {
    w.dycl_g = ws_alloc<__nv_bfloat16>(w, (size_t)Fg * Nk);
    w.wt = ws_alloc<__nv_bfloat16>(w, (size_t)tp.nwin() * tp.C * Nk);
    if (w.f32) w.wt32 = ws_alloc<float>(w, (size_t)tp.nwin() * tp.C * tp.Np);
  }
  w.xclw = w.share_x ? w.xcl : ws_alloc<__nv_bfloat16>(w, (size_t)planes * Fw * tp.Cp);
  w.dycl_w = (w.share_dy && w.dycl_g) ? w.dycl_g : ws_alloc<__nv_bfloat16>(w, (size_t)Fw * tp.Np);
  w.dwf = ws_alloc<float>(w, (size_t)tp.nwin() * tp.N * tp.C);

  // ---- grad-input: one group per output phase (psi_h, psi_w); its windows have phi(r) == psi
  if (tp.dgrad_ok) {
    const int bn = pick_bn(tp.C, Fg);
    TcGemmParams& p = w.dg;
    memset(&p, 0, sizeof(p));
    p.mode = MODE_ROWS;
    p.n_cblocks = (Nk + BK - 1) / BK;
    p.kq_last = (Nk - (p.n_cblocks - 1) * BK + 15) / 16;
    const int Sh = tp.dh.S, Sw = tp.dw.S;
    std::vector<std::vector<Win>> groups(Sh * Sw);
    for (int ph = 0; ph < Sh; ++ph)
      for (int pw = 0; pw < Sw; ++pw) {
        const int grp = ph * Sw + pw;
        for (int rh = 0; rh < tp.dh.K; ++rh)
          for (int rw = 0; rw < tp.dw.K; ++rw) {
            if (tp.dh.phi(rh) != ph || tp.dw.phi(rw) != pw) continue;
            groups[grp].push_back({-tp.dh.delta(rh) * w.gdy_g.Wp - tp.dw.delta(rw), 0, rh * tp.dw.K + rw});
          }
        p.g_out_off[grp] = ph * tp.dh.xs + pw * tp.dw.xs;
      }
    const RowsTiling rt = rows_tiling(Fg, (tp.C + bn - 1) / bn, Sh * Sw, bn, p.n_cblocks, tp.nwin() / (Sh * Sw));
    p.cfg = use_small_cfg(bn) ? 1 : 0;
    rows_schedule(p, groups, bn, rt.G);
    p.rsplit = rt.rs;
    set_b_res(p, bn, (tp.C + bn - 1) / bn);
    const int b_box = set_pair(p, bn, rt);
    // MN-major view of a [N][C] weight: dims (C, N), 64 K (= N) rows per box
    w.wt_ident = !w.f32 && tp.fast_fold && tp.nw == 1 && tp.nwin() == 1 && tp.wstr[0][2] == tp.C &&
                 tp.wstr[0][3] == 1 && tp.C % 8 == 0 && !p.b_res && getenv("SYNO_TC_NO_WZC") == nullptr;
    w.ms_dg_b_mn = map_spec(tp.C, tp.N, 1, tp.C, (int64_t)tp.N * tp.C, 64);
    w.ms_dg_a = map_spec(Nk, Fg, 1, Nk, Fg * Nk, 64);
    p.tma_a = make_map(w.dycl_g, w.ms_dg_a);
    p.tma_b = make_map(w.wt, Nk, tp.C, tp.nwin(), Nk, (int64_t)tp.C * Nk, b_box);
    p.Hp = w.gdy_g.Hp;
    p.Wp = w.gdy_g.Wp;
    p.lo_h = w.gdy_g.lo_h;
    p.lo_w = w.gdy_g.lo_w;
    p.H = (int)tp.dh.E;
    p.W = (int)tp.dw.E;
    p.n_img = tp.n_img;
    p.o_img = tp.x_img;
    p.o_h = tp.dh.xs * Sh;
    p.o_w = tp.dw.xs * Sw;
    p.o_n = tp.x_c;
    p.n_ext = tp.C;
    p.out_kind = rt.rs > 1 ? OUT_F32_ATOMIC : w.f32 ? OUT_F32 : OUT_BF16;
    p.scale = (float)tp.scale;
    w.bn_dg = bn;
    w.t_dg[0] = (int)rt.m_tiles;
    w.t_dg[1] = (tp.C + bn - 1) / bn;
    w.t_dg[2] = Sh * Sw * rt.rs;
    if (rt.rs > 1 && !w.f32) w.dxsc = ws_alloc<float>(w, (size_t)tp.x_numel());
  }

  // ---- grad-weight: both operands channels-last over the forward's flat
  // padded grid, read MN-major (K = pixel rows): a window is a row shift
  {
    // M = (window, 64-channel block of C_in) pairs, N = C_out, K = pixel rows
    // the forward's tile-count rule decides the grad-weight tile width too: the
    // l3/l4 grad-weights take 128-wide tiles (ResNet-18 step 1.356 -> 1.317 ms,
    // ResNet-34 and QKV unchanged; SYNO_TC_WG_BN_FILL=0 disables)
    static const bool wg_fill = !(getenv("SYNO_TC_WG_BN_FILL") && atoi(getenv("SYNO_TC_WG_BN_FILL")) == 0);
    const int bn = pick_bn(tp.N, wg_fill ? F : -1);
    TcGemmParams& p = w.wg;
    memset(&p, 0, sizeof(p));
    w.ms_wg_a = map_spec(tp.Cp, Fw, planes, tp.Cp, Fw * tp.Cp, 64);
    w.ms_wg_b = map_spec(tp.Np, Fw, 1, tp.Np, Fw * tp.Np, 64);
    p.tma_a = make_map(w.xclw, w.ms_wg_a);
    p.tma_b = make_map(w.dycl_w, w.ms_wg_b);
    p.mode = MODE_WGRAD;
    p.n_cblocks = (int)((Fw + BK - 1) / BK);
    p.n_win = tp.nwin();
    const int ncb = (tp.Cp + 63) / 64;
    for (int rh = 0; rh < tp.dh.K; ++rh)
      for (int rw = 0; rw < tp.dw.K; ++rw) {
        const int wi = rh * tp.dw.K + rw;
        p.a_shift[wi] = tp.dh.delta(rh) * w.gx.Wp + tp.dw.delta(rw);
        p.a_plane[wi] = tp.dh.phi(rh) * w.gx.Sw + tp.dw.phi(rw);
        for (int cb = 0; cb < ncb; ++cb) {
          if (p.n_pairs >= MAXPAIR) fail(SYNO_E_UNSUPPORTED, "too many (window, channel block) pairs");
          p.pair_win[p.n_pairs] = (int16_t)wi;
          p.pair_cb[p.n_pairs] = (int16_t)cb;
          ++p.n_pairs;
        }
      }
    const int m_tiles = (p.n_pairs + 1) / 2, n_tiles = (tp.N + bn - 1) / bn;
    // split-K sized to fill the grid once; long contractions (>= 64 pixel
    // blocks per split) fill it twice (measured: QKV 0.184 -> 0.178 ms,
    // ResNet-18's short splits slower at two waves); SYNO_TC_WG_WAVES overrides
    static const int waves_env = getenv("SYNO_TC_WG_WAVES") ? atoi(getenv("SYNO_TC_WG_WAVES")) : 0;
    p.cfg = use_small_cfg(bn) ? 1 : 0;
    auto split_for = [&](int waves) {
      const int k = std::max(1, (waves * sm_count() * (p.cfg ? 2 : 1)) / std::max(1, m_tiles * n_tiles));
      return std::min(k, std::max(1, p.n_cblocks / 4));
    };
    int ksplit = split_for(waves_env > 0 ? waves_env : 1);
    if (waves_env <= 0 && p.n_cblocks / ksplit >= 64) ksplit = split_for(2);
    p.ksplit = ksplit;
    // CTA pair (BN = 256, two or more M tiles): each CTA stages half of the
    // dy columns; SYNO_TC_PAIR=0 / SYNO_TC_WG_PAIR=0 disable
    static const bool wg_pair = !(getenv("SYNO_TC_PAIR") && atoi(getenv("SYNO_TC_PAIR")) == 0) &&
                                !(getenv("SYNO_TC_WG_PAIR") && atoi(getenv("SYNO_TC_WG_PAIR")) == 0);
    const bool pair_wg = wg_pair && bn == 256 && m_tiles >= 2 && getenv("SYNO_TC_FIXUP") == nullptr;
    if (pair_wg) p.cfg = CFG_PAIR;
    p.m_ext = tp.C;
    p.n_ext = tp.N;
    p.o_m = 1;
    p.o_n = tp.C;
    for (int wi = 0; wi < tp.nwin(); ++wi) p.g_out_off[wi] = (int64_t)wi * tp.N * tp.C;
    p.out_kind = OUT_F32_ATOMIC;
    p.scale = (float)tp.scale;
    p.out = w.dwf;
    p.a_rows = 64;
    p.a_tx = (uint32_t)BM * BK * 2 * (pair_wg ? 2 : 1);  // the pair kernel stages two K blocks
    p.a_stage_bytes = (int)p.a_tx;
    p.b_tx = (uint32_t)(pair_wg ? bn / 2 * 2 : bn) * BK * 2;
    w.bn_wg = bn;
    w.t_wg[0] = m_tiles;
    w.t_wg[1] = n_tiles;
    w.t_wg[2] = ksplit;
    // single weight whose fold is a pure permutation of (rh, rw, n, ci): the
    // last split of each tile writes dW itself
    // measured slower than the separate chain-rule kernel (the last split's
    // strided dW writes serialise in the GEMM tail): opt-in only
    bool perm = tp.fast_fold && tp.nw == 1 && getenv("SYNO_TC_FIXUP") != nullptr;
    const int64_t ext[4] = {tp.dh.K, tp.dw.K, tp.N, tp.C};
    for (int l = 0; l < 4 && perm; ++l) perm = ext[l] == 1 || tp.wstr[0][l] != 0;
    if (perm) {
      w.wg_fixup = true;
      p.fix_cnt = ws_alloc<unsigned>(w, (size_t)m_tiles * n_tiles);
      for (int rh = 0; rh < tp.dh.K; ++rh)
        for (int rw = 0; rw < tp.dw.K; ++rw)
          p.fix_win_off[rh * tp.dw.K + rw] = rh * tp.wstr[0][0] + rw * tp.wstr[0][1];
      p.fix_s_co = tp.wstr[0][2];
      p.fix_s_ci = tp.wstr[0][3];
      p.fix_f32 = w.f32 ? 1 : 0;
    }
  }

  if (tc_log()) {
    log_pack("ws x", nullptr, w.gx);
    log_pack("ws xw", nullptr, w.gxw);
    log_pack("ws dy_g", nullptr, w.gdy_g);
    log_pack("ws dy_w", nullptr, w.gdy_w);
    fprintf(stderr, "[tc] ws share_x=%d share_dy=%d\n", (int)w.share_x, (int)w.share_dy);
  }
  w.x_ident = pack_identity(w.gx, dt);
  w.xw_ident = pack_identity(w.gxw, dt);
  w.dyg_ident = tp.dgrad_ok && pack_identity(w.gdy_g, dt);
  w.dyw_ident = pack_identity(w.gdy_w, dt);

  // ---- fast chain rule: per weight, thread mode or split block mode
  if (tp.fast_fold) {
    const int64_t ext[4] = {tp.dh.K, tp.dw.K, tp.N, tp.C};
    int64_t need = 0, outs = 0;
    for (int j = 0; j < tp.nw; ++j) {
      int64_t oc = 1, R = 1;
      for (int l = 0; l < 4; ++l) (tp.wstr[j][l] ? oc : R) *= ext[l];
      int nsplit = 0;
      if (R > 64) nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(256, R / 1024));
      w.chain_nsplit[j] = nsplit;
      if (nsplit) {
        need = std::max(need, oc * nsplit);
        outs = std::max(outs, oc);
      }
    }
    // fused side chains (chain_side_ok): one partial per (block, window)
    need = std::max(need, ((int64_t)tp.N * tp.C + 255) / 256 * 16);
    need = std::max(need, ((int64_t)tp.N * tp.C / 4 + 31) / 32 * 16);  // chain_v4 warp partials
    outs = std::max<int64_t>(outs, 1);
    if (need) {
      w.chain_partial = ws_alloc<float>(w, (size_t)need);
      w.chain_counter = ws_alloc<unsigned>(w, (size_t)outs);
      cuda_check(cudaMemsetAsync(w.chain_counter, 0, (size_t)outs * sizeof(unsigned), g_ws_stream),
                 "memset(chain counter)");
    }
  }
}

static FoldArgs fold_args(const TcPlan& tp, const Bindings& b, DType dt, bool dgrad, bool split, __nv_bfloat16* dst) {
  FoldArgs f{};
  f.nw = tp.nw;
  f.f32 = dt == DT_F32;
  for (int j = 0; j < tp.nw; ++j) {
    f.w[j] = b.w.at(j);
    for (int l = 0; l < 4; ++l) f.s[j][l] = tp.wstr[j][l];
  }
  f.ext[0] = tp.dh.K;
  f.ext[1] = tp.dw.K;
  f.ext[2] = dgrad ? tp.C : tp.N;
  f.ext[3] = dgrad ? tp.N : tp.C;
  f.sl_a = dgrad ? 3 : 2;
  f.sl_b = dgrad ? 2 : 3;
  f.Bp = dgrad ? tp.Np : tp.Cp;
  f.split = split;
  f.out = dst;
  return f;
}

template <typename TI, int V>
static void launch_prep(const void* src, const PackGeom& g, __nv_bfloat16* dst, const PackPlan& pp,
                        const FoldArgs& f, cudaStream_t stream) {
  const uint32_t n_pack = pp.grid.x * pp.grid.y;
  const uint32_t fold_gx = (uint32_t)f.ext[2];
  const uint32_t n_fold = fold_gx * (uint32_t)((f.Bp + 63) / 64);
  launch_k(prep_kernel<TI, V>, n_pack + n_fold, 256, 0, stream, static_cast<const TI*>(src), dst, g, pp.rpb, pp.rows,
           pp.grid.x, n_pack, f, fold_gx);
}

// Pack the activation operand and fold the weight operand of one GEMM in a
// single launch (they are independent); false when the fold is not of the
// direct kind (the caller then launches them separately).
static bool pack_and_fold(const TcPlan& tp, const Bindings& b, DType dt, const void* src, const PackGeom& g,
                          __nv_bfloat16* packed, bool dgrad, bool split, __nv_bfloat16* folded, cudaStream_t stream) {
  const int KK = tp.dh.K * tp.dw.K;
  if (!tp.fast_fold || KK <= 1 || KK > 16 || getenv("SYNO_TC_NO_PREP_FUSE")) return false;
  if (skip_class("pack") || skip_class("fold")) return false;
  const PackPlan pp = pack_plan(src, dt, g);
  PackGeom gf = g;
  gf.flat = pp.flat;
  log_pack(dgrad ? "prep(dgrad)" : "prep(fwd)", src, g);
  const FoldArgs f = fold_args(tp, b, dt, dgrad, split, folded);
  const double fold_elems = (double)KK * f.ext[2] * f.Bp;
  const int id = prof_begin("pack_cl", 0.0, pack_bytes(dt, g) + fold_elems * (split ? 6 : 2), stream);
  note_launch();
  if (dt == DT_BF16) {
    if (pp.V == 8) launch_prep<__nv_bfloat16, 8>(src, gf, packed, pp, f, stream);
    else if (pp.V == 4) launch_prep<__nv_bfloat16, 4>(src, gf, packed, pp, f, stream);
    else launch_prep<__nv_bfloat16, 1>(src, gf, packed, pp, f, stream);
  } else {
    if (pp.V == 4) launch_prep<float, 4>(src, gf, packed, pp, f, stream);
    else launch_prep<float, 1>(src, gf, packed, pp, f, stream);
  }
  cuda_check(cudaGetLastError(), "prep_kernel");
  prof_end(id, stream);
  return true;
}

static void fold_fast(const TcPlan& tp, const Bindings& b, DType dt, bool dgrad, bool split, __nv_bfloat16* dst,
                      cudaStream_t stream) {
  if (skip_class("fold")) return;
  FoldArgs f{};
  f.nw = tp.nw;
  f.f32 = dt == DT_F32;
  for (int j = 0; j < tp.nw; ++j) {
    f.w[j] = b.w.at(j);
    for (int l = 0; l < 4; ++l) f.s[j][l] = tp.wstr[j][l];
  }
  f.ext[0] = tp.dh.K;
  f.ext[1] = tp.dw.K;
  f.ext[2] = dgrad ? tp.C : tp.N;
  f.ext[3] = dgrad ? tp.N : tp.C;
  f.sl_a = dgrad ? 3 : 2;
  f.sl_b = dgrad ? 2 : 3;
  f.Bp = dgrad ? tp.Np : tp.Cp;
  f.split = split;
  f.out = dst;
  const int KK = f.ext[0] * f.ext[1];
  const int64_t rows = (int64_t)KK * f.ext[2];
  const double elems = (double)rows * f.Bp;
  const int id = prof_begin("weight_fold", 0.0, elems * (split ? 6 : 2) + elems * tp.nw * (f.f32 ? 4 : 2), stream);
  note_launch();
  // read order: the first weight's smaller stride of (a, b) goes inner
  const int a_inner = std::llabs(tp.wstr[0][f.sl_a]) < std::llabs(tp.wstr[0][f.sl_b]) ? 1 : 0;
  if (KK == 1) {
    const size_t sm = (size_t)32 * 33 * sizeof(float);
    launch_k(fold_tile_kernel<32, 32>, dim3((unsigned)((f.ext[2] + 31) / 32), (unsigned)((f.Bp + 31) / 32)), 256, sm, stream, f, a_inner);
  } else if (KK <= 16) {
    launch_k(fold_direct_kernel, dim3((unsigned)f.ext[2], (unsigned)((f.Bp + 63) / 64)), 256, 0, stream, f);
  } else {
    if (rows > 65535) fail(SYNO_E_UNSUPPORTED, "fold: too many operand rows");
    dim3 grid((unsigned)std::min(8, (f.Bp + 127) / 128), (unsigned)rows);
    launch_k(fold_kernel, grid, 128, 0, stream, f);
  }
  cuda_check(cudaGetLastError(), "fold kernel");
  prof_end(id, stream);
}

// Forward + grad-input B operands in one launch (KK <= 9).
static bool fold_dual(const TcPlan& tp, const Bindings& b, DType dt, bool split, __nv_bfloat16* wf,
                      __nv_bfloat16* wt, cudaStream_t stream) {
  const int KK = tp.dh.K * tp.dw.K;
  // measured slower than two direct folds for the ResNet shapes (few tiles,
  // serial windows per thread); opt-in until the tiling is reworked
  static const bool on = getenv("SYNO_TC_DUAL_FOLD") != nullptr;
  if (KK > 9 || !on) return false;
  if (skip_class("fold")) return true;
  FoldDual d{};
  FoldArgs& f = d.f;
  f.nw = tp.nw;
  f.f32 = dt == DT_F32;
  for (int j = 0; j < tp.nw; ++j) {
    f.w[j] = b.w.at(j);
    for (int l = 0; l < 4; ++l) f.s[j][l] = tp.wstr[j][l];
  }
  f.ext[0] = tp.dh.K;
  f.ext[1] = tp.dw.K;
  f.ext[2] = tp.N;
  f.ext[3] = tp.C;
  f.Bp = tp.Cp;
  f.split = split;
  f.out = wf;
  d.out_t = wt;
  d.Np = tp.Np;
  const double elems = (double)KK * tp.N * tp.C;
  const int id = prof_begin("weight_fold", 0.0, elems * (split ? 12 : 4) + elems * tp.nw * (f.f32 ? 4 : 2), stream);
  note_launch();
  const int gy = (std::max(tp.C, tp.Np) + 31) / 32;
  const int gx = (std::max(tp.N, tp.Np) + 31) / 32;
  launch_k(fold_dual_kernel, dim3((unsigned)gx, (unsigned)gy), 256, (size_t)KK * 32 * 33 * sizeof(float), stream, d);
  cuda_check(cudaGetLastError(), "fold_dual_kernel");
  prof_end(id, stream);
  return true;
}

// Whether weight j2's gradient can ride along j's chain_nc pass (side output).
static bool chain_side_ok(const TcPlan& tp, int j, int j2) {
  if (j2 == j || tp.dh.K * tp.dw.K > 16) return false;
  if (!(tp.wstr[j][2] != 0 && tp.wstr[j][3] != 0)) return false;
  return tp.wstr[j2][2] == 0 && tp.wstr[j2][3] == 0;
}

static void chain_fast(const TcPlan& tp, const TcWs& w, const Bindings& b, DType dt, int j, bool zero_dwf,
                       cudaStream_t stream, int side = -1) {
  if (skip_class("chain")) return;
  ChainArgs c{};
  c.dwf = w.dwf;
  c.zero_dwf = zero_dwf ? 1 : 0;
  c.nw = tp.nw;
  c.j = j;
  c.f32 = dt == DT_F32;
  for (int k = 0; k < tp.nw; ++k) {
    c.w[k] = b.w.at(k);
    for (int l = 0; l < 4; ++l) c.s[k][l] = tp.wstr[k][l];
  }
  c.ext[0] = tp.dh.K;
  c.ext[1] = tp.dw.K;
  c.ext[2] = tp.N;
  c.ext[3] = tp.C;
  c.out_count = c.R = 1;
  for (int l = 0; l < 4; ++l) {
    if (tp.wstr[j][l]) {
      c.out_l[c.nout++] = l;
      c.out_count *= c.ext[l];
    } else {
      c.red_l[c.nred++] = l;
      c.R *= c.ext[l];
    }
  }
  if (c.out_count >= INT32_MAX || c.R >= INT32_MAX) fail(SYNO_E_UNSUPPORTED, "chain rule: 2^31 or more elements");
  c.out = b.dw.at(j);
  const double bytes = (double)c.out_count * c.R * 4 + (double)c.out_count * (c.f32 ? 4 : 2);
  const int id = prof_begin("weight_chain", 0.0, bytes, stream);
  note_launch();
  const int nsplit = w.chain_nsplit[j];
  if (!nsplit && tp.wstr[j][2] != 0 && tp.wstr[j][3] != 0 && c.ext[0] * c.ext[1] <= 16) {
    ChainNC h{};
    h.Kh = (int)c.ext[0];
    h.Kw = (int)c.ext[1];
    h.N = (int)c.ext[2];
    h.C = (int)c.ext[3];
    h.so_n = (int32_t)tp.wstr[j][2];
    h.so_c = (int32_t)tp.wstr[j][3];
    h.oh = tp.wstr[j][0] != 0 || h.Kh == 1;
    h.ow = tp.wstr[j][1] != 0 || h.Kw == 1;
    h.so_h = (int32_t)tp.wstr[j][0];
    h.so_w = (int32_t)tp.wstr[j][1];
    for (int k = 0; k < tp.nw; ++k)
      for (int l = 0; l < 4; ++l) h.sw[k][l] = k == j ? 0 : (int32_t)tp.wstr[k][l];
    const int64_t nthreads = (int64_t)h.N * h.C;
    // dense [n][ci][windows] layout (OIHW-like): outputs of consecutive (n, ci) are contiguous
    const int kko = (h.oh ? h.Kh : 1) * (h.ow ? h.Kw : 1);
    const bool win_dense = (h.oh && h.ow) ? (h.so_w == 1 && h.so_h == h.Kw) || (h.Kh == 1 && h.so_w == 1) ||
                                                (h.Kw == 1 && h.so_h == 1)
                           : h.oh ? (h.Kh == 1 || h.so_h == 1) : h.ow ? (h.Kw == 1 || h.so_w == 1) : true;
    h.dense = win_dense && h.so_c == kko && h.so_n == h.C * kko;
    h.side_j = -1;
    if (side >= 0) {
      h.side_j = side;
      for (int k = 0; k < tp.nw; ++k)
        for (int l = 0; l < 4; ++l) h.side_sw[k][l] = k == side ? 0 : (int32_t)tp.wstr[k][l];
      h.side_oh = tp.wstr[side][0] != 0 || h.Kh == 1;
      h.side_ow = tp.wstr[side][1] != 0 || h.Kw == 1;
      h.side_so_h = (int32_t)tp.wstr[side][0];
      h.side_so_w = (int32_t)tp.wstr[side][1];
      h.side_out = b.dw.at(side);
      h.partial = w.chain_partial;
      h.counter = w.chain_counter;
    }
    const size_t sm = (size_t)256 * (kko + (side >= 0 ? 17 : 0)) * sizeof(float);
    const unsigned grid = (unsigned)((nthreads + 255) / 256);
    static const bool win_split = getenv("SYNO_TC_NO_CHAIN_WIN") == nullptr;
    const bool aligned = (reinterpret_cast<uintptr_t>(c.out) & 15) == 0 && (reinterpret_cast<uintptr_t>(c.dwf) & 15) == 0;
    auto launch_once = [&]() {
      // vectorised form: 3 x 3 windows, dense [n][ci][window outputs], four ci per thread
      static const bool v4_on = getenv("SYNO_TC_NO_CHAIN_V4") == nullptr;  // A/B switch
      const bool v4 = v4_on && h.Kh == 3 && h.Kw == 3 && h.dense && h.C % 4 == 0 &&
                      // single-weight convolutions: only where one thread per element would need
                      // many waves (64 x 64: chain_win 6.6 us vs 8.8 us; 512 x 512: 17.0 vs 14.2 us)
                      ((tp.nw == 1 && side < 0 && h.oh && h.ow && nthreads >= 65536) ||
                       (tp.nw == 2 && side >= 0 && h.oh != h.ow)) &&
                      (reinterpret_cast<uintptr_t>(c.dwf) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(c.out) & (c.f32 ? 3 : 7)) == 0;
      if (v4) {
        // SYNO_TC_V4_ONE=<pairs>: problems that small run as one block walking its
        // elements (no cross-block side reduction) -- measured slower (64 x 64
        // conv3x3 18.4 vs 8.8 us, sep_shared 16.3 vs 14.8 us), so off by default
        // side output reduced through global warp partials (no shared memory, no
        // block-level tree) where the last warp has few partials to sum: up to 128
        // warps (64 x 64 sep_shared chain 12.7 -> 10.6 us, 128 x 128 12.7 -> 10.9;
        // 512 x 512 would sum 2048: 14.9 -> 21 us); SYNO_TC_V4_WRED=0/1 forces it
        static const int wred_env = getenv("SYNO_TC_V4_WRED") ? atoi(getenv("SYNO_TC_V4_WRED")) : -1;
        const bool v4_wred = wred_env >= 0 ? wred_env != 0 : nthreads / 4 / 32 <= 128;
        static const int64_t one_max = getenv("SYNO_TC_V4_ONE") ? atoll(getenv("SYNO_TC_V4_ONE")) : 0;
        // SYNO_TC_V4_BLOCK: threads per block (A/B: a smaller block can co-reside with the
        // concurrent grad-input GEMM's CTAs, whose registers fill most of each SM)
        static const int v4_block = getenv("SYNO_TC_V4_BLOCK") ? atoi(getenv("SYNO_TC_V4_BLOCK")) : 256;
        const unsigned g4 = nthreads <= one_max ? 1u : (unsigned)((nthreads / 4 + v4_block - 1) / v4_block);
        if (side < 0) launch_k(chain_v4_kernel<3, 3, true, true, false>, g4, v4_block, 0, stream, c, h);
        else if (v4_wred && g4 > 1 && h.oh) launch_k(chain_v4_kernel<3, 3, true, false, true, true>, g4, v4_block, 0, stream, c, h);
        else if (v4_wred && g4 > 1) launch_k(chain_v4_kernel<3, 3, false, true, true, true>, g4, v4_block, 0, stream, c, h);
        else if (h.oh) launch_k(chain_v4_kernel<3, 3, true, false, true>, g4, v4_block, 0, stream, c, h);
        else launch_k(chain_v4_kernel<3, 3, false, true, true>, g4, v4_block, 0, stream, c, h);
      } else if (tp.nw == 1 && side < 0 && h.Kh * h.Kw == 1 && h.so_c == 1 && h.so_n == h.C && aligned) {
        const int64_t n = (int64_t)h.N * h.C;
        launch_k(chain_cast_kernel, (unsigned)((n / 4 + 256) / 256), 256, 0, stream, c.dwf, c.out, n, c.f32,
                 c.zero_dwf);
      } else if (win_split && tp.nw == 1 && side < 0 && (h.oh || h.Kh == 1) && (h.ow || h.Kw == 1) && h.Kh * h.Kw > 1) {
        launch_k(chain_win_kernel, dim3(grid, (unsigned)(h.Kh * h.Kw)), 256, 0, stream, c, h);
      } else if (h.Kh == 3 && h.Kw == 3) launch_k(chain_nc_kernel<3, 3>, grid, 256, sm, stream, c, h);
      else if (h.Kh == 1 && h.Kw == 1) launch_k(chain_nc_kernel<1, 1>, grid, 256, sm, stream, c, h);
      else launch_k(chain_nc_kernel<0, 0>, grid, 256, sm, stream, c, h);
    };
    launch_once();
    cuda_check(cudaGetLastError(), "chain kernel");
    prof_end(id, stream);
    // SYNO_TC_CHAIN_TWICE (timing experiment only; the second pass reads the
    // zeroed dWf): the same launch again with its code already fetched
    static const bool twice = getenv("SYNO_TC_CHAIN_TWICE") != nullptr;
    if (twice) {
      const int id2 = prof_begin("weight_chain_warm", 0.0, bytes, stream);
      launch_once();
      prof_end(id2, stream);
    }
    return;
  }
  const bool ci_out = tp.wstr[j][3] != 0;
  const int chunk = ci_out ? 64 : 0;
  const int cw_max = ci_out ? std::min(64, (int)c.ext[3]) : (int)c.ext[3];
  const size_t sm_n = (size_t)c.ext[0] * c.ext[1] * (cw_max + 1) * sizeof(float);
  if (!nsplit && tp.wstr[j][2] != 0 && sm_n <= 48 * 1024) {
    // n is an output loop: one block per (output channel, 64 input channels)
    ChainN h{};
    h.KK = (int)(c.ext[0] * c.ext[1]);
    h.C = (int)c.ext[3];
    h.Kw = (int)c.ext[1];
    h.ci_chunk = chunk;
    h.ci_q = -1;
    const int P = cw_max + 1;
    const int32_t smul[4] = {(int32_t)c.ext[1] * P, P, 0, 1};
    int ol[3], n_ol = 0, rl[3], n_rl = 0;
    for (int l : {0, 1, 3}) {
      if (tp.wstr[j][l]) ol[n_ol++] = l;
      else if (c.ext[l] > 1) rl[n_rl++] = l;
    }
    std::sort(ol, ol + n_ol, [&](int x, int y) { return tp.wstr[j][x] > tp.wstr[j][y]; });
    h.n_ol = n_ol;
    h.n_rl = n_rl;
    for (int q = 0; q < n_ol; ++q) {
      const int l = ol[q];
      if (l == 3) h.ci_q = q;
      h.ol_ext[q] = (int)c.ext[l];
      h.ol_sm[q] = smul[l];
      h.ol_out[q] = (int32_t)tp.wstr[j][l];
      for (int k = 0; k < tp.nw; ++k) h.ol_w[q][k] = k == j ? 0 : (int32_t)tp.wstr[k][l];
    }
    for (int q = 0; q < n_rl; ++q) {
      const int l = rl[q];
      h.rl_ext[q] = (int)c.ext[l];
      h.rl_sm[q] = smul[l];
      for (int k = 0; k < tp.nw; ++k) h.rl_w[q][k] = k == j ? 0 : (int32_t)tp.wstr[k][l];
    }
    h.n_out = (int32_t)tp.wstr[j][2];
    for (int k = 0; k < tp.nw; ++k) h.n_w[k] = k == j ? 0 : (int32_t)tp.wstr[k][2];
    if (!ci_out) h.ci_chunk = 0;
    const unsigned gy = ci_out ? (unsigned)((c.ext[3] + chunk - 1) / chunk) : 1u;
    launch_k(chain_n_kernel, dim3((unsigned)c.ext[2], gy), 256, sm_n, stream, c, h);
  } else if (!nsplit) {
    launch_k(chain_thread_kernel, (unsigned)((c.out_count + 255) / 256), 256, 0, stream, c);
  } else {
    c.r_chunk = (c.R + nsplit - 1) / nsplit;
    c.partial = w.chain_partial;
    c.counter = w.chain_counter;
    const int ns = (int)((c.R + c.r_chunk - 1) / c.r_chunk);
    launch_k(chain_block_kernel, dim3((unsigned)c.out_count, (unsigned)ns), 256, 0, stream, c);
  }
  cuda_check(cudaGetLastError(), "chain kernel");
  prof_end(id, stream);
}

static TcWs& workspace(TcPlan& tp, DType dt, cudaStream_t stream) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(tp.mu);
  auto key = std::make_tuple(dev, (void*)stream, (int)dt);
  auto it = tp.ws.find(key);
  if (it != tp.ws.end()) return *it->second;
  auto w = std::make_unique<TcWs>();
  // the zero fills go on the caller's stream (cudaMemset would run on the
  // legacy default stream, unordered against non-blocking streams)
  g_ws_stream = stream;
  build_ws(tp, *w, dt);
  g_ws_stream = nullptr;
  TcWs& ref = *w;
  tp.ws[key] = std::move(w);
  return ref;
}

// Folded weights into the B operand: bf16 folds straight into it; fp32
// folds in fp32 and is split into (hi, lo, hi) parts.
static void fold_into(TcWs& w, const DevStage& fold, DType dt, const Bindings& b, float* f32_tmp,
                      __nv_bfloat16* dst, int64_t rows, int Cp, cudaStream_t stream) {
  if (!w.f32) {
    run_stage(dt, fold, b, dst, false, stream);
    return;
  }
  run_stage(dt, fold, b, f32_tmp, false, stream);
  split_rows(f32_tmp, dst, rows, Cp, LO_B, stream);
}

static bool tc_dtype(DType dt) { return dt == DT_BF16 || dt == DT_F32; }

// MODE_ROWS launch into `out`; a split-K launch accumulates fp32 atomically
// (into `out` itself for fp32, else into `acc` followed by a cast).
static void rows_gemm(TcGemmParams& p, int bn, const int* t, void* out, bool f32, float* acc, int64_t numel,
                      cudaStream_t stream, const char* name, double flops) {
  if (p.rsplit <= 1) {
    p.out = out;
    gemm(p, bn, t[0], t[1], t[2], stream, name, flops);
    return;
  }
  float* target = f32 ? static_cast<float*>(out) : acc;
  if (f32) zero_fill(target, (size_t)numel * sizeof(float), stream);  // acc is kept zeroed by the cast
  p.out = target;
  gemm(p, bn, t[0], t[1], t[2], stream, name, flops);
  if (!f32) cast_to_bf16(target, out, numel, stream);
}

bool tc_forward(TcPlan& tp, DType dt, const Bindings& b, cudaStream_t stream) {
  if (!tc_dtype(dt)) return false;
  TcWs& w = workspace(tp, dt, stream);
  TcGemmParams p = w.fwd;
  w.wt_src.clear();
  bool fused = false;
  const bool w_zero = w.wf_ident && aligned16(b.w.at(0));
  if (w_zero) p.tma_b = make_map(b.w[0], w.ms_fwd_b);
  if (w.x_ident && aligned16(b.x)) {
    p.tma_a = make_map(b.x, w.ms_fwd_a);
  } else if (!w_zero && pack_and_fold(tp, b, dt, b.x, w.gx, w.xcl, false, w.f32, w.wf, stream)) {
    w.packed_x_src = b.x;
    fused = true;
  } else {
    pack_cl(b.x, dt, w.gx, w.xcl, stream);
    w.packed_x_src = b.x;
  }
  if (fused || w_zero) {
    // operand folded by the fused launch / read in place
  } else if (tp.fast_fold && tp.dgrad_ok && fold_dual(tp, b, dt, w.f32, w.wf, w.wt, stream)) {
    w.wt_src = b.w;
  } else if (tp.fast_fold) {
    fold_fast(tp, b, dt, false, w.f32, w.wf, stream);
  } else {
    fold_into(w, tp.fold_fwd, dt, b, w.wf32, w.wf, (int64_t)tp.nwin() * tp.N, tp.Cp, stream);
  }
  rows_gemm(p, w.bn_fwd, w.t_fwd, b.y, w.f32, w.ysc, tp.y_numel(), stream, "tc_gemm_fwd", tp.flops);
  return true;
}

bool tc_backward(TcPlan& tp, DType dt, const Bindings& b, cudaStream_t stream) {
  if (!tc_dtype(dt)) return false;
  if (b.dx && !tp.dgrad_ok) return false;
  TcWs& w = workspace(tp, dt, stream);
  bool any_w = false;
  for (auto* q : b.dw) any_w = any_w || q;
  bool dy_w_packed = false;
  static const bool concurrent = getenv("SYNO_TC_SERIAL_BWD") == nullptr;
  const bool fork = concurrent && !prof_active() && b.dx && any_w;
  cudaStream_t wstream = stream;
  if (b.dx) {
    TcGemmParams p = w.dg;
    const bool wt_zero = w.wt_ident && aligned16(b.w.at(0));
    if (wt_zero) {
      p.tma_b = make_map(b.w[0], w.ms_dg_b_mn);
      p.b_mn = 1;
    }
    const bool wt_ready = wt_zero || (b.w_unchanged && !w.wt_src.empty() && w.wt_src == b.w);
    bool fused = false;
    if (w.dyg_ident && aligned16(b.dy)) {
      p.tma_a = make_map(b.dy, w.ms_dg_a);
    } else if (!wt_ready && pack_and_fold(tp, b, dt, b.dy, w.gdy_g, w.dycl_g, true, w.f32, w.wt, stream)) {
      dy_w_packed = w.share_dy;
      fused = true;
    } else {
      pack_cl(b.dy, dt, w.gdy_g, w.dycl_g, stream);
      dy_w_packed = w.share_dy;
    }
    if (wt_ready || fused) {
      // the forward folded the grad-input operand from these same weights
    } else if (tp.fast_fold) {
      fold_fast(tp, b, dt, true, w.f32, w.wt, stream);
    } else {
      fold_into(w, tp.fold_dgrad, dt, b, w.wt32, w.wt, (int64_t)tp.nwin() * tp.C, tp.Np, stream);
    }
    if (fork) {
      if (!w.side) {
        cuda_check(cudaStreamCreateWithFlags(&w.side, cudaStreamNonBlocking), "cudaStreamCreate(side)");
        cuda_check(cudaEventCreateWithFlags(&w.ev_fork, cudaEventDisableTiming), "cudaEventCreate(fork)");
        cuda_check(cudaEventCreateWithFlags(&w.ev_join, cudaEventDisableTiming), "cudaEventCreate(join)");
      }
      // the packed dy (and the rest of the stream's prior work) is ready for grad-weight
      cuda_check(cudaEventRecord(w.ev_fork, stream), "cudaEventRecord(fork)");
      cuda_check(cudaStreamWaitEvent(w.side, w.ev_fork, 0), "cudaStreamWaitEvent(fork)");
      wstream = w.side;
    }
    rows_gemm(p, w.bn_dg, w.t_dg, b.dx, w.f32, w.dxsc, tp.x_numel(), stream, "tc_gemm_dgrad", tp.flops);
  }
  if (any_w) {
    cudaStream_t stream = wstream;  // grad-weight work: the side stream when forked
    TcGemmParams p = w.wg;
    if (w.xw_ident && aligned16(b.x)) p.tma_a = make_map(b.x, w.ms_wg_a);
    else if (!(b.x_unchanged && w.share_x && w.packed_x_src == b.x)) pack_cl(b.x, dt, w.gxw, w.xclw, stream);
    if (w.dyw_ident && aligned16(b.dy)) p.tma_b = make_map(b.dy, w.ms_wg_b);
    else if (!dy_w_packed) pack_cl(b.dy, dt, w.gdy_w, w.dycl_w, stream);
    // fast chain kernels leave dWf zeroed behind them (it starts zeroed)
    static const bool memset_dwf = getenv("SYNO_TC_ZERO_FILL") != nullptr;  // A/B switch
    const bool fixup = w.wg_fixup && b.dw.size() == 1 && b.dw[0] && !memset_dwf;
    p.fix_out = fixup ? b.dw[0] : nullptr;
    if (!tp.fast_fold || memset_dwf) zero_fill(w.dwf, (size_t)tp.nwin() * tp.N * tp.C * sizeof(float), stream);
    gemm(p, w.bn_wg, w.t_wg[0], w.t_wg[1], w.t_wg[2], stream, "tc_gemm_wgrad", tp.flops);
    // chain rule through the fold, into each requested weight gradient
    Bindings cb = b;
    cb.stages = {w.dwf};
    if (!fixup) {
      static const bool fuse_side = getenv("SYNO_TC_NO_SIDE_CHAIN") == nullptr;
      std::vector<int> done(tp.chain.size(), 0);
      for (size_t j = 0; j < tp.chain.size(); ++j) {
        if (j >= b.dw.size() || !b.dw[j] || done[j]) continue;
        if (!tp.fast_fold) {
          run_stage(dt, tp.chain[j], cb, b.dw[j], false, stream);
          continue;
        }
        int side = -1;
        for (size_t j2 = 0; fuse_side && side < 0 && j2 < tp.chain.size(); ++j2)
          if (j2 < b.dw.size() && b.dw[j2] && !done[j2] && chain_side_ok(tp, (int)j, (int)j2)) side = (int)j2;
        done[j] = 1;
        if (side >= 0) done[side] = 1;
        bool zero = true;  // the last pass over dWf leaves it zeroed
        for (size_t j2 = 0; j2 < tp.chain.size(); ++j2)
          if (j2 < b.dw.size() && b.dw[j2] && !done[j2]) zero = false;
        chain_fast(tp, w, b, dt, (int)j, zero && !memset_dwf, stream, side);
      }
    }
  }
  if (fork) {
    cuda_check(cudaEventRecord(w.ev_join, w.side), "cudaEventRecord(join)");
    cuda_check(cudaStreamWaitEvent(stream, w.ev_join, 0), "cudaStreamWaitEvent(join)");
  }
  return true;
}

}  // namespace syno
