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
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>

#include "tc_gemm.cuh"

namespace syno {

using namespace tc;

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

// ---------------------------------------------------------------------------
// Packing kernels (bandwidth-bound layout transforms)
// ---------------------------------------------------------------------------

struct PackGeom {
  int64_t s_img, s_c, s_h, s_w;  // source element strides
  int32_t C, Hin, Win;           // source extents
  int32_t Sh, Sw;                // phase counts (strides)
  int32_t lo_h, lo_w, Hp, Wp;    // padded plane grid
  int32_t n_img;
  int32_t Cp;                    // channels-last pitch (multiple of 8)
  int64_t Fpitch;                // channel-major row pitch (multiple of 8)
};

// dst[plane][img][hp][wp][cp] (flat pixel f = ((plane*n_img + img)*Hp + hp)*Wp + wp),
// zero outside the source.  A block moves 32 consecutive flat pixels x 64
// channels through shared memory: lanes walk pixels for the NCHW reads
// (coalesced along w), 8 threads per pixel write 16-byte channel chunks.
template <typename TI>
__global__ void __launch_bounds__(256) pack_cl_kernel(const TI* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                                      PackGeom g, int64_t total_pix) {
  __shared__ __nv_bfloat16 tile[64][34];
  const int64_t f0 = (int64_t)blockIdx.x * 32;
  const int cb = blockIdx.y;
  const int t = threadIdx.x;
  {
    const int lane = t & 31, warp = t >> 5;
    const int64_t f = f0 + lane;
    bool inb = f < total_pix;
    const TI* row = src;
    if (inb) {
      const int wp = (int)(f % g.Wp);
      int64_t q = f / g.Wp;
      const int hp = (int)(q % g.Hp);
      q /= g.Hp;
      const int img = (int)(q % g.n_img);
      const int plane = (int)(q / g.n_img);
      const int hi = g.Sh * (hp - g.lo_h) + plane / g.Sw;
      const int wi = g.Sw * (wp - g.lo_w) + plane % g.Sw;
      inb = hi >= 0 && hi < g.Hin && wi >= 0 && wi < g.Win;
      row = src + img * g.s_img + (int64_t)hi * g.s_h + (int64_t)wi * g.s_w;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int cl = warp * 8 + k;
      const int c = cb * 64 + cl;
      float v = 0.f;
      if (inb && c < g.C) v = (float)row[c * g.s_c];
      tile[cl][lane] = __float2bfloat16(v);
    }
  }
  __syncthreads();
  const int w = t / 8, cc = (t % 8) * 8;
  const int64_t f = f0 + w;
  const int c0 = cb * 64 + cc;
  if (f < total_pix && c0 < g.Cp) {
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = tile[cc + k][w];
    *reinterpret_cast<uint4*>(dst + f * g.Cp + c0) = *reinterpret_cast<const uint4*>(v);
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
  int64_t Ep() const { return E + lo + hi; }
  int64_t dEp() const { return E + dlo + dhi; }
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
  double flops = 0;  // algorithmic FLOPs of one GEMM (= codegen.flops, unstaged, batch included)
  bool dgrad_ok = false;
  DevStage fold_fwd, fold_dgrad;
  std::vector<DevStage> chain;    // dW_j from the folded gradient
  std::vector<int64_t> w_numel;
  std::mutex mu;                  // guards ws
  std::map<std::pair<int, void*>, std::unique_ptr<struct TcWs>> ws;  // per (device, stream)
  int nwin() const { return dh.K * dw.K; }
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

TcPlanPtr tc_build(const Plan& plan, cudaStream_t stream) {
  TcPlan* raw = try_match(plan);
  if (!raw) return TcPlanPtr();
  TcPlanPtr tp(raw);
  tp->flops = (double)plan.flops_unstaged;
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

template <int BN>
static void launch_gemm(const TcGemmParams& p, unsigned grid, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};  // per-device bit
  constexpr int smem = smem_bytes<BN>();
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cuda_check(cudaFuncSetAttribute(tc_gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
               "cudaFuncSetAttribute(tc_gemm)");
    configured.fetch_or(bit);
  }
  note_launch();
  static unsigned long long* trace_buf = nullptr;
  const bool want_trace = getenv("SYNO_TC_TRACE") != nullptr;
  if (want_trace && !trace_buf) cuda_check(cudaMalloc(&trace_buf, 64 * sizeof(unsigned long long)), "trace");
  if (!want_trace) {
    tc_gemm_kernel<BN><<<grid, THREADS, smem, stream>>>(p);
  } else {
    TcGemmParams q = p;
    q.trace = trace_buf;
    cuda_check(cudaMemsetAsync(trace_buf, 0, 64 * sizeof(unsigned long long), stream), "trace memset");
    tc_gemm_kernel<BN><<<grid, THREADS, smem, stream>>>(q);
    unsigned long long h[64];
    cuda_check(cudaMemcpyAsync(h, trace_buf, sizeof(h), cudaMemcpyDeviceToHost, stream), "trace copy");
    cuda_check(cudaStreamSynchronize(stream), "trace sync");
    fprintf(stderr, "[tc trace BN=%d mode=%d tiles=%d grid=%u] setup %.2f us |", BN, p.mode,
            p.m_tiles * p.n_tiles * p.z_tiles, grid, (h[1] - h[0]) / 1e3);
    for (int i = 0; i < 14 && h[2 + i * 4]; ++i)
      fprintf(stderr, " t%d: prod %.2f mma %.2f epi %.2f-%.2f |", i, (h[2 + i * 4] - h[0]) / 1e3,
              h[3 + i * 4] ? (h[3 + i * 4] - h[0]) / 1e3 : -1.0, h[4 + i * 4] ? (h[4 + i * 4] - h[0]) / 1e3 : -1.0,
              h[5 + i * 4] ? (h[5 + i * 4] - h[0]) / 1e3 : -1.0);
    fprintf(stderr, "\n   tile0 windows: b_full seen at");
    for (int i = 40; i < 49; ++i) fprintf(stderr, " %.2f", h[i] ? (h[i] - h[0]) / 1e3 : -1.0);
    fprintf(stderr, "\n   tile0 windows: b_empty free at");
    for (int i = 50; i < 59; ++i) fprintf(stderr, " %.2f", h[i] ? (h[i] - h[0]) / 1e3 : -1.0);
    fprintf(stderr, "\n   tile1 windows 1-4 cycles (wait, issue, commit):");
    for (int i = 59; i < 63; ++i)
      fprintf(stderr, " (%llu, %llu, %llu)", h[i] & 0xFFFFF, (h[i] >> 20) & 0xFFFFF, (h[i] >> 40) & 0xFFFFF);
    fprintf(stderr, "\n");
  }
  cuda_check(cudaGetLastError(), "tc_gemm_kernel");
}

static int sm_count() {
  int dev = 0, n = 148;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
  return n;
}

// Persistent launch: one CTA per SM walks the (n fastest, m, z) tile grid.
static void gemm(TcGemmParams& p, int bn, int m_tiles, int n_tiles, int z_tiles, cudaStream_t stream,
                 const char* name, double flops) {
  p.m_tiles = m_tiles;
  p.n_tiles = n_tiles;
  p.z_tiles = z_tiles;
  const int a_region = bn == 64 ? a_region_bytes<64>() : bn == 128 ? a_region_bytes<128>() : a_region_bytes<256>();
  p.a_stages = std::max(1, std::min(8, a_region / p.a_stage_bytes));
  const int64_t tiles = (int64_t)m_tiles * n_tiles * z_tiles;
  if (tiles <= 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, sm_count());
  const int id = prof_begin(name, flops, 0.0, stream);
  if (bn == 64) launch_gemm<64>(p, grid, stream);
  else if (bn == 128) launch_gemm<128>(p, grid, stream);
  else launch_gemm<256>(p, grid, stream);
  prof_end(id, stream);
}

static int mgroup_of(int bn) { return bn == 64 ? mgroup<64>() : bn == 128 ? mgroup<128>() : mgroup<256>(); }

static int pick_bn(int n) { return n <= 64 ? 64 : n <= 128 ? 128 : 256; }

static void pack_cl(const void* src, DType dt, const PackGeom& g, __nv_bfloat16* dst, cudaStream_t stream) {
  const int64_t pix = (int64_t)g.Sh * g.Sw * g.n_img * g.Hp * g.Wp;
  dim3 grid((unsigned)((pix + 31) / 32), (unsigned)((g.Cp + 63) / 64));
  const double src_elems = (double)g.n_img * g.C * g.Hin * g.Win;
  const int id = prof_begin("pack_cl", 0.0, src_elems * (dt == DT_BF16 ? 2 : 4) + (double)pix * g.Cp * 2, stream);
  note_launch();
  if (dt == DT_BF16) pack_cl_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>((const __nv_bfloat16*)src, dst, g, pix);
  else pack_cl_kernel<float><<<grid, 256, 0, stream>>>((const float*)src, dst, g, pix);
  cuda_check(cudaGetLastError(), "pack_cl_kernel");
  prof_end(id, stream);
}

static PackGeom geom(const TcPlan& tp, bool dy_side, bool grad_pad) {
  PackGeom g{};
  g.n_img = tp.n_img;
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
  const int64_t F = (int64_t)g.n_img * g.Hp * g.Wp;
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

static void rows_schedule(TcGemmParams& p, std::vector<std::vector<Win>> groups, int bn) {
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
  }
  p.n_win = n;
  const int G = bn >= 256 ? 1 : 256 / bn;  // tc::mgroup<BN>()
  p.a_rows = (G * BM + span + 63) / 64 * 64;
  p.a_tx = (uint32_t)p.a_rows * BK * 2;
  p.a_stage_bytes = (int)p.a_tx;
  p.b_tx = (uint32_t)bn * BK * 2;
  p.base_mode = base_mode();
  p.dbg = getenv("SYNO_TC_DEBUG") ? atoi(getenv("SYNO_TC_DEBUG")) : 0;
}

// Per (device, stream) workspace of an operator: packed operands, folded
// weights, the fp32 grad-weight accumulator and the fully built GEMM
// parameters (their TMA maps point into the workspace, so they are encoded
// once).  Steady-state calls only launch kernels: no allocation, no host
// synchronisation, CUDA-graph capturable.
struct TcWs {
  __nv_bfloat16 *xcl = nullptr, *wf = nullptr, *dycl_g = nullptr, *dycl_w = nullptr, *wt = nullptr;
  float* dwf = nullptr;
  PackGeom gx{}, gdy_g{}, gdy_w{};
  bool share_dy = false;
  TcGemmParams fwd, dg, wg;
  int bn_fwd = 0, bn_dg = 0, bn_wg = 0;
  int t_fwd[3] = {0, 0, 0}, t_dg[3] = {0, 0, 0}, t_wg[3] = {0, 0, 0};
  std::vector<void*> owned;
  ~TcWs() {
    for (void* q : owned) cudaFree(q);
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
  return a.lo_h == b.lo_h && a.lo_w == b.lo_w && a.Hp == b.Hp && a.Wp == b.Wp;
}

template <typename T>
static T* ws_alloc(TcWs& w, size_t count) {
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc(tc workspace)");
  w.owned.push_back(p);
  return static_cast<T*>(p);
}

static void build_ws(TcPlan& tp, TcWs& w) {
  w.gx = geom(tp, false, false);
  const int planes = w.gx.Sh * w.gx.Sw;
  const int64_t F = (int64_t)w.gx.n_img * w.gx.Hp * w.gx.Wp;
  w.xcl = ws_alloc<__nv_bfloat16>(w, (size_t)planes * F * tp.Cp);
  w.wf = ws_alloc<__nv_bfloat16>(w, (size_t)tp.nwin() * tp.N * tp.Cp);

  // ---- forward: y = sum_win sum_ci Xcl[plane][flat + shift] Wf[win][n][ci]
  {
    const int bn = pick_bn(tp.N);
    TcGemmParams& p = w.fwd;
    memset(&p, 0, sizeof(p));
    p.mode = MODE_ROWS;
    p.n_cblocks = (tp.Cp + BK - 1) / BK;
    std::vector<std::vector<Win>> groups(1);
    for (int rh = 0; rh < tp.dh.K; ++rh)
      for (int rw = 0; rw < tp.dw.K; ++rw)
        groups[0].push_back({tp.dh.delta(rh) * w.gx.Wp + tp.dw.delta(rw), tp.dh.phi(rh) * w.gx.Sw + tp.dw.phi(rw),
                             rh * tp.dw.K + rw});
    rows_schedule(p, groups, bn);
    p.tma_a = make_map(w.xcl, tp.Cp, F, planes, tp.Cp, F * tp.Cp, 64);
    p.tma_b = make_map(w.wf, tp.Cp, tp.N, tp.nwin(), tp.Cp, (int64_t)tp.N * tp.Cp, bn);
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
    p.out_kind = OUT_BF16;
    p.scale = (float)tp.scale;
    w.bn_fwd = bn;
    w.t_fwd[0] = (int)((F + (int64_t)mgroup_of(bn) * BM - 1) / ((int64_t)mgroup_of(bn) * BM));
    w.t_fwd[1] = (tp.N + bn - 1) / bn;
    w.t_fwd[2] = 1;
  }

  // ---- backward operands
  w.gdy_g = geom(tp, true, true);
  w.gdy_w = geom(tp, true, false);
  w.share_dy = same_grid(w.gdy_g, w.gdy_w);
  const int64_t Fg = (int64_t)w.gdy_g.n_img * w.gdy_g.Hp * w.gdy_g.Wp;
  if (tp.dgrad_ok) {
    w.dycl_g = ws_alloc<__nv_bfloat16>(w, (size_t)Fg * tp.Np);
    w.wt = ws_alloc<__nv_bfloat16>(w, (size_t)tp.nwin() * tp.C * tp.Np);
  }
  w.dycl_w = (w.share_dy && w.dycl_g) ? w.dycl_g : ws_alloc<__nv_bfloat16>(w, (size_t)F * tp.Np);
  w.dwf = ws_alloc<float>(w, (size_t)tp.nwin() * tp.N * tp.C);

  // ---- grad-input: one group per output phase (psi_h, psi_w); its windows have phi(r) == psi
  if (tp.dgrad_ok) {
    const int bn = pick_bn(tp.C);
    TcGemmParams& p = w.dg;
    memset(&p, 0, sizeof(p));
    p.mode = MODE_ROWS;
    p.n_cblocks = (tp.Np + BK - 1) / BK;
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
    rows_schedule(p, groups, bn);
    p.tma_a = make_map(w.dycl_g, tp.Np, Fg, 1, tp.Np, Fg * tp.Np, 64);
    p.tma_b = make_map(w.wt, tp.Np, tp.C, tp.nwin(), tp.Np, (int64_t)tp.C * tp.Np, bn);
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
    p.out_kind = OUT_BF16;
    p.scale = (float)tp.scale;
    w.bn_dg = bn;
    w.t_dg[0] = (int)((Fg + (int64_t)mgroup_of(bn) * BM - 1) / ((int64_t)mgroup_of(bn) * BM));
    w.t_dg[1] = (tp.C + bn - 1) / bn;
    w.t_dg[2] = Sh * Sw;
  }

  // ---- grad-weight: both operands channels-last over the forward's flat
  // padded grid, read MN-major (K = pixel rows): a window is a row shift
  {
    // M = (window, 64-channel block of C_in) pairs, N = C_out, K = pixel rows
    const int bn = pick_bn(tp.N);
    TcGemmParams& p = w.wg;
    memset(&p, 0, sizeof(p));
    p.tma_a = make_map(w.xcl, tp.Cp, F, planes, tp.Cp, F * tp.Cp, 64);
    p.tma_b = make_map(w.dycl_w, tp.Np, F, 1, tp.Np, F * tp.Np, 64);
    p.mode = MODE_WGRAD;
    p.n_cblocks = (int)((F + BK - 1) / BK);
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
    int ksplit = std::max(1, (4 * sm_count()) / std::max(1, m_tiles * n_tiles));
    ksplit = std::min(ksplit, std::max(1, p.n_cblocks / 4));
    p.ksplit = ksplit;
    p.m_ext = tp.C;
    p.n_ext = tp.N;
    p.o_m = 1;
    p.o_n = tp.C;
    for (int wi = 0; wi < tp.nwin(); ++wi) p.g_out_off[wi] = (int64_t)wi * tp.N * tp.C;
    p.out_kind = OUT_F32_ATOMIC;
    p.scale = (float)tp.scale;
    p.out = w.dwf;
    p.a_rows = 64;
    p.a_tx = (uint32_t)BM * BK * 2;
    p.a_stage_bytes = BM * BK * 2;
    p.b_tx = (uint32_t)bn * BK * 2;
    w.bn_wg = bn;
    w.t_wg[0] = m_tiles;
    w.t_wg[1] = n_tiles;
    w.t_wg[2] = ksplit;
  }
}

static TcWs& workspace(TcPlan& tp, cudaStream_t stream) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(tp.mu);
  auto key = std::make_pair(dev, (void*)stream);
  auto it = tp.ws.find(key);
  if (it != tp.ws.end()) return *it->second;
  auto w = std::make_unique<TcWs>();
  build_ws(tp, *w);
  TcWs& ref = *w;
  tp.ws[key] = std::move(w);
  return ref;
}

bool tc_forward(TcPlan& tp, DType dt, const Bindings& b, cudaStream_t stream) {
  if (dt != DT_BF16) return false;
  TcWs& w = workspace(tp, stream);
  pack_cl(b.x, dt, w.gx, w.xcl, stream);
  run_stage(dt, tp.fold_fwd, b, w.wf, false, stream);
  TcGemmParams& p = w.fwd;
  p.out = b.y;
  gemm(p, w.bn_fwd, w.t_fwd[0], w.t_fwd[1], w.t_fwd[2], stream, "tc_gemm_fwd", tp.flops);
  return true;
}

bool tc_backward(TcPlan& tp, DType dt, const Bindings& b, cudaStream_t stream) {
  if (dt != DT_BF16) return false;
  if (b.dx && !tp.dgrad_ok) return false;
  TcWs& w = workspace(tp, stream);
  bool any_w = false;
  for (auto* q : b.dw) any_w = any_w || q;
  bool dy_w_packed = false;
  if (b.dx) {
    pack_cl(b.dy, dt, w.gdy_g, w.dycl_g, stream);
    dy_w_packed = w.share_dy;
    run_stage(dt, tp.fold_dgrad, b, w.wt, false, stream);
    TcGemmParams& p = w.dg;
    p.out = b.dx;
    gemm(p, w.bn_dg, w.t_dg[0], w.t_dg[1], w.t_dg[2], stream, "tc_gemm_dgrad", tp.flops);
  }
  if (any_w) {
    pack_cl(b.x, dt, w.gx, w.xcl, stream);
    if (!dy_w_packed) pack_cl(b.dy, dt, w.gdy_w, w.dycl_w, stream);
    cuda_check(cudaMemsetAsync(w.dwf, 0, (size_t)tp.nwin() * tp.N * tp.C * sizeof(float), stream), "memset(dWf)");
    gemm(w.wg, w.bn_wg, w.t_wg[0], w.t_wg[1], w.t_wg[2], stream, "tc_gemm_wgrad", tp.flops);
    // chain rule through the fold, into each requested weight gradient
    Bindings cb = b;
    cb.stages = {w.dwf};
    for (size_t j = 0; j < tp.chain.size(); ++j) {
      if (j >= b.dw.size() || !b.dw[j]) continue;
      run_stage(dt, tp.chain[j], cb, b.dw[j], false, stream);
    }
  }
  return true;
}

}  // namespace syno
