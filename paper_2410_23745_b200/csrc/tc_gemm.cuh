// tcgen05 implicit-GEMM kernel (sm_100a): TMA -> SMEM (128B swizzle) ->
// tcgen05.mma (bf16 x bf16 -> fp32 in TMEM) -> tcgen05.ld -> masked affine
// epilogue.  The operands are fetched by TMA from packed operand layouts
// (tc.cu); the k schedule and the epilogue address map come from
// TcGemmParams, so one kernel serves forward (windows x channel blocks),
// grad-input (flipped windows, one group per output phase) and grad-weight
// (split-K over pixel rows, one window per group, MN-major operands).
//
// MODE_ROWS loads ONE halo tile of A per (phase plane, channel block) --
// the 128 output rows plus the span of the window row shifts -- and
// addresses every window as a row-shifted view of it (descriptor start
// address + base offset), so A crosses L2 once instead of once per window.
//
// Persistent: a CTA walks tiles t = blockIdx.x, +gridDim.x, ...  Warp roles
// (320 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer
// (one lane), warps 2..9 = epilogue (TMEM lane quarter = warp % 4; the two
// warps of a quarter take alternate 32-column chunks).  The
// accumulator is double-buffered in TMEM so the epilogue of tile i overlaps
// the main loop of tile i+1.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

namespace syno {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;                 // one 128-byte swizzle row of bf16
constexpr int MAXWIN = 64;
constexpr int MAXCHUNK = 32;
constexpr int EPI_WARPS = 8;  // two per TMEM lane quarter, splitting the column chunks
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr int RING_BYTES = 192 * 1024;  // A ring (halo / dy tiles) + B ring
// Epilogue staging (CFG 0 / pair): per epilogue warp a 32-row x 32-column
// bf16 block with an 80-byte row pitch.  Outputs whose N dim is contiguous
// (QKV-like) are transposed through it so that each warp store writes
// 8 rows x 64 contiguous bytes instead of 32 rows x 16 bytes: the per-lane
// row stores cost 32 L1 wavefronts per instruction and made the epilogue,
// not the MMAs, the limit of such GEMMs (1x1 K=64 launches: 48 us store-bound).
constexpr int EPI_ROW_WORDS = 20;
constexpr int EPI_STAGE_BYTES = 8 * 32 * EPI_ROW_WORDS * 4;

// MODE_ROWS processes G = 256/BN consecutive 128-row M tiles per step: one
// contiguous A halo and one B tile per window feed G accumulators, cutting
// the operand traffic per output row by ~G (B is the small weight tile that
// every M tile needs).  Four B stages; the rest of the ring is A.
template <int BN>
__host__ __device__ constexpr int mgroup() {
  return BN >= 256 ? 1 : 256 / BN;
}
// CFG 0: one CTA per SM (192 KB ring, 512 TMEM columns, G up to mgroup).
// CFG 1: two CTAs per SM (104 KB ring, <= 256 TMEM columns, G = 1): the
// second CTA hides the first one's fixed costs (setup, first loads,
// epilogue tail) and the next kernel's CTAs can start beside a tail CTA.
// CFG 2 (CTA pair, BN = 256, MODE_ROWS): a cluster of two CTAs on one TPC
// computes a 256 x 256 tile with tcgen05.mma.cta_group::2 issued by the
// leader.  Each CTA stages its own 128-row A halo tile and HALF of the B
// tile (128 of the 256 N rows), so one 256 x 256 x 64 k-step moves 32 KB
// per SM from L2 instead of 48 KB for a 128 x 256 tile, and the ring holds
// six k-steps instead of four.  Each CTA's TMEM holds its own 128 rows.
constexpr int CFG_PAIR = 2;
template <int CFG>
__host__ __device__ constexpr int ring_bytes() {
  return CFG == 1 ? 104 * 1024 : RING_BYTES;
}
template <int BN, int CFG>
__host__ __device__ constexpr int gmax() {
  return CFG ? 1 : mgroup<BN>();
}
template <int BN, int CFG = 0>
__host__ __device__ constexpr int b_stages() {
  return CFG == CFG_PAIR ? 6 : CFG && BN >= 128 ? 3 : 4;
}
// B rows one CTA stages per k-step (the pair splits N)
template <int BN, int CFG = 0>
__host__ __device__ constexpr int b_rows() {
  return CFG == CFG_PAIR ? BN / 2 : BN;
}
template <int BN, int CFG = 0>
__host__ __device__ constexpr int a_region_bytes() {
  return ring_bytes<CFG>() - b_stages<BN, CFG>() * b_rows<BN, CFG>() * BK * 2;
}

enum Mode : int32_t {
  MODE_ROWS = 0,   // A rows = flat padded pixels (halo tile, window = row shift); k = (chunk, cblock, window)
  // M = (window, 64-channel block of C_in) pairs, two per tile; N = C_out;
  // k = pixel rows; MN-major channels-last tiles of x (row-shifted per
  // window) and dy.  Output dWf[window][co][ci], fp32 split-K atomics that
  // coalesce along ci.
  MODE_WGRAD = 1,
};

constexpr int MAXPAIR = 160;

enum OutKind : int32_t { OUT_BF16 = 0, OUT_F32 = 1, OUT_F32_ATOMIC = 2 };

struct alignas(64) TcGemmParams {
  CUtensorMap tma_a;   // 3-D: [K elems][rows][plane]
  CUtensorMap tma_b;   // 3-D: [K elems][rows][plane]
  int32_t mode;
  int32_t n_cblocks;   // MODE_ROWS: channel blocks of 64; MODE_WGRAD: pixel blocks per window
  int32_t n_win;
  int32_t ksplit;      // MODE_WGRAD split of the pixel blocks
  int32_t rsplit;      // MODE_ROWS split of the channel blocks (>1: fp32 atomic output)
  int32_t G;           // MODE_ROWS M tiles per step (<= gmax<BN, CFG>(); fewer for small problems)
  int32_t cfg;         // host-side: kernel configuration (CFG template argument) to launch
  // MODE_ROWS, one N tile and one channel block: the B tiles of all b_res
  // windows stay resident in shared memory (loaded once per CTA), so the
  // window loop issues no B loads and no per-window commits
  int32_t b_res;
  // MODE_ROWS: B read MN-major (64-wide N atoms of 64 K rows, 8 KB apart):
  // a QKV-like grad-input reads the [N_out][C] weight in place, no transpose
  int32_t b_mn;
  int32_t a_shift[MAXWIN];   // MODE_ROWS: row shift of A per window; MODE_WGRAD: B row (pixel) shift
  int32_t a_plane[MAXWIN];   // MODE_WGRAD: plane (phase) of x per window
  int32_t b_plane[MAXWIN];   // MODE_ROWS: B plane (packed weight window) per window
  // MODE_ROWS chunks: windows [chunk_w0, chunk_w1) share A plane chunk_plane and min shift chunk_pmin
  int32_t chunk_plane[MAXCHUNK], chunk_w0[MAXCHUNK], chunk_w1[MAXCHUNK], chunk_pmin[MAXCHUNK];
  int32_t g_chunk0[8], g_chunk1[8];  // chunk range of each group (blockIdx-level z)
  int32_t g_nwin[8];                 // windows of each group (host: sum of its chunks' windows)
  int32_t k_per;                     // channel blocks (MODE_ROWS) / pixel blocks (MODE_WGRAD) per split
  int32_t kq_last;                   // MODE_ROWS: 16-wide K steps holding data in the last channel block
                                     // (a 3-channel stem padded to 8 issues 1 MMA per window, not 4)
  // MODE_WGRAD pairs: M rows [64h, 64h+64) of tile mt are pair 2*mt+h = (window, channel block)
  int32_t n_pairs;
  int16_t pair_win[MAXPAIR], pair_cb[MAXPAIR];
  int64_t g_out_off[MAXWIN];
  int32_t a_rows;       // MODE_ROWS: halo rows per A stage (G*128 + span, multiple of 64)
  int32_t a_stage_bytes;  // smem slot of one A stage (multiple of 1024)
  int32_t a_stages;
  uint32_t a_tx, b_tx;  // transaction bytes of one A / B stage
  int32_t base_mode;    // 1: set the descriptor base offset for row-shifted A views
  int32_t dbg;          // profiling switches: 1 = skip epilogue stores, 2 = skip MMAs, 4/8 = skip A/B loads
  unsigned long long* trace;  // profiling: %globaltimer stamps of CTA 0 (null = off)
  // tile grid: t -> (nt fastest, then mt, then z)
  int32_t m_tiles, n_tiles, z_tiles;
  // epilogue: row index r of the M tile -> output coordinates
  //   MODE_ROWS: flat = mtile*128 + r; (img, hp, wp) by Hp, Wp; h = hp - lo_h ...
  //   MODE_WGRAD: row = C_out index
  int32_t Hp, Wp, lo_h, lo_w, H, W, n_img;
  int64_t o_img, o_h, o_w, o_n, o_m;
  int32_t m_ext, n_ext;
  // MODE_WGRAD split-K fixup: the last split to finish an output tile turns
  // the tile's fp32 sums into the weight gradient itself (single-weight
  // operators whose fold is a pure permutation), replacing the chain-rule
  // launch; it also re-zeroes the tile's accumulator for the next call
  void* fix_out;                // dW (null: off)
  unsigned* fix_cnt;            // per (m_tile, n_tile) arrival counters, zero between calls
  int64_t fix_win_off[MAXWIN];  // dW offset of window w
  int64_t fix_s_ci, fix_s_co;   // dW strides of ci and co
  int32_t fix_f32;
  int32_t out_kind;
  float scale;
  void* out;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
              );
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef SYNO_MBAR_SUSPEND
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)
     );
#else
  // spin on the non-suspending probe: the wait is on the critical path of
  // the producer -> MMA -> epilogue hand-offs
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity));
#endif
}

// The issue-path helpers (waits, arrives, TMA, commits) carry no "memory"
// clobber: they are ordered among themselves as volatile asm, the producer
// and MMA warps touch memory only through them, and a clobber would force
// every kernel parameter to be re-read from the constant bank after each
// one (measured: dependent LDCU chains in the per-k-step loops).
//
// Long waits (the epilogue warps waiting a whole tile for the accumulator):
// the suspending probe with a time hint parks the warp instead of spinning,
// so eight idle epilogue warps do not compete with the producer / MMA warps
// for issue slots and the barrier unit.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x10000)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
     );
}

// CTA-pair helpers (CFG_PAIR)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t n_clusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (same offset) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar));
}
// TMA load into this CTA's shared memory whose completion is signalled on an
// mbarrier of either CTA of the pair (the leader's full barrier)
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t cluster_bar, int c0,
                                                 int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(cluster_bar), "r"(c0), "r"(c1), "r"(c2)
     );
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// MMA from the low words of two K-major SWIZZLE_128B descriptors (start
// address >> 4 | LBO 1 << 16); the high word (SBO 1024 B, version, swizzle)
// is the constant DESC_HI, so the issue loop advances 32-bit words only.
constexpr uint32_t DESC_HI = (1024u >> 4) | (1u << 14) | (2u << 29);
__device__ __forceinline__ uint32_t desc_lo(uint32_t smem_addr) { return (smem_addr >> 4) | (1u << 16); }
template <bool PAIR>
__device__ __forceinline__ void mma_lo(uint32_t tmem_d, uint32_t a_lo, uint32_t b_lo, uint32_t idesc, uint32_t acc) {
  if constexpr (PAIR)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
        "mov.b64 da, {%1, %5};\n\tmov.b64 db, {%2, %5};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(acc), "n"(DESC_HI));
  else
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
        "mov.b64 da, {%1, %5};\n\tmov.b64 db, {%2, %5};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(acc), "n"(DESC_HI));
}

// commit the leader's MMAs to the same barrier in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
     );
}

// K-major, 128-byte swizzle smem descriptor (canonical ((8,m),(T,2)) : ((8T,SBO),(1,T))),
// starting `row` 128-byte rows into a 1024-byte aligned tile.
__device__ __forceinline__ uint64_t sw128_desc(const void* smem, int row = 0, int base_mode = 0) {
  uint64_t addr = smem_u32(smem) + (uint32_t)row * 128u;
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFF;              // start address
  d |= (uint64_t)(16 >> 4) << 16;         // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                 // sm100 descriptor version
  if (base_mode) d |= (uint64_t)((addr >> 7) & 7) << 49;  // swizzle phase of an unaligned start
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

// Issued by the whole (converged) warp with warp-uniform operands; one
// elected lane executes the tcgen05 instruction.  Keeping the loop and the
// operand math warp-wide lets ptxas hold descriptors in uniform registers
// instead of wrapping every issue in an R2UR/ELECT waterfall loop.
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
     );
}

__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(e));
  return e != 0;
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

struct TileInfo {
  int mt, nt, g, ks, kb0, nkb;
  int cb0, cb1;  // MODE_ROWS channel-block range of this split
};

// Persistent tile walk without per-tile integer division: the first tile
// and the stride are decomposed once into (n, m, z) digits and each step
// adds the stride's digits with carries.  The per-tile k-step count and the
// split widths come precomputed from the host (g_nwin, k_per).
struct TileWalk {
  int nt, mt, z, dn, dm, dz;
  __device__ __forceinline__ void init(const TcGemmParams& p, int t0, int step) {
    nt = t0 % p.n_tiles;
    int q = t0 / p.n_tiles;
    mt = q % p.m_tiles;
    z = q / p.m_tiles;
    dn = step % p.n_tiles;
    q = step / p.n_tiles;
    dm = q % p.m_tiles;
    dz = q / p.m_tiles;
  }
  __device__ __forceinline__ void next(const TcGemmParams& p) {
    nt += dn;
    int c = 0;
    if (nt >= p.n_tiles) {
      nt -= p.n_tiles;
      c = 1;
    }
    mt += dm + c;
    c = 0;
    if (mt >= p.m_tiles) {
      mt -= p.m_tiles;
      c = 1;
    }
    z += dz + c;
  }
};

__device__ __forceinline__ TileInfo tile_info(const TcGemmParams& p, const TileWalk& w) {
  TileInfo ti;
  ti.nt = w.nt;
  ti.mt = w.mt;
  const int z = w.z;
  if (p.mode == MODE_ROWS) {
    const int rs = p.rsplit > 1 ? p.rsplit : 1;
    ti.g = rs == 1 ? z : z / rs;
    ti.ks = z - ti.g * rs;
    const int per = p.k_per;
    ti.cb0 = ti.ks * per;
    ti.cb1 = min(p.n_cblocks, ti.cb0 + per);
    ti.kb0 = 0;
    ti.nkb = p.g_nwin[ti.g] * max(0, ti.cb1 - ti.cb0);  // MMA k-steps (one per window x channel block)
  } else {
    ti.cb0 = ti.cb1 = 0;
    ti.g = p.ksplit == 1 ? z : z / p.ksplit;
    ti.ks = z - ti.g * p.ksplit;
    const int per = p.k_per;
    ti.kb0 = ti.ks * per;
    const int kb1 = min(p.n_cblocks, ti.kb0 + per);
    ti.nkb = kb1 > ti.kb0 ? kb1 - ti.kb0 : 0;
  }
  return ti;
}

// Ring position: slot index and phase parity, advanced incrementally (a
// runtime-sized ring would otherwise cost an integer division per k-step on
// the latency-critical producer / MMA loops).
struct Ring {
  int s = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ int slot(int) const { return s; }
  __device__ __forceinline__ uint32_t phase(int) const { return ph; }
  __device__ __forceinline__ void next(int n) {
    if (++s == n) {
      s = 0;
      ph ^= 1u;
    }
  }
};

template <int BN, int MODE, int CFG>
__global__ void __launch_bounds__(THREADS, CFG == 1 ? 2 : 1) tc_gemm_kernel(const __grid_constant__ TcGemmParams p) {
  pdl_trigger();
  constexpr bool PAIR = CFG == CFG_PAIR;
  static_assert(!PAIR || BN == 256 || (BN == 128 && MODE == MODE_ROWS), "CTA pair: BN = 256, or 128 (rows mode)");
  // KM: 64-element K blocks per ring stage.  The pair grad-weight kernel
  // stages two (3 x 64 KB per CTA), halving the barrier hand-offs per MAC.
  constexpr int KM = PAIR && MODE == MODE_WGRAD ? 2 : 1;
  constexpr int BSTAGES = KM == 2 ? 3 : b_stages<BN, CFG>();
  constexpr int B_BYTES = b_rows<BN, CFG>() * BK * 2 * KM;
  static_assert(BSTAGES * B_BYTES == b_stages<BN, CFG>() * b_rows<BN, CFG>() * BK * 2, "B ring size");
  constexpr int G = gmax<BN, CFG>();
  constexpr uint32_t ACC_COLS = G * BN;          // one accumulator buffer: G sub-tiles
  constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;   // double-buffered (512 for CFG 0)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  const int b_res = MODE == MODE_ROWS ? p.b_res : 0;
  uint8_t* sb = b_res ? smem + ring_bytes<CFG>() - b_res * B_BYTES : smem + a_region_bytes<BN, CFG>();
  uint64_t* a_full = reinterpret_cast<uint64_t*>(smem + ring_bytes<CFG>());
  uint64_t* a_empty = a_full + 8;
  uint64_t* b_full = a_empty + 8;
  uint64_t* b_empty = b_full + BSTAGES;
  uint64_t* tfull = b_empty + BSTAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  volatile uint32_t* fix_last = tmem_slot + 1;  // MODE_WGRAD fixup: this CTA finished the tile last

  // warp index through a shuffle: the compiler then knows it is warp-uniform,
  // so each role's loops run on the uniform datapath (descriptors, ring
  // counters and parameter reads in uniform registers, no R2UR per MMA)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int n_tiles_total = p.m_tiles * p.n_tiles * p.z_tiles;
  const int AST = p.a_stages;
  // profiling switches (SYNO_TC_DEBUG) are compiled in only with `make DBG=1`:
  // their runtime tests cost the issue loops measurably
#ifdef SYNO_TC_DBG_SWITCHES
  const int dbg = p.dbg;
#else
  constexpr int dbg = 0;
#endif
  // CTA pair: both CTAs walk the same pair tiles (m_tiles counts pairs of
  // 128-row M tiles; this CTA takes M tile 2 * pair + rank)
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int t_first = PAIR ? (int)cluster_id_x() : (int)blockIdx.x;
  const int t_step = PAIR ? (int)n_clusters_x() : (int)gridDim.x;
  auto tinfo = [&](const TileWalk& w) {
    TileInfo ti = tile_info(p, w);
    if (PAIR) ti.mt = 2 * ti.mt + (int)rank;
    return ti;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < AST; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < BSTAGES; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 2 * EPI_WARPS : EPI_WARPS);  // pair: both CTAs' epilogues arrive at the leader
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // the peer's barriers are initialised before any remote signal
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // barrier init, TMEM allocation and the tensormap prefetch overlapped the
  // previous kernel; from here on global memory is touched
  pdl_wait();
  // profiling: event log of every CTA on SM 0.  trace[0] counts CTAs; CTA
  // slot s owns entries [64 + s*1024, +1024): 256 per role (start, producer,
  // MMA, epilogue), each entry (globaltimer, kind | tile << 8 | w << 24 |
  // cta << 40); the roles write with private counters (no atomics in the loops).
  // Compiled in only with -DSYNO_TC_TRACE_EVENTS (`make TRACE=1`): the
  // checks cost the latency-critical issue loops ~15% otherwise.
#ifdef SYNO_TC_TRACE_EVENTS
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const bool tr = p.trace != nullptr && smid == 0;
  __shared__ uint32_t tr_slot;
  if (tr && threadIdx.x == 0) tr_slot = (uint32_t)atomicAdd(p.trace, 1ull);
  __syncthreads();
  uint32_t tr_n = 0;
  const int tr_role = warp == 0 ? 1 : warp == 1 ? 2 : 3;
#else
  constexpr bool tr = false;
  constexpr uint32_t tr_slot = 0;
  uint32_t tr_n = 0;
  constexpr int tr_role = 0;
#endif
  auto ev = [&](int kind, int tile, int w) {
    if (tr && tr_slot < 7) {
      // SM cycle counter (every traced CTA runs on SM 0); the viewer converts at 1.965 GHz
      const unsigned long long t = clock64();
      const int role = threadIdx.x == 0 && kind == 0 ? 0 : tr_role;
      if (tr_n < 127) {
        unsigned long long* e = p.trace + 64 + tr_slot * 1024 + role * 256 + tr_n * 2;
        e[0] = t;
        e[1] = (unsigned long long)kind | ((unsigned long long)(tile & 0xFFFF) << 8) |
               ((unsigned long long)(w & 0xFFFF) << 24) | ((unsigned long long)blockIdx.x << 40);
        ++tr_n;
      }
    }
  };
  if (threadIdx.x == 0) {
    ev(0, 0, 0);
    tr_n = 0;
  }

  // profiling switches 1024 (MMA warp ignores every barrier) + 2048 (the other
  // roles do nothing): the bare MMA issue stream over the kernel's tiles
  const bool bare = (dbg & 1024) && (dbg & 2048);
  if (bare && warp != 1) {
  } else if (warp == 0) {
    // ---------------- TMA producer: the whole warp walks the schedule, one
    // elected lane issues (operands stay warp-uniform).
    if (elect_one()) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tma_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tma_b)) : "memory");
    }
    __syncwarp();
    Ring ra, rb;
    uint32_t pcount = 0;
    if (b_res && blockIdx.x < n_tiles_total) {
      if (elect_one()) {
        if (dbg & 8) {
          mbar_arrive(&b_full[0]);
        } else {
          mbar_expect_tx(&b_full[0], p.b_tx * (uint32_t)b_res);
          for (int w = 0; w < b_res; ++w) tma_load_3d(sb + w * B_BYTES, &p.tma_b, &b_full[0], 0, 0, p.b_plane[w]);
        }
      }
      __syncwarp();
    }
    TileWalk tw;
    tw.init(p, t_first, t_step);
    for (int t = t_first; t < n_tiles_total; t += t_step, ++pcount, tw.next(p)) {
      const TileInfo ti = tinfo(tw);
      if constexpr (MODE == MODE_ROWS) {
        for (int c = p.g_chunk0[ti.g]; c < p.g_chunk1[ti.g]; ++c) {
          for (int cb = ti.cb0; cb < ti.cb1; ++cb) {
            // one halo tile of A for this plane and channel block
            const int as = ra.slot(AST);
            mbar_wait(&a_empty[as], ra.phase(AST) ^ 1u);
            if (lane == 0) ev(1, (int)pcount, c * 64 + cb);  // A slot free, load issued
            const int row0 = ti.mt * p.G * BM + p.chunk_pmin[c];
            const int nbox = p.a_rows / 64;
            if (elect_one()) {
              if constexpr (PAIR) {
                // both halves land on the leader's barrier
                if (rank == 0) mbar_expect_tx(&a_full[as], 2 * p.a_tx);
                const uint32_t bar = peer_addr(&a_full[as], 0);
                #pragma unroll 1
                for (int j = 0; j < nbox; ++j)
                  tma_load_3d_pair(sa + as * p.a_stage_bytes + j * 8192, &p.tma_a, bar, cb * BK, row0 + 64 * j,
                                   p.chunk_plane[c]);
              } else if (dbg & 4) {
                mbar_arrive(&a_full[as]);
              } else {
                mbar_expect_tx(&a_full[as], p.a_tx);
                #pragma unroll 1
                for (int j = 0; j < nbox; ++j)
                  tma_load_3d(sa + as * p.a_stage_bytes + j * 8192, &p.tma_a, &a_full[as], cb * BK, row0 + 64 * j,
                              p.chunk_plane[c]);
              }
            }
            __syncwarp();
            ra.next(AST);
            for (int w = p.chunk_w0[c]; w < p.chunk_w1[c] && !b_res; ++w) {
              const int bs = rb.slot(BSTAGES);
              mbar_wait(&b_empty[bs], rb.phase(BSTAGES) ^ 1u);
              if (lane == 0) ev(2, (int)pcount, w);  // B slot free, load issued
              if (elect_one()) {
                if constexpr (PAIR) {
                  // this CTA's half of the N rows
                  if (rank == 0) mbar_expect_tx(&b_full[bs], 2 * p.b_tx);
                  if (p.b_mn) {
#pragma unroll 1
                    for (int h = 0; h < BN / 128; ++h)
                      tma_load_3d_pair(sb + bs * B_BYTES + h * 8192, &p.tma_b, peer_addr(&b_full[bs], 0),
                                       ti.nt * BN + (int)rank * (BN / 2) + h * 64, cb * BK, p.b_plane[w]);
                  } else {
                    tma_load_3d_pair(sb + bs * B_BYTES, &p.tma_b, peer_addr(&b_full[bs], 0), cb * BK,
                                     ti.nt * BN + (int)rank * (BN / 2), p.b_plane[w]);
                  }
                } else if (dbg & 8) {
                  mbar_arrive(&b_full[bs]);
                } else {
                  mbar_expect_tx(&b_full[bs], p.b_tx);
                  if (p.b_mn) {
#pragma unroll 1
                    for (int h = 0; h < BN / 64; ++h)
                      tma_load_3d(sb + bs * B_BYTES + h * 8192, &p.tma_b, &b_full[bs], ti.nt * BN + h * 64, cb * BK,
                                  p.b_plane[w]);
                  } else {
                    tma_load_3d(sb + bs * B_BYTES, &p.tma_b, &b_full[bs], cb * BK, ti.nt * BN, p.b_plane[w]);
                  }
                }
              }
              __syncwarp();
              rb.next(BSTAGES);
            }
          }
        }
      } else {
        for (int i = 0; i < (ti.nkb + KM - 1) / KM; ++i) {
          const int kb = ti.kb0 + KM * i;
          const int as = ra.slot(AST);
          mbar_wait(&a_empty[as], ra.phase(AST) ^ 1u);
          if (elect_one()) {
            if (!PAIR || rank == 0) mbar_expect_tx(&a_full[as], PAIR ? 2 * p.a_tx : p.a_tx);
#pragma unroll
            for (int h = 0; h < BM / 64; ++h) {
              int pr = ti.mt * 2 + h;
              if (pr >= p.n_pairs) pr = 0;  // masked rows (beyond the pairs): reload a valid pair
              const int w = p.pair_win[pr];
#pragma unroll
              for (int kq = 0; kq < KM; ++kq) {
                // K block kb + kq at +16 KB (the last split's odd tail reads zero dy rows)
                if constexpr (PAIR)
                  tma_load_3d_pair(sa + as * p.a_stage_bytes + kq * 16384 + h * 8192, &p.tma_a,
                                   peer_addr(&a_full[as], 0), p.pair_cb[pr] * 64, (kb + kq) * BK + p.a_shift[w],
                                   p.a_plane[w]);
                else
                  tma_load_3d(sa + as * p.a_stage_bytes + h * 8192, &p.tma_a, &a_full[as], p.pair_cb[pr] * 64,
                              kb * BK + p.a_shift[w], p.a_plane[w]);
              }
            }
          }
          __syncwarp();
          ra.next(AST);
          const int bs = rb.slot(BSTAGES);
          mbar_wait(&b_empty[bs], rb.phase(BSTAGES) ^ 1u);
          if (elect_one()) {
            if constexpr (PAIR) {
              // this CTA's half of the N columns
              if (rank == 0) mbar_expect_tx(&b_full[bs], 2 * p.b_tx);
#pragma unroll
              for (int kq = 0; kq < KM; ++kq)
#pragma unroll
                for (int h = 0; h < BN / 128; ++h)
                  tma_load_3d_pair(sb + bs * B_BYTES + kq * 16384 + h * 8192, &p.tma_b, peer_addr(&b_full[bs], 0),
                                   ti.nt * BN + (int)rank * (BN / 2) + h * 64, (kb + kq) * BK, 0);
            } else {
              mbar_expect_tx(&b_full[bs], p.b_tx);
#pragma unroll
              for (int h = 0; h < BN / 64; ++h)
                tma_load_3d(sb + bs * B_BYTES + h * 8192, &p.tma_b, &b_full[bs], ti.nt * BN + h * 64, kb * BK, 0);
            }
          }
          __syncwarp();
          rb.next(BSTAGES);
        }
      }
    }
  } else if (warp == 1) {
   // CTA pair: the leader issues every MMA of the pair; the peer's warp 1 only owns its TMEM allocation
   if (!PAIR || rank == 0) {
    // ---------------- MMA issuer: warp-wide loop, elected-lane issue
    constexpr bool mn = MODE == MODE_WGRAD;
    const int b_mn = MODE == MODE_ROWS ? p.b_mn : 0;
    const uint32_t bk_step = b_mn ? 128u : 2u;
    const uint32_t idesc =
        mn ? idesc_bf16(PAIR ? 2 * BM : BM, BN, 1, 1) : idesc_bf16(PAIR ? 2 * BM : BM, BN, 0, b_mn);
    Ring ra, rb;
    uint32_t tcount = 0;
    const uint32_t sa_u = smem_u32(sa), sb_u = smem_u32(sb);
    const int a_stage_bytes = p.a_stage_bytes, Gr = p.G, n_cb = p.n_cblocks;
    const int kq_last = p.kq_last > 0 ? p.kq_last : BK / 16;
    if (b_res && blockIdx.x < n_tiles_total && !(dbg & 1024)) mbar_wait(&b_full[0], 0);  // resident B tiles landed
    TileWalk tw;
    tw.init(p, t_first, t_step);
    for (int t = t_first; t < n_tiles_total; t += t_step, ++tcount, tw.next(p)) {
      const TileInfo ti = tinfo(tw);
      const uint32_t acc = tcount & 1u;
      if (lane == 0) ev(9, (int)tcount, 0);  // MMA warp: next tile decoded
      if (!(dbg & 1024)) mbar_wait(&tempty[acc], ((tcount >> 1) & 1u) ^ 1u);  // epilogue drained this buffer
      if (lane == 0) ev(5, (int)tcount, 0);  // MMA warp: accumulator free
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t dst = tmem + acc * ACC_COLS;
      uint32_t accumulate = 0;
      if constexpr (!mn) {
        // descriptor low words advance by 16-byte units: a row of the
        // swizzled tile is 8, a 16-element K step 2
        const int c1 = p.g_chunk1[ti.g];
        for (int c = p.g_chunk0[ti.g]; c < c1; ++c) {
          const int w0 = p.chunk_w0[c], w1 = p.chunk_w1[c], pmin = p.chunk_pmin[c];
          for (int cb = ti.cb0; cb < ti.cb1; ++cb) {
            const int nk = cb == n_cb - 1 ? kq_last : BK / 16;
            if (!(dbg & 1024)) mbar_wait(&a_full[ra.s], ra.ph);
            if (lane == 0) ev(3, (int)tcount, c * 64 + cb);  // MMA warp: A halo ready
            const uint32_t a_lo0 = desc_lo(sa_u + (uint32_t)(ra.s * a_stage_bytes)) - (uint32_t)pmin * 8u;
            if (b_res) asm volatile("tcgen05.fence::after_thread_sync;");
            for (int w = w0; w < w1; ++w) {
              if (!b_res) {
                if (!(dbg & 1024)) mbar_wait(&b_full[rb.s], rb.ph);
                if (lane == 0) ev(4, (int)tcount, w);  // MMA warp: B window ready
                asm volatile("tcgen05.fence::after_thread_sync;");
              }
              const uint32_t b_addr = sb_u + (uint32_t)((b_res ? w : rb.s) * B_BYTES);
              // MN-major: LBO = 8 KB between 64-wide N atoms, K step = two 8-row groups (2 KB)
              const uint32_t b_lo = b_mn ? ((b_addr >> 4) | ((8192u >> 4) << 16)) : desc_lo(b_addr);
              // profiling switch 32: every window reads the aligned halo start (wrong values, timing only)
              const uint32_t a_lo = (dbg & 32) ? a_lo0 + (uint32_t)pmin * 8u : a_lo0 + (uint32_t)p.a_shift[w] * 8u;
              if (!(dbg & 2)) {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                  if (g >= Gr) break;
#pragma unroll
                  for (int k = 0; k < BK / 16; ++k)
                    if (k < nk)
                      mma_lo<PAIR>(dst + g * BN, a_lo + (uint32_t)(g * BM * 8 + k * 2), b_lo + (uint32_t)(k * bk_step),
                                   idesc, (accumulate || k > 0) ? 1u : 0u);
                }
              }
              accumulate = 1;
              if (lane == 0) ev(11, (int)tcount, w);  // MMA warp: window issued
              if (b_res) {
                // resident B: nothing to release
              } else if (dbg & 16) {
                if (elect_one()) mbar_arrive(&b_empty[rb.s]);  // profiling only: no MMA reads B
                __syncwarp();
              } else if constexpr (PAIR) {
                mma_commit_pair(&b_empty[rb.s]);
              } else {
                mma_commit(&b_empty[rb.s]);
              }
              rb.next(BSTAGES);
            }
            // halo tile free once its windows' MMAs finish
            if constexpr (PAIR) mma_commit_pair(&a_empty[ra.s]);
            else mma_commit(&a_empty[ra.s]);
            ra.next(AST);
          }
        }
      } else {
        for (int i = 0; i < (ti.nkb + KM - 1) / KM; ++i) {
          const int as = ra.slot(AST), bs = rb.slot(BSTAGES);
          if (!(dbg & 1024)) {
            mbar_wait(&a_full[as], ra.phase(AST));
            mbar_wait(&b_full[bs], rb.phase(BSTAGES));
          }
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint64_t da = sw128_mn_desc(sa + as * p.a_stage_bytes, 8192);
          const uint64_t db = sw128_mn_desc(sb + bs * B_BYTES, 8192);
#pragma unroll
          for (int k = 0; k < KM * BK / 16; ++k) {
            // MN-major K advance: two 8-row k groups (2 x 1024 B) per 16 K;
            // the second 64-block of a KM = 2 stage starts 16 KB further
            const uint64_t ko = (uint64_t)((k & 3) * 128 + (k >> 2) * (16384 >> 4));
            if constexpr (PAIR)
              mma_bf16_pair(dst, da + ko, db + ko, idesc, accumulate);
            else
              mma_bf16(dst, da + ko, db + ko, idesc, accumulate);
            accumulate = 1;
          }
          if constexpr (PAIR) {
            mma_commit_pair(&a_empty[as]);
            mma_commit_pair(&b_empty[bs]);
          } else {
            mma_commit(&a_empty[as]);
            mma_commit(&b_empty[bs]);
          }
          ra.next(AST);
          rb.next(BSTAGES);
        }
      }
      if (lane == 0) ev(6, (int)tcount, 0);  // MMA warp: tile issued
      if (accumulate) {
        if constexpr (PAIR) mma_commit_pair(&tfull[acc]);
        else mma_commit(&tfull[acc]);
      } else {
        if (elect_one()) {
          mbar_arrive(&tfull[acc]);
          if constexpr (PAIR) mbar_arrive_cluster(peer_addr(&tfull[acc], 1));
        }
        __syncwarp();
      }
      if (lane == 0) ev(10, (int)tcount, 0);  // MMA warp: tile committed
    }
   }
  } else {
    // epilogue warps: TMEM lane quarter = warp % 4, column-chunk parity = (warp - 2) / 4
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    uint32_t tcount = 0;
    TileWalk tw;
    tw.init(p, t_first, t_step);
    for (int t = t_first; t < n_tiles_total; t += t_step, ++tcount, tw.next(p)) {
      const TileInfo ti = tinfo(tw);
      const uint32_t acc = tcount & 1u;
      if (dbg & 64) mbar_wait(&tfull[acc], (tcount >> 1) & 1u);
      else mbar_wait_sleep(&tfull[acc], (tcount >> 1) & 1u);
      if (warp == 2 && lane == 0) ev(7, (int)tcount, 0);  // epilogue: accumulator full
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // profiling switch 256: no TMEM reads or stores (release the buffer at once)
      const int nsub = (dbg & 256) ? 0 : MODE == MODE_ROWS ? p.G : 1;
      const bool have = ti.nkb > 0;
      const float scale = p.scale;
#pragma unroll 1
      for (int g = 0; g < nsub; ++g) {
        bool ok;
        int64_t off;
        if constexpr (MODE == MODE_ROWS) {
          // 32-bit row decode (the padded grid has < 2^31 rows per plane,
          // host-checked): 64-bit div / mod are subroutine calls
          const uint32_t flat = (uint32_t)((ti.mt * p.G + g) * BM + r);
          const uint32_t tq = flat / (uint32_t)p.Wp;
          const int wp = (int)(flat - tq * (uint32_t)p.Wp);
          const uint32_t img = tq / (uint32_t)p.Hp;
          const int hp = (int)(tq - img * (uint32_t)p.Hp);
          const int h = hp - p.lo_h, w = wp - p.lo_w;
          ok = (int)img < p.n_img && h >= 0 && h < p.H && w >= 0 && w < p.W;
          off = p.g_out_off[ti.g] + (int64_t)img * p.o_img + (int64_t)h * p.o_h + (int64_t)w * p.o_w;
        } else {
          const int pr = ti.mt * 2 + (r >> 6);
          const int ci = pr < p.n_pairs ? p.pair_cb[pr] * 64 + (r & 63) : p.m_ext;
          ok = pr < p.n_pairs && ci < p.m_ext;
          off = ok ? p.g_out_off[p.pair_win[pr]] + (int64_t)ci * p.o_m : 0;
        }
        if (!have && p.out_kind == OUT_F32_ATOMIC) ok = false;
#pragma unroll 1
        for (int c = half * 32; c < BN; c += 64) {
          const int n0 = ti.nt * BN + c;
          if (n0 >= p.n_ext) break;  // warp-uniform
          float v[32];
          tmem_ld32(tmem + acc * ACC_COLS + (uint32_t)(g * BN) + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
          const int nlim = min(32, p.n_ext - n0);
          const int64_t os = p.o_n;
          if constexpr (MODE == MODE_ROWS && CFG != 1) {
            if (p.out_kind == OUT_BF16 && os == 1 && nlim == 32 && !(dbg & 1)) {
              __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(p.out) + n0;
              const bool al = !ok || ((reinterpret_cast<uintptr_t>(ob + off) & 15) == 0);
              if (__all_sync(0xffffffffu, al)) {
                // staged: my row's 32 values -> smem row `lane`, then each
                // store instruction covers 8 rows x 64 contiguous bytes
                uint32_t* stg = reinterpret_cast<uint32_t*>(smem + ring_bytes<CFG>() + 512) +
                                (warp - 2) * (32 * EPI_ROW_WORDS);
                uint4* mine = reinterpret_cast<uint4*>(stg + lane * EPI_ROW_WORDS);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                  __align__(16) __nv_bfloat162 h2[4];
#pragma unroll
                  for (int e = 0; e < 4; ++e)
                    h2[e] = __floats2bfloat162_rn(have ? v[q4 * 8 + 2 * e] * scale : 0.f,
                                                  have ? v[q4 * 8 + 2 * e + 1] * scale : 0.f);
                  mine[q4] = *reinterpret_cast<const uint4*>(h2);
                }
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const int rr = i * 8 + (lane >> 2), seg = lane & 3;
                  const uint4 val = reinterpret_cast<const uint4*>(stg + rr * EPI_ROW_WORDS)[seg];
                  const int okr = __shfl_sync(0xffffffffu, ok ? 1 : 0, rr);
                  const long long offr = __shfl_sync(0xffffffffu, (long long)off, rr);
                  if (okr) reinterpret_cast<uint4*>(ob + offr)[seg] = val;
                }
                __syncwarp();
                continue;
              }
            }
          }
          if (!ok || (dbg & 1)) {
            // masked row (pad pixel / beyond the extent): nothing to store
          } else if (MODE == MODE_WGRAD || p.out_kind == OUT_F32_ATOMIC) {
            float* o = reinterpret_cast<float*>(p.out) + off + (int64_t)n0 * os;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < nlim) atomicAdd(o + (int64_t)j * os, v[j] * scale);
          } else if (p.out_kind == OUT_BF16) {
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + off + (int64_t)n0 * os;
            if (nlim == 32 && os == 1 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
              // N contiguous in the output (QKV-like): four 16-byte stores per thread
              uint4* o4 = reinterpret_cast<uint4*>(o);
#pragma unroll
              for (int q4 = 0; q4 < 4; ++q4) {
                __align__(16) __nv_bfloat162 h2[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  h2[e] = __floats2bfloat162_rn(have ? v[q4 * 8 + 2 * e] * scale : 0.f,
                                                have ? v[q4 * 8 + 2 * e + 1] * scale : 0.f);
                o4[q4] = *reinterpret_cast<const uint4*>(h2);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j < nlim) o[(int64_t)j * os] = __float2bfloat16_rn(have ? v[j] * scale : 0.f);
            }
          } else {
            float* o = reinterpret_cast<float*>(p.out) + off + (int64_t)n0 * os;
            if (nlim == 32 && os == 1 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
              float4* o4 = reinterpret_cast<float4*>(o);
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4)
                o4[q4] = have ? make_float4(v[4 * q4] * scale, v[4 * q4 + 1] * scale, v[4 * q4 + 2] * scale,
                                            v[4 * q4 + 3] * scale)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j < nlim) o[(int64_t)j * os] = have ? v[j] * scale : 0.f;
            }
          }
        }
      }  // sub-tiles
      // release the accumulator buffer to the MMA warp (one arrive per warp)
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (warp == 2 && lane == 0) ev(8, (int)tcount, 0);  // epilogue: drained
      if (lane == 0) {
        if constexpr (PAIR) mbar_arrive_cluster(peer_addr(&tempty[acc], 0));  // the leader's MMA warp waits
        else mbar_arrive(&tempty[acc]);
      }
      if constexpr (MODE == MODE_WGRAD) {
        if (p.fix_out) {
          // every epilogue warp's atomics for this tile are issued
          asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
          if (warp == 2 && lane == 0) {
            __threadfence();
            const int tile_mn = ti.mt * p.n_tiles + ti.nt;
            const unsigned prev = atomicAdd(p.fix_cnt + tile_mn, 1u);
            *fix_last = prev == (unsigned)(p.ksplit - 1) ? 1u : 0u;
            if (*fix_last) p.fix_cnt[tile_mn] = 0u;  // ready for the next call (stream order)
          }
          asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
          if (*fix_last) {
            __threadfence();
            const int pr = ti.mt * 2 + (r >> 6);
            const int ci = pr < p.n_pairs ? p.pair_cb[pr] * 64 + (r & 63) : p.m_ext;
            if (ci < p.m_ext) {
              const int w = p.pair_win[pr];
              float* src = reinterpret_cast<float*>(p.out) + p.g_out_off[w] + (int64_t)ci * p.o_m;
              const int64_t dst = p.fix_win_off[w] + (int64_t)ci * p.fix_s_ci;
#pragma unroll 1
              for (int c = half * 32; c < BN; c += 64) {
                const int n0 = ti.nt * BN + c;
                if (n0 >= p.n_ext) break;
                const int nlim = min(32, p.n_ext - n0);
#pragma unroll 4
                for (int j = 0; j < nlim; ++j) {
                  float* e = src + (int64_t)(n0 + j) * p.o_n;
                  const float v = __ldcg(e);
                  *e = 0.f;
                  const int64_t o = dst + (int64_t)(n0 + j) * p.fix_s_co;
                  if (p.fix_f32) reinterpret_cast<float*>(p.fix_out)[o] = v;
                  else reinterpret_cast<__nv_bfloat16*>(p.fix_out)[o] = __float2bfloat16(v);
                }
              }
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  // pair: neither CTA leaves (or frees TMEM) while the other may still signal it
  if constexpr (PAIR) cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

template <int BN, int CFG = 0>
constexpr int smem_bytes() {
  return 1024 + ring_bytes<CFG>() + 512 + (CFG != 1 ? EPI_STAGE_BYTES : 0);
}

}  // namespace tc
}  // namespace syno
