// Device engine: index tables (K1), the universal stage kernels and the
// per-operator device plan.  Host-visible interface used by the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "plan.hpp"

namespace syno {

enum DType : int { DT_F32 = 0, DT_BF16 = 1, DT_F64 = 2 };

constexpr int MAXA = 10;    // axes of a stage
constexpr int MAXT = 8;     // terms of a stage (phantoms included)
constexpr int MAXTAB = 4;   // axis-only coordinate tables per term
constexpr int MAXMIX = 4;   // axis x reduce coordinate tables per term

struct KTerm {
  const void* ptr;
  int32_t kind;             // 0 = input dtype, 1 = accumulator dtype, 2 = phantom
  int32_t n_atab, n_mix;
  int32_t pad_;
  int64_t base;
  int64_t lin[MAXA];        // axis-linear offset coefficients
  const int32_t* atab[MAXTAB];
  int32_t atab_s[MAXTAB][MAXA];
  const int32_t* mtab[MAXMIX];
  int32_t mtab_s[MAXMIX][MAXA];
  const int32_t* mri[MAXMIX];  // per flat-reduce index into mtab
  const int32_t* rtab;         // per flat-reduce offset (-1: out of range), null if none
};

struct KStage {
  int32_t n_axes, n_terms;
  int32_t out_acc;          // output in accumulator dtype (stage buffers, scatter scratch)
  int32_t pad_;
  int64_t axis_ext[MAXA];
  int64_t out_count;        // prod(axis_ext)
  int64_t R;                // prod(red_ext)
  int64_t r_chunk;          // reduce iterations per blockIdx.y
  double scale;
  void* out;
  KTerm terms[MAXT];
  KTerm target;             // scatter form only
  // On-the-fly coordinate programs (stages whose index tables would exceed
  // the table budget): per term (terms, then target) a record
  //   [ncoord, (code_off, code_len, n, stride) x ncoord]
  // followed by the int64 postfix code; null when tables are used.
  const int64_t* prog;
  int32_t prog_term_off[MAXT + 1];
  int32_t n_red;
  int32_t pad2_;
  int64_t red_ext[16];
  // Scatter form: deterministic fixed-point accumulation (engine.cu fx_add):
  // per output element one signed 64-bit word (fp32/bf16) or a 128-bit
  // (lo, hi) pair (f64), scaled by 2^shift with the shift derived from a
  // bound on every partial sum: fx_mult * prod(fx_max[0..fx_n)) (the max |v|
  // of each loaded term, computed on the device by maxabs_kernel).
  unsigned long long* fx;
  const double* fx_max;
  int32_t fx_n;
  int32_t pad3_;
  double fx_mult;
};

// One device-resident stage: tables plus a descriptor with null pointers
// for the run-time tensors (bound per launch).
// Tiled gather form (engine.cu, stage_tile_kernel): the stage's axes split
// into F (read together with reduces through mixed tables), I (read only
// through per-thread axis parts) and B (not read by any reduce-dependent
// term).  One CTA computes the reduce sum for a tile of F x I outputs,
// staging the per-(F, r) offset rows of every reduce-dependent term in
// shared memory once per CTA; a finish stage multiplies in the
// reduce-invariant terms, sums the reduce splits in a fixed order and
// broadcasts over B.
struct TileArgs {
  int32_t nF, nI;
  int32_t faxis[MAXA], iaxis[MAXA];
  int32_t fext[MAXA], iext[MAXA];
  int32_t NF, NI;
  int32_t TF, TI, TR;       // CTA tile: TI x TF outputs, TR threads per output along the reduce
  int32_t RC;               // reduce chunk staged in shared memory
  int32_t n_rt;             // reduce-dependent terms
  int32_t rterm[MAXT];
  int32_t nIb;              // CTAs along I
  int32_t ffast;            // lanes run along F (else along I)
  int32_t scatter;          // scatter form: rterm's last entry (-1) is the target
  int32_t n_inv;            // scatter form: reduce-invariant terms (a per-thread factor)
  int32_t inv[MAXT];
  void* acc;                // [S][NF][NI] accumulator scratch
};

struct DevStage;
struct TileInfo {
  TileArgs a;
  int64_t splits = 1;
  int64_t ctas = 1;
  size_t smem = 0;
  std::shared_ptr<DevStage> finish;
};

struct DevStage {
  CStage cs;
  KStage k;
  std::shared_ptr<TileInfo> tile;  // tiled gather form, when it applies
  // Scatter form with axes that neither the target nor any reduce-dependent
  // term reads: `pre` (a gather stage) first sums the reduce-invariant terms
  // over those axes into a scratch tensor, which this stage then scatters.
  std::shared_ptr<DevStage> pre;
  // Lane-contiguous layout: `perm_in` copies one input with a permuted axis
  // order (TK_PERM, perm_count elements) so that the tile kernel's lanes read
  // it with unit stride; this stage reads the copy instead of the input.
  std::shared_ptr<DevStage> perm_in;
  int64_t perm_count = 0;
  // ... and for a scatter whose target is written along a strided axis: the
  // scatter accumulates into a permuted copy of the target (accumulator
  // precision) and `perm_out` restores the target's own layout.
  std::shared_ptr<DevStage> perm_out;
  // Factored gather: `gpre` sums the product of the terms that alone read
  // some reduce loops over those loops (TK_PRE, gpre_count elements); this
  // stage then reduces the rest (the reference's rfactor, for any stage).
  std::shared_ptr<DevStage> gpre;
  int64_t gpre_count = 0;
  std::vector<int> term_slot;   // CTensor of each term, to bind pointers
  int32_t* tables = nullptr;    // owned device allocation
  int64_t* prog = nullptr;      // owned device allocation (program fallback)
  size_t table_entries = 0;
  bool dead = false;
};

struct TcPlan;  // tensor-core path (tc.cu)
struct TcPlanDeleter {
  void operator()(TcPlan* p) const;
};
using TcPlanPtr = std::unique_ptr<TcPlan, TcPlanDeleter>;

struct GatherGemm;  // gathered-operand tensor-core path (engine.cu)

struct DevPlan {
  int device = -1;
  std::shared_ptr<GatherGemm> gg;  // null unless the operator is a gathered GEMM
  // Universal-engine stages are built on first use (the tensor-core path
  // usually makes them unnecessary); guarded by `mu`.
  std::mutex mu;
  bool have_forward = false, have_backward = false;
  std::vector<DevStage> forward, grad_x, bwd_staged;
  std::vector<std::vector<DevStage>> grad_w;
  TcPlanPtr tc;  // null when the operator is not contraction-shaped
  // Readiness of what the builds enqueued (index tables, folds) on the
  // building stream: other streams wait on these instead of the host
  // synchronising after every build.
  cudaEvent_t ev_plan = nullptr, ev_fwd = nullptr, ev_bwd = nullptr;
  ~DevPlan();
};



struct Bindings {
  const void* x = nullptr;
  std::vector<const void*> w;
  void* y = nullptr;
  const void* dy = nullptr;
  void* dx = nullptr;
  std::vector<void*> dw;
  std::vector<void*> stages;  // t_k buffers
  std::vector<void*> dstages; // gradients of t_k (staged backward)
  const void* scratch = nullptr;  // tiled form: the reduce sums read by the finish stage
  const void* perm = nullptr;     // DevStage::perm_in's copy (TK_PERM)
  const void* pre = nullptr;      // DevStage::gpre's partial sums (TK_PRE)
  bool x_unchanged = false;   // syno_backward_ex(SYNO_BWD_X_UNCHANGED)
  bool w_unchanged = false;   // syno_backward_ex(SYNO_BWD_W_UNCHANGED)
};

// Build one device stage (K1 tables) / launch it through the universal kernel.
void build_dev_stage(const CStage& cs, DevStage* ds, cudaStream_t stream);
void release_dev_stage(DevStage& ds);
void run_stage(DType dt, const DevStage& ds, const Bindings& b, void* out, bool out_acc, cudaStream_t stream);

// Host-only: does the operator take the gathered-GEMM tensor-core path
// (engine.cu GatherGemm) for fp32 / bf16?
bool gg_matches(const Plan& plan);
// the staged nest (forward and backward) is far cheaper than the unstaged
// contraction the tensor-core paths compute: stay on the stage engine
bool staged_cheaper(const Plan& plan);

// Builds tables on `stream` (K1) for every stage of the plan.
DevPlan* build_dev_plan(const Plan& plan, cudaStream_t stream);

// Make `stream` wait for the plan's device-side builds (no-op while capturing).
void wait_built(cudaEvent_t ev, cudaStream_t stream);

// Launches. All pointers are device pointers; tensors are dense row-major.
void run_forward(const Plan& plan, DevPlan& dp, DType dt, const Bindings& b, cudaStream_t stream);
void run_backward(const Plan& plan, DevPlan& dp, DType dt, const Bindings& b, cudaStream_t stream);

// K1 debug/parity hook: raw int64 values of one coordinate of one term over
// the full loop grid of a stage (row-major over axes then reduces).
void eval_coordinate_grid(const CStage& s, int term, int coord, int64_t* out_dev, cudaStream_t stream);

void cuda_check(cudaError_t e, const char* what);

// Programmatic dependent launch: every library kernel is launched with
// programmatic stream serialization, triggers its dependents as soon as it
// starts and waits for its predecessor grid before its first global memory
// access.  The next kernel's launch and CTA scheduling then overlap this
// kernel's tail; semantics stay serial because every kernel waits before
// touching memory (griddepcontrol.wait is a no-op without the attribute).
// SYNO_NO_PDL=1 disables the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();

// Profiling only: SYNO_SKIP=pack,fold,chain,cast,zero,gemm suppresses those
// launches (wrong results) so a step's time can be attributed per class.
bool skip_class(const char* name);

// Stream-ordered zero fill as a library kernel (part of the PDL chain,
// unlike cudaMemsetAsync).
void zero_fill(void* ptr, size_t bytes, cudaStream_t stream);

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

// Process-wide count of kernels this library launched (syno_launch_count).
void note_launch();
uint64_t launch_count();

// Optional per-launch timing (syno_profile_begin/end): when enabled, every
// library launch is bracketed by CUDA events on its own stream and tagged
// with the kernel class and its algorithmic FLOPs / bytes.  Off by default
// and never enabled inside a CUDA-graph capture.
int prof_begin(const char* name, double flops, double bytes, cudaStream_t stream);
void prof_end(int id, cudaStream_t stream);
void prof_rename(int id, const char* name);
struct ProfStat {
  std::string name;
  int64_t launches = 0;
  double ms = 0, flops = 0, bytes = 0;
};
void prof_enable(bool on);
// true between syno_profile_begin/end: launches are serialised on the caller's
// stream (no side-stream fork) so per-launch durations never overlap
bool prof_active();
std::vector<ProfStat> prof_collect();

}  // namespace syno
