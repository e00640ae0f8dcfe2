// Universal device engine for synthesized-operator stages.
//
//  K1  k1_build_table   integer index tables: coordinate programs evaluated
//                       with Python floor semantics (symexpr.py:242-245) over
//                       their iterator grids; -1 marks out-of-range
//                       (codegen.py:535-541 valid mask).
//  K2/K3 stage_kernel   gather + product + reduce of one stage
//                       (codegen.py:515-546), fp32/f64 accumulation,
//                       optional reduce split across blockIdx.y.
//  K6/K7 scatter form   the reference's np.add.at gradient (codegen.py:727-742)
//                       with device atomics, for targets that do not invert.
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <set>

#include "engine.hpp"
#include "tc.hpp"

namespace syno {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(SYNO_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool skip_class(const char* name) {
  static const std::string list = [] {
    const char* e = getenv("SYNO_SKIP");
    return std::string(e ? e : "");
  }();
  if (list.empty()) return false;
  return ("," + list + ",").find("," + std::string(name) + ",") != std::string::npos;
}

bool pdl_enabled() {
  static const bool on = getenv("SYNO_NO_PDL") == nullptr;
  return on;
}

__global__ void __launch_bounds__(256) zero_fill_kernel(uint4* p, int64_t n16, uint8_t* tail, int tail_bytes) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
  if (blockIdx.x == 0 && (int)threadIdx.x < tail_bytes) tail[threadIdx.x] = 0;
}

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

void zero_fill(void* ptr, size_t bytes, cudaStream_t stream) {
  if (!bytes || skip_class("zero")) return;
  // library buffers are 16-byte aligned (cudaMalloc / pool); a misaligned
  // pointer falls back to the runtime memset
  if (reinterpret_cast<uintptr_t>(ptr) & 15) {
    cuda_check(cudaMemsetAsync(ptr, 0, bytes, stream), "cudaMemsetAsync");
    return;
  }
  const int64_t n16 = (int64_t)(bytes / 16);
  const int tail = (int)(bytes - (size_t)n16 * 16);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n16 + 255) / 256, 148 * 8));
  note_launch();
  launch_k(zero_fill_kernel, (unsigned)blocks, 256, 0, stream, static_cast<uint4*>(ptr), n16,
           static_cast<uint8_t*>(ptr) + n16 * 16, tail);
}

namespace {
struct ProfRec {
  std::string name;
  cudaEvent_t a = nullptr, b = nullptr;
  double flops = 0, bytes = 0;
};
std::mutex g_prof_mu;
std::atomic<bool> g_prof_on{false};
std::vector<ProfRec> g_prof;
}  // namespace

// Inside a CUDA-graph capture the events become event-record nodes
// (cudaEventRecordExternal), so a profiled graph replay times every launch
// without host launch latency between them.
static cudaError_t record_prof_event(cudaEvent_t e, cudaStream_t stream) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &st);
  if (st == cudaStreamCaptureStatusActive) return cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal);
  return cudaEventRecord(e, stream);
}

void prof_enable(bool on) {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  for (auto& r : g_prof) {
    if (r.a) cudaEventDestroy(r.a);
    if (r.b) cudaEventDestroy(r.b);
  }
  g_prof.clear();
  g_prof_on = on;
}

bool prof_active() { return g_prof_on.load(std::memory_order_relaxed); }

int prof_begin(const char* name, double flops, double bytes, cudaStream_t stream) {
  if (!g_prof_on.load(std::memory_order_relaxed)) return -1;
  ProfRec r;
  r.name = name;
  r.flops = flops;
  r.bytes = bytes;
  cuda_check(cudaEventCreate(&r.a), "cudaEventCreate(prof)");
  cuda_check(cudaEventCreate(&r.b), "cudaEventCreate(prof)");
  cuda_check(record_prof_event(r.a, stream), "cudaEventRecord(prof)");
  std::lock_guard<std::mutex> lock(g_prof_mu);
  g_prof.push_back(r);
  return (int)g_prof.size() - 1;
}

void prof_rename(int id, const char* name) {
  if (id < 0) return;
  std::lock_guard<std::mutex> lock(g_prof_mu);
  if (id < (int)g_prof.size()) g_prof[id].name = name;
}

void prof_end(int id, cudaStream_t stream) {
  if (id < 0) return;
  cudaEvent_t b;
  {
    std::lock_guard<std::mutex> lock(g_prof_mu);
    if (id >= (int)g_prof.size()) return;
    b = g_prof[id].b;
  }
  cuda_check(record_prof_event(b, stream), "cudaEventRecord(prof)");
}

std::vector<ProfStat> prof_collect() {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  std::vector<ProfStat> out;
  for (auto& r : g_prof) {
    cuda_check(cudaEventSynchronize(r.b), "cudaEventSynchronize(prof)");
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, r.a, r.b), "cudaEventElapsedTime(prof)");
    auto it = std::find_if(out.begin(), out.end(), [&](const ProfStat& s) { return s.name == r.name; });
    if (it == out.end()) {
      out.push_back(ProfStat{r.name});
      it = out.end() - 1;
    }
    it->launches += 1;
    it->ms += ms;
    it->flops += r.flops;
    it->bytes += r.bytes;
  }
  return out;
}

// ---------------------------------------------------------------------------
// K1: coordinate programs
// ---------------------------------------------------------------------------

enum : int64_t { BC_LOOP = 0, BC_CONST = 1, BC_ADD = 2, BC_SUB = 3, BC_MUL = 4, BC_FDIV = 5, BC_MOD = 6 };
constexpr int MAXL = 24;     // loops a table may depend on
constexpr int MAXPROG = 16;  // programs summed into one table
constexpr int MAXSTACK = 32;

static void compile_prog(const CE& e, const std::vector<int>& local, std::vector<int64_t>* code) {
  switch (e->op) {
    case COp::Loop: {
      int idx = (int)(std::find(local.begin(), local.end(), e->loop) - local.begin());
      if (idx >= (int)local.size()) fail(SYNO_E_GRAPH, "coordinate program references a foreign loop");
      code->push_back(BC_LOOP); code->push_back(idx);
      return;
    }
    case COp::Const: code->push_back(BC_CONST); code->push_back(e->value); return;
    default: break;
  }
  compile_prog(e->lhs, local, code);
  compile_prog(e->rhs, local, code);
  int64_t op = e->op == COp::Add ? BC_ADD : e->op == COp::Sub ? BC_SUB : e->op == COp::Mul ? BC_MUL
               : e->op == COp::FloorDiv ? BC_FDIV : BC_MOD;
  code->push_back(op); code->push_back(0);
}

static int prog_depth(const CE& e) {
  if (e->op == COp::Loop || e->op == COp::Const) return 1;
  return std::max(prog_depth(e->lhs), prog_depth(e->rhs) + 1);
}

__host__ __device__ inline int64_t dev_floordiv(int64_t a, int64_t b) {
  if (b == 0) return 0;
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
__host__ __device__ inline int64_t dev_mod(int64_t a, int64_t b) {
  if (b == 0) return 0;
  int64_t r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) r += b;
  return r;
}

__device__ int64_t eval_prog(const int64_t* code, int64_t len, const int64_t* vals) {
  int64_t st[MAXSTACK];
  int sp = 0;
  for (int64_t i = 0; i < len; ++i) {
    int64_t op = code[2 * i], arg = code[2 * i + 1];
    if (op == BC_LOOP) { st[sp++] = vals[arg]; continue; }
    if (op == BC_CONST) { st[sp++] = arg; continue; }
    int64_t b = st[--sp], a = st[--sp];
    int64_t r;
    switch (op) {
      case BC_ADD: r = a + b; break;
      case BC_SUB: r = a - b; break;
      case BC_MUL: r = a * b; break;
      case BC_FDIV: r = dev_floordiv(a, b); break;
      default: r = dev_mod(a, b); break;
    }
    st[sp++] = r;
  }
  return st[0];
}

constexpr int K1_INLINE = 256;  // int64 words of program code passed in the kernel parameters

struct K1Args {
  int32_t nprog, ndeps;
  int64_t dep_ext[MAXL];
  int64_t count;
  const int64_t* code;      // device code, or null: icode
  int64_t icode[K1_INLINE];
  int64_t prog_off[MAXPROG];
  int64_t prog_len[MAXPROG];
  int64_t n[MAXPROG];       // extent for the range check, <= 0: no check
  int64_t stride[MAXPROG];
  int32_t* out;             // table mode
  int64_t* out_raw;         // raw mode: the single program's value
};

__global__ void k1_build_table(const __grid_constant__ K1Args a) {
  pdl_trigger();
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.count) return;
  int64_t vals[MAXL];
  int64_t rem = i;
  for (int k = a.ndeps - 1; k >= 0; --k) {
    vals[k] = rem % a.dep_ext[k];
    rem /= a.dep_ext[k];
  }
  if (a.out_raw) {
    a.out_raw[i] = eval_prog((a.code ? a.code : a.icode) + a.prog_off[0], a.prog_len[0], vals);
    return;
  }
  int64_t sum = 0;
  bool ok = true;
  for (int p = 0; p < a.nprog; ++p) {
    int64_t v = eval_prog((a.code ? a.code : a.icode) + a.prog_off[p], a.prog_len[p], vals);
    if (a.n[p] > 0 && (v < 0 || v >= a.n[p])) ok = false;
    sum += v * a.stride[p];
  }
  a.out[i] = ok ? (int32_t)sum : -1;
}

// Largest index table (entries) a coordinate may get before the stage
// falls back to on-the-fly programs.  SYNO_TABLE_LIMIT lowers it (tests use
// it to drive the program path on small operators).
// A table is built once per (operator, device) and read row by row by the
// tiled kernels, so even a 2^29-entry (2 GB) table costs one K1 pass plus
// one coalesced read -- far less than evaluating its program at every one of
// the (larger) grid's points.
static int64_t table_limit() {
  const char* e = getenv("SYNO_TABLE_LIMIT");
  return e ? std::max<int64_t>(1, atoll(e)) : ((int64_t)1 << 29) + 1;
}

struct ProgSpec {
  CE e;
  int64_t n, stride;
};

struct TabSpec {
  std::vector<int> deps;
  std::vector<int64_t> dep_ext;
  std::vector<ProgSpec> progs;
  int64_t count = 1;
  size_t offset = 0;
};

static void launch_k1(const TabSpec& t, int32_t* out, int64_t* out_raw, cudaStream_t stream) {
  if ((int)t.deps.size() > MAXL) fail(SYNO_E_UNSUPPORTED, "index table depends on too many loops");
  if ((int)t.progs.size() > MAXPROG) fail(SYNO_E_UNSUPPORTED, "too many coordinates in one index table");
  K1Args a{};
  a.nprog = (int)t.progs.size();
  a.ndeps = (int)t.deps.size();
  for (size_t k = 0; k < t.deps.size(); ++k) a.dep_ext[k] = t.dep_ext[k];
  a.count = t.count;
  std::vector<int64_t> code;
  for (size_t p = 0; p < t.progs.size(); ++p) {
    if (prog_depth(t.progs[p].e) > MAXSTACK) fail(SYNO_E_UNSUPPORTED, "coordinate expression too deep");
    a.prog_off[p] = (int64_t)code.size();
    size_t before = code.size();
    compile_prog(t.progs[p].e, t.deps, &code);
    a.prog_len[p] = (int64_t)(code.size() - before) / 2;
    a.n[p] = t.progs[p].n;
    a.stride[p] = t.progs[p].stride;
  }
  if (code.empty()) code.push_back(0);
  int64_t* dcode = nullptr;
  if (code.size() <= (size_t)K1_INLINE) {
    // small programs travel in the launch parameters: no copy, no host sync
    memcpy(a.icode, code.data(), code.size() * sizeof(int64_t));
    a.code = nullptr;
  } else {
    cuda_check(cudaMallocAsync((void**)&dcode, code.size() * sizeof(int64_t), stream), "cudaMallocAsync(code)");
    cuda_check(cudaMemcpyAsync(dcode, code.data(), code.size() * sizeof(int64_t), cudaMemcpyHostToDevice, stream),
               "cudaMemcpyAsync(code)");
    a.code = dcode;
  }
  a.out = out;
  a.out_raw = out_raw;
  if (t.count > 0) {
    int64_t blocks = (t.count + 255) / 256;
    note_launch();
    launch_k(k1_build_table, (unsigned)blocks, 256, 0, stream, a);
    cuda_check(cudaGetLastError(), "k1_build_table");
  }
  if (dcode) {
    // the host copy of `code` must outlive the async memcpy (rare: long programs)
    cuda_check(cudaStreamSynchronize(stream), "k1 sync");
    cuda_check(cudaFreeAsync(dcode, stream), "cudaFreeAsync(code)");
  }
}

void eval_coordinate_grid(const CStage& s, int term, int coord, int64_t* out_dev, cudaStream_t stream) {
  const CTerm& t = term < (int)s.terms.size() ? s.terms[term] : s.target;
  TabSpec tab;
  for (int l = 0; l < s.nloops(); ++l) {
    tab.deps.push_back(l);
    tab.dep_ext.push_back(s.ext(l));
    tab.count *= s.ext(l);
  }
  tab.progs.push_back({t.coords.at(coord), 0, 1});
  launch_k1(tab, nullptr, out_dev, stream);
}

// ---------------------------------------------------------------------------
// Stage construction (host)
// ---------------------------------------------------------------------------

struct Fixup {
  const int32_t** field;
  int table;
};

static std::vector<int64_t> row_major_strides(const std::vector<int64_t>& ext) {
  std::vector<int64_t> s(ext.size(), 1);
  for (int k = (int)ext.size() - 2; k >= 0; --k) s[k] = s[k + 1] * ext[k + 1];
  return s;
}

static int64_t dep_product(const CStage& s, const std::vector<int>& deps) {
  int64_t n = 1;
  for (int l : deps) n *= s.ext(l);
  return n;
}

// A mixed coordinate (depends on axes AND reduces) that is provably inside
// [0, n) needs no bound check, so its top-level parts (c_sum_parts) can be
// tabulated separately: axis-linear parts become lin coefficients,
// axis-only parts one axis table, reduce-only parts the reduce table, and
// the remaining mixed parts one table per dependency set.  Each part table
// holds non-negative entries (biased by the part's minimum, folded into
// `base`), so -1 stays the out-of-range sentinel.  Done only when it makes
// the largest mixed table smaller; false leaves the coordinate whole.
static void add_fix_table(const CStage& s, TabSpec&& tab, KTerm* k, bool axis_only, int A,
                          std::vector<TabSpec>* tabs, std::vector<Fixup>* fix);

static bool split_in_range(const CStage& s, const CE& c, int64_t n, int64_t st, int A, KTerm* k,
                           std::vector<TabSpec>* tabs, std::vector<Fixup>* fix, std::vector<ProgSpec>* rprogs) {
  static const bool off = getenv("SYNO_NO_SPLIT") != nullptr;  // A/B switch
  if (off) return false;
  std::vector<int64_t> ext;
  for (int l = 0; l < s.nloops(); ++l) ext.push_back(s.ext(l));
  int64_t lo, hi;
  if (!c_range(c, ext, &lo, &hi) || lo < 0 || hi >= n) return false;
  int64_t c0;
  std::vector<std::pair<int64_t, CE>> parts;
  c_sum_parts(c, &c0, &parts);
  std::vector<int> whole;
  c_loops(c, &whole);
  struct Part { int64_t coef; CE atom; std::vector<int> deps; int64_t alo, ahi; };
  std::vector<Part> ps;
  std::map<std::vector<int>, int> mixed_groups;
  std::vector<int> axis_deps;
  int64_t biggest = 0;
  for (auto& [coef, a] : parts) {
    Part q{coef, a, {}, 0, 0};
    c_loops(a, &q.deps);
    if (!c_range(a, ext, &q.alo, &q.ahi)) return false;
    const double span = (double)std::llabs(coef) * (double)st * (double)(q.ahi - q.alo);
    if (span >= 2147483647.0) return false;
    const bool ax = q.deps.back() < A, rd = q.deps.front() >= A;
    if (!ax && !rd) {
      mixed_groups.emplace(q.deps, 0);
      biggest = std::max(biggest, dep_product(s, q.deps));
    } else if (ax && a->op != COp::Loop) {
      for (int l : q.deps) axis_deps.push_back(l);
    }
    ps.push_back(q);
  }
  if (biggest >= dep_product(s, whole)) return false;  // no smaller table than the whole coordinate
  const int new_atab = axis_deps.empty() ? 0 : 1;
  if (k->n_atab + new_atab > MAXTAB || k->n_mix + (int)mixed_groups.size() > MAXMIX) return false;
  k->base += c0 * st;
  // biased part: coef*st*(atom - b) >= 0 with b = alo (coef > 0) or ahi (coef < 0)
  auto biased = [&](const Part& q, int64_t* bias) {
    *bias = q.coef > 0 ? q.alo : q.ahi;
    k->base += q.coef * st * *bias;
    return *bias == 0 ? q.atom : c_bin(COp::Sub, q.atom, c_const(*bias));
  };
  TabSpec atab;
  std::map<std::vector<int>, TabSpec> mtabs;
  for (auto& q : ps) {
    const bool ax = q.deps.back() < A, rd = q.deps.front() >= A;
    if (ax && q.atom->op == COp::Loop) {
      k->lin[q.atom->loop] += q.coef * st;
      continue;
    }
    int64_t bias;
    CE e = biased(q, &bias);
    if (rd) {
      rprogs->push_back({e, 0, q.coef * st});
    } else if (ax) {
      atab.progs.push_back({e, 0, q.coef * st});
    } else {
      TabSpec& t = mtabs[q.deps];
      t.progs.push_back({e, 0, q.coef * st});
    }
  }
  if (!atab.progs.empty()) {
    std::set<int> u(axis_deps.begin(), axis_deps.end());
    atab.deps.assign(u.begin(), u.end());
    add_fix_table(s, std::move(atab), k, true, A, tabs, fix);
  }
  for (auto& [deps, t] : mtabs) {
    t.deps = deps;
    add_fix_table(s, std::move(t), k, false, A, tabs, fix);
  }
  return true;
}

static void build_kterm(const CStage& s, const CTerm& t, KTerm* k, std::vector<TabSpec>* tabs,
                        std::vector<Fixup>* fix, bool* dead) {
  memset(k, 0, sizeof(KTerm));
  const int A = (int)s.axis_ext.size();
  const int L = s.nloops();
  k->kind = t.t.kind == TK_PHANTOM ? 2 : (t.t.kind == TK_STAGE || t.t.kind == TK_DSTAGE || t.t.kind == TK_SCRATCH || t.t.kind == TK_PRE ? 1 : 0);
  if (t.t.numel() >= (int64_t)INT32_MAX) fail(SYNO_E_UNSUPPORTED, "tensor has 2^31 or more elements");
  auto strides = row_major_strides(t.t.extents);
  if (t.coords.size() != t.t.extents.size()) fail(SYNO_E_SHAPE, "access rank does not match tensor rank");
  std::vector<ProgSpec> rprogs;
  std::vector<int> all_red;
  std::vector<int64_t> red_ext;
  int64_t R = 1;
  for (int l = A; l < L; ++l) {
    all_red.push_back(l);
    red_ext.push_back(s.ext(l));
    R *= s.ext(l);
  }
  for (size_t d = 0; d < t.coords.size(); ++d) {
    const CE& c = t.coords[d];
    int64_t n = t.t.extents[d], st = strides[d];
    std::vector<int> deps;
    c_loops(c, &deps);
    if (deps.empty()) {
      int64_t v = c_eval(c, nullptr);
      if (v < 0 || v >= n) *dead = true;
      else k->base += v * st;
      continue;
    }
    if (c->op == COp::Loop && n >= s.ext(c->loop)) {
      if (c->loop < A) k->lin[c->loop] += st;
      else rprogs.push_back({c, 0, st});
      continue;
    }
    bool axis_only = deps.back() < A, red_only = deps.front() >= A;
    if (!axis_only && !red_only && split_in_range(s, c, n, st, A, k, tabs, fix, &rprogs)) continue;
    if (red_only) {
      rprogs.push_back({c, n, st});
      continue;
    }
    TabSpec tab;
    tab.deps = deps;
    tab.progs.push_back({c, n, st});
    add_fix_table(s, std::move(tab), k, axis_only, A, tabs, fix);
  }
  if (!rprogs.empty()) {
    TabSpec rt;
    rt.deps = all_red;
    rt.dep_ext = red_ext;
    rt.count = R;
    rt.progs = rprogs;
    fix->push_back({&k->rtab, (int)tabs->size()});
    tabs->push_back(rt);
  }
}

// Linear-form compression of a mixed table.  A coordinate such as
//     (L3 + ((L1 + L2) + 640) // 768) - 3          (L1, L2 axes, L3 a reduce)
// reads its axis loops only through one linear form u = L1 + L2 + 640; its
// table then needs one entry per (u, reduce) -- 3327 x 1024 -- instead of
// one per (L1, L2, reduce) -- 1024 x 2304 x 1024, over the table budget.  The
// table is built over a virtual loop V = u - u_min (loop id nloops()), and
// the axes index it with strides c_a * stride(V).
struct LinForm {
  std::vector<std::pair<int, int64_t>> coef;  // (axis loop, coefficient of u)
  int64_t k0 = 0, umin = 0, ext = 0;
  CE expr;  // the coordinate with u replaced by (V + umin)
};

static bool linear_node(const CE& e) {
  switch (e->op) {
    case COp::Loop:
    case COp::Const: return true;
    case COp::Add:
    case COp::Sub: return linear_node(e->lhs) && linear_node(e->rhs);
    case COp::Mul:
      return (e->lhs->op == COp::Const && linear_node(e->rhs)) || (e->rhs->op == COp::Const && linear_node(e->lhs));
    default: return false;
  }
}

static void all_nodes(const CE& e, std::vector<CE>* out) {
  out->push_back(e);
  if (e->lhs) all_nodes(e->lhs, out);
  if (e->rhs) all_nodes(e->rhs, out);
}

static CE replace_node(const CE& e, const std::string& key, const CE& repl) {
  if (c_render(e) == key) return repl;
  if (!e->lhs) return e;
  return c_bin(e->op, replace_node(e->lhs, key, repl), replace_node(e->rhs, key, repl));
}

static bool linear_form(const CStage& s, const CE& c, int A, LinForm* f) {
  static const bool off = getenv("SYNO_NO_LINFORM") != nullptr;  // A/B switch
  if (off) return false;
  const int L = s.nloops();
  std::vector<int> deps, axd;
  c_loops(c, &deps);
  for (int l : deps)
    if (l < A) axd.push_back(l);
  if (axd.size() < 2) return false;
  std::vector<CE> nodes;
  all_nodes(c, &nodes);
  std::sort(nodes.begin(), nodes.end(),
            [](const CE& a, const CE& b) { return c_render(a).size() > c_render(b).size(); });
  for (const CE& n : nodes) {
    std::vector<int> nl;
    c_loops(n, &nl);
    if (nl != axd || !linear_node(n)) continue;
    const std::string key = c_render(n);
    std::vector<int> rest;
    c_loops(replace_node(c, key, c_const(0)), &rest);
    bool clean = true;
    for (int l : rest) clean = clean && l >= A;
    if (!clean) continue;
    std::vector<int64_t> v(L + 1, 0);
    f->k0 = c_eval(n, v.data());
    f->coef.clear();
    int64_t lo = f->k0, hi = f->k0;
    for (int a : axd) {
      v.assign(L + 1, 0);
      v[a] = 1;
      const int64_t ca = c_eval(n, v.data()) - f->k0;
      f->coef.push_back({a, ca});
      lo += std::min<int64_t>(0, ca * (s.ext(a) - 1));
      hi += std::max<int64_t>(0, ca * (s.ext(a) - 1));
    }
    // linear check at the corners of the axis ranges
    v.assign(L + 1, 0);
    int64_t want = f->k0;
    for (auto& p : f->coef) {
      v[p.first] = s.ext(p.first) - 1;
      want += p.second * (s.ext(p.first) - 1);
    }
    if (c_eval(n, v.data()) != want) continue;
    f->umin = lo;
    f->ext = hi - lo + 1;
    f->expr = replace_node(c, key, c_bin(COp::Add, c_loop(L), c_const(lo)));
    return true;
  }
  return false;
}

static void add_fix_table(const CStage& s, TabSpec&& tab, KTerm* k, bool axis_only, int A,
                          std::vector<TabSpec>* tabs, std::vector<Fixup>* fix) {
  std::vector<int> deps = tab.deps;
  tab.dep_ext.clear();
  tab.count = 1;
  for (int l : deps) {
    tab.dep_ext.push_back(s.ext(l));
    tab.count *= s.ext(l);
  }
  LinForm lf;
  bool lin = false;
  // tables of 2^24 entries or more (SYNO_LINFORM_MIN lowers it for the parity tests)
  static const double lin_min = getenv("SYNO_LINFORM_MIN") ? atof(getenv("SYNO_LINFORM_MIN")) : 16777216.0;
  if (!axis_only && (double)tab.count >= lin_min && tab.progs.size() == 1 && linear_form(s, tab.progs[0].e, A, &lf)) {
    std::vector<int> d2{s.nloops()};
    std::vector<int64_t> e2{lf.ext};
    int64_t n2 = lf.ext;
    for (int l : deps)
      if (l >= A) {
        d2.push_back(l);
        e2.push_back(s.ext(l));
        n2 *= s.ext(l);
      }
    if (n2 * 4 <= tab.count || lin_min < 16777216.0) {
      lin = true;
      deps = d2;
      tab.deps = d2;
      tab.dep_ext = e2;
      tab.count = n2;
      tab.progs[0].e = lf.expr;
    }
  }
  if (tab.count >= table_limit()) fail(SYNO_E_UNSUPPORTED, "index table too large");
  auto tstr = row_major_strides(tab.dep_ext);
  int tid = (int)tabs->size();
  tabs->push_back(tab);
  if (axis_only) {
    if (k->n_atab >= MAXTAB) fail(SYNO_E_UNSUPPORTED, "too many axis tables in one term");
    int m = k->n_atab++;
    for (size_t q = 0; q < deps.size(); ++q) k->atab_s[m][deps[q]] = (int32_t)tstr[q];
    fix->push_back({&k->atab[m], tid});
    return;
  }
  if (k->n_mix >= MAXMIX) fail(SYNO_E_UNSUPPORTED, "too many mixed tables in one term");
  int m = k->n_mix++;
  CE ri = c_const(0);
  for (size_t q = 0; q < deps.size(); ++q) {
    if (lin && q == 0) {
      // the virtual loop V = u - umin: axes index it through u's coefficients
      for (auto& p : lf.coef) k->mtab_s[m][p.first] += (int32_t)(p.second * tstr[0]);
      ri = c_bin(COp::Add, ri, c_const((lf.k0 - lf.umin) * tstr[0]));
    } else if (deps[q] < A) {
      k->mtab_s[m][deps[q]] = (int32_t)tstr[q];
    } else {
      ri = c_bin(COp::Add, ri, c_bin(COp::Mul, c_loop(deps[q]), c_const(tstr[q])));
    }
  }
  fix->push_back({&k->mtab[m], tid});
  std::vector<int> all_red;
  std::vector<int64_t> red_ext;
  int64_t R = 1;
  for (int l = A; l < s.nloops(); ++l) {
    all_red.push_back(l);
    red_ext.push_back(s.ext(l));
    R *= s.ext(l);
  }
  TabSpec rt;
  rt.deps = all_red;
  rt.dep_ext = red_ext;
  rt.count = R;
  rt.progs.push_back({ri, 0, 1});
  fix->push_back({&k->mri[m], (int)tabs->size()});
  tabs->push_back(rt);
}

void release_dev_stage(DevStage& ds) {
  // callers have synchronised the device (DevPlan / TcPlan teardown)
  if (ds.tile && ds.tile->finish) release_dev_stage(*ds.tile->finish);
  ds.tile.reset();
  if (ds.pre) release_dev_stage(*ds.pre);
  ds.pre.reset();
  if (ds.perm_in) release_dev_stage(*ds.perm_in);
  ds.perm_in.reset();
  if (ds.perm_out) release_dev_stage(*ds.perm_out);
  ds.perm_out.reset();
  if (ds.gpre) release_dev_stage(*ds.gpre);
  ds.gpre.reset();
  if (ds.tables) cudaFreeAsync(ds.tables, nullptr);
  ds.tables = nullptr;
  if (ds.prog) cudaFree(ds.prog);
  ds.prog = nullptr;
}

// Program fallback: every coordinate of every term is kept as postfix code
// over the loop digits (axes, then reduces) and evaluated per grid point.
static void build_prog_stage(const CStage& cs, DevStage* ds) {
  KStage& k = ds->k;
  const int L = cs.nloops();
  if ((int)cs.red_ext.size() > 16) fail(SYNO_E_UNSUPPORTED, "stage has too many reduces for the program fallback");
  std::vector<int> loops(L);
  for (int l = 0; l < L; ++l) loops[l] = l;
  std::vector<int64_t> meta, code;
  std::vector<const CTerm*> terms;
  for (auto& t : cs.terms) terms.push_back(&t);
  if (cs.scatter) terms.push_back(&cs.target);
  std::vector<std::vector<int64_t>> recs;
  for (size_t ti = 0; ti < terms.size(); ++ti) {
    const CTerm& t = *terms[ti];
    auto strides = row_major_strides(t.t.extents);
    std::vector<int64_t> rec{(int64_t)t.coords.size()};
    for (size_t d = 0; d < t.coords.size(); ++d) {
      if (prog_depth(t.coords[d]) > MAXSTACK) fail(SYNO_E_UNSUPPORTED, "coordinate expression too deep");
      const int64_t off = (int64_t)code.size();
      compile_prog(t.coords[d], loops, &code);
      rec.push_back(off);
      rec.push_back(((int64_t)code.size() - off) / 2);
      rec.push_back(t.t.extents[d]);
      rec.push_back(strides[d]);
    }
    recs.push_back(rec);
  }
  for (size_t ti = 0; ti < recs.size(); ++ti) {
    k.prog_term_off[ti] = (int32_t)meta.size();
    meta.insert(meta.end(), recs[ti].begin(), recs[ti].end());
  }
  // code offsets become absolute (code follows the metadata)
  const int64_t base = (int64_t)meta.size();
  for (size_t ti = 0; ti < recs.size(); ++ti) {
    int64_t* r = meta.data() + k.prog_term_off[ti];
    for (int64_t d = 0; d < r[0]; ++d) r[1 + 4 * d] += base;
  }
  meta.insert(meta.end(), code.begin(), code.end());
  cuda_check(cudaMalloc((void**)&ds->prog, meta.size() * sizeof(int64_t)), "cudaMalloc(programs)");
  cuda_check(cudaMemcpy(ds->prog, meta.data(), meta.size() * sizeof(int64_t), cudaMemcpyHostToDevice),
             "cudaMemcpy(programs)");
  k.prog = ds->prog;
  k.n_red = (int)cs.red_ext.size();
  for (size_t r = 0; r < cs.red_ext.size(); ++r) k.red_ext[r] = cs.red_ext[r];
  for (int t = 0; t < k.n_terms; ++t) {
    KTerm& kt = k.terms[t];
    memset(&kt, 0, sizeof(KTerm));
    const int tk = cs.terms[t].t.kind;
    kt.kind = tk == TK_PHANTOM ? 2 : (tk == TK_STAGE || tk == TK_DSTAGE || tk == TK_SCRATCH || tk == TK_PRE ? 1 : 0);
  }
  memset(&k.target, 0, sizeof(KTerm));
}

static void build_dev_stage_impl(const CStage& cs, DevStage* ds, cudaStream_t stream, bool allow_tile);

// Lane-contiguous layout for heavy gather stages.  The tile kernel's lanes
// run along the stage axis the lead gathered term's LAST coordinate reads;
// when that coordinate does not advance by one along any stage axis (e.g.
// x[b, (32 co + h + r) % 64, ..., (s // 64 + 16) % 32]: lanes walk a 4 KB
// channel stride), but another coordinate does, the input is copied once
// with that dimension innermost and the stage reads the copy: a warp's
// gathers then touch one or two 32-byte sectors instead of 32.
// SYNO_NO_PERM=1 disables (A/B switch).
static bool lane_contiguous_layout(const CStage& cs, CStage* main, CStage* perm, int64_t* count) {
  static const bool off = getenv("SYNO_NO_PERM") != nullptr;
  // heavy stages only (an extra copy launch); SYNO_PERM_MIN_POINTS lowers
  // the threshold so the parity tests exercise the transform at small sizes
  static const double min_points = getenv("SYNO_PERM_MIN_POINTS") ? atof(getenv("SYNO_PERM_MIN_POINTS")) : 4194304.0;
  if (off || cs.grid_points() < min_points) return false;
  const int A = (int)cs.axis_ext.size(), L = cs.nloops();
  // lead term: for a scatter its target; else the first input (operator
  // dtype) whose coordinates move with a reduce
  int lead = -1;
  if (cs.scatter) {
    if (cs.target.t.kind != TK_DX && cs.target.t.kind != TK_DW) return false;
    lead = 0;
  }
  for (size_t t = 0; t < cs.terms.size() && lead < 0; ++t) {
    const CTerm& T = cs.terms[t];
    if (T.t.kind != TK_X && T.t.kind != TK_W && T.t.kind != TK_DY) continue;
    for (auto& c : T.coords) {
      std::vector<int> d;
      c_loops(c, &d);
      for (int l : d)
        if (l >= A) lead = (int)t;
    }
  }
  if (lead < 0) return false;
  const CTerm& T = cs.scatter ? cs.target : cs.terms[lead];
  const int D = (int)T.coords.size();
  if (D < 2 || T.t.numel() > ((int64_t)1 << 28)) return false;
  // unit-stride score of coordinate d as the LAST coordinate: the tile
  // planner's lanes then walk the highest stage axis l it reads, so the score
  // is how often coord(l + 1) - coord(l) == 1 at random grid points
  uint64_t seed = 0x9e3779b97f4a7c15ull;
  auto rnd = [&](int64_t n) {
    seed ^= seed << 13;
    seed ^= seed >> 7;
    seed ^= seed << 17;
    return (int64_t)(seed % (uint64_t)n);
  };
  auto score = [&](int d) {
    std::vector<int> dl;
    c_loops(T.coords[d], &dl);
    int lane = -1;
    for (int l : dl)
      if (l < A) lane = std::max(lane, l);
    double best = 0;
    for (int l : dl) {
      if (l != lane || cs.ext(l) < 2) continue;
      int hit = 0;
      const int n = 128;
      std::vector<int64_t> v(L);
      for (int i = 0; i < n; ++i) {
        for (int q = 0; q < L; ++q) v[q] = rnd(cs.ext(q));
        v[l] = rnd(cs.ext(l) - 1);
        const int64_t a = c_eval(T.coords[d], v.data());
        ++v[l];
        hit += c_eval(T.coords[d], v.data()) - a == 1;
      }
      best = std::max(best, (double)hit / n);
    }
    return best;
  };
  static const bool log = getenv("SYNO_PERM_LOG") != nullptr;
  const double last = score(D - 1);
  if (log) fprintf(stderr, "[perm] stage %s\n[perm] lead term %d, last-coordinate score %.2f\n", cs.describe().c_str(), lead, last);
  if (last >= 0.5) return false;
  int dstar = -1;
  double bs = 0.75;
  for (int d = 0; d + 1 < D; ++d) {
    const double sc = score(d);
    if (log) fprintf(stderr, "[perm]   coordinate %d score %.2f\n", d, sc);
    if (sc >= bs) {
      bs = sc;
      dstar = d;
    }
  }
  if (dstar < 0) return false;
  std::vector<int> order;  // new dimension k holds old dimension order[k]
  for (int d = 0; d < D; ++d)
    if (d != dstar) order.push_back(d);
  order.push_back(dstar);
  CTensor P;
  P.kind = TK_PERM;
  for (int k = 0; k < D; ++k) P.extents.push_back(T.t.extents[order[k]]);
  if (cs.scatter) {
    // accumulate into P (permuted target, accumulator precision); restore:
    // target[j] = P[i] with i_k = j[order[k]] (an affine stage over the target)
    *main = cs;
    P.kind = TK_SCRATCH;
    std::vector<CE> c2;
    for (int k = 0; k < D; ++k) c2.push_back(cs.target.coords[order[k]]);
    main->target.coords = c2;
    main->target.t = P;
    // cs.out keeps the target tensor: callers dispatch on it (dx / dw_j /
    // an intermediate's gradient); the sums have its element count
    *perm = CStage();
    perm->axis_ext = T.t.extents;
    CTerm src;
    src.t = P;
    for (int k = 0; k < D; ++k) src.coords.push_back(c_loop(order[k]));
    perm->terms.push_back(src);
    perm->out = T.t;
    *count = P.numel();
    return true;
  }
  // the copy: P[i_0..i_{D-1}] = T[j] with j[order[k]] = i_k (an affine stage)
  *perm = CStage();
  perm->axis_ext = P.extents;
  CTerm src;
  src.t = T.t;
  src.coords.resize(D);
  for (int k = 0; k < D; ++k) src.coords[order[k]] = c_loop(k);
  perm->terms.push_back(src);
  perm->out = P;
  // every term of the stage that reads the same tensor reads the copy
  *main = cs;
  for (auto& U : main->terms) {
    if (!(U.t == T.t)) continue;
    std::vector<CE> c2;
    for (int k = 0; k < D; ++k) c2.push_back(U.coords[order[k]]);
    U.coords = c2;
    U.t = P;
  }
  *count = P.numel();
  return true;
}

void build_dev_stage(const CStage& cs, DevStage* ds, cudaStream_t stream) {
  CStage main_cs, perm_cs;
  int64_t count = 0;
  if (lane_contiguous_layout(cs, &main_cs, &perm_cs, &count)) {
    auto pst = std::make_shared<DevStage>();
    build_dev_stage_impl(perm_cs, pst.get(), stream, false);
    (cs.scatter ? ds->perm_out : ds->perm_in) = pst;
    ds->perm_count = count;
    build_dev_stage_impl(main_cs, ds, stream, true);
    return;
  }
  build_dev_stage_impl(cs, ds, stream, true);
}

// The tiled gather form of a gather stage (TileArgs, engine.hpp), decided
// from the built terms: reduce-dependent terms are those with a reduce or
// mixed table; F = axes their mixed tables read, I = other axes they read,
// B = the rest.  The finish stage (axes = the stage's, one reduce over the
// splits) reads the scratch sums as a TK_SCRATCH term and multiplies in the
// reduce-invariant terms.
static void build_tile(const CStage& cs, DevStage* ds, cudaStream_t stream) {
  static const bool off = getenv("SYNO_NO_TILE") != nullptr;  // A/B switch
  const KStage& k = ds->k;
  if (off || k.prog || ds->dead || k.R < 8 || k.out_count == 0) return;
  const bool scatter = cs.scatter;
  const int A = k.n_axes;
  std::vector<int> rt, inv;
  std::vector<bool> inF(A, false), inI(A, false);
  auto mixed_axes = [&](const KTerm& T) {
    for (int m = 0; m < T.n_mix; ++m)
      for (int a = 0; a < A; ++a) inF[a] = inF[a] || T.mtab_s[m][a] != 0;
  };
  for (int t = 0; t < k.n_terms; ++t) {
    const KTerm& T = k.terms[t];
    if (!T.rtab && T.n_mix == 0) {
      inv.push_back(t);
      continue;
    }
    rt.push_back(t);
    mixed_axes(T);
  }
  if (scatter) {
    // the target must move with the reduce (else the sum belongs in a gather)
    if (!k.target.rtab && k.target.n_mix == 0) return;
    mixed_axes(k.target);
  } else if (rt.empty()) {
    return;
  }
  auto thread_axes = [&](const KTerm& T) {
    for (int a = 0; a < A; ++a) {
      bool used = T.lin[a] != 0;
      for (int m = 0; m < T.n_atab; ++m) used = used || T.atab_s[m][a] != 0;
      inI[a] = inI[a] || (used && !inF[a]);
    }
  };
  for (int t : rt) thread_axes(k.terms[t]);
  if (scatter) {
    // every grid point contributes: all axes are enumerated (F or I)
    for (int a = 0; a < A; ++a) inI[a] = !inF[a];
  }
  auto info = std::make_shared<TileInfo>();
  TileArgs& a = info->a;
  memset(&a, 0, sizeof(a));
  a.scatter = scatter ? 1 : 0;
  // lanes should walk the axis the first loaded reduce-dependent term reads
  // contiguously (its last coordinate) -- for a scatter the target's, so the
  // atomics of a warp hit neighbouring words: that axis goes innermost of its
  // group and, when it is an F axis, the lanes run along F
  int contig = -1;
  const CTerm* lead = scatter ? &cs.target : nullptr;
  for (int t : rt) {
    if (lead) break;
    if (k.terms[t].kind != 2) lead = &cs.terms[t];
  }
  if (lead && !lead->coords.empty()) {
    std::vector<int> d;
    c_loops(lead->coords.back(), &d);
    for (int l : d)
      if (l < A && (inF[l] || inI[l])) contig = l;  // the highest such axis
  }
  std::vector<int> forder, iorder;
  for (int x = 0; x < A; ++x) {
    if (x == contig) continue;
    if (inF[x]) forder.push_back(x);
    else if (inI[x]) iorder.push_back(x);
  }
  if (contig >= 0) (inF[contig] ? forder : iorder).push_back(contig);
  a.ffast = contig >= 0 && inF[contig] ? 1 : 0;
  int64_t NF = 1, NI = 1;
  for (int x : forder) {
    a.faxis[a.nF] = x;
    a.fext[a.nF++] = (int32_t)k.axis_ext[x];
    NF *= k.axis_ext[x];
  }
  for (int x : iorder) {
    a.iaxis[a.nI] = x;
    a.iext[a.nI++] = (int32_t)k.axis_ext[x];
    NI *= k.axis_ext[x];
  }
  if (NF * NI >= (int64_t)1 << 30) return;
  a.NF = (int32_t)NF;
  a.NI = (int32_t)NI;
  if (scatter) rt.push_back(-1);  // the target's row comes last
  if ((int)rt.size() > MAXT) return;
  a.n_rt = (int32_t)rt.size();
  for (size_t q = 0; q < rt.size(); ++q) a.rterm[q] = rt[q];
  if (scatter) {
    a.n_inv = (int32_t)inv.size();
    for (size_t q = 0; q < inv.size(); ++q) a.inv[q] = inv[q];
  }
  if (a.ffast) {
    // one warp of F combinations; the rest of the CTA along I reuses the rows
    a.TF = (int32_t)std::min<int64_t>(NF, 32);
    a.TI = (int32_t)std::min<int64_t>(NI, 256 / a.TF);
  } else {
    a.TI = (int32_t)std::min<int64_t>(NI, 256);
    a.TF = (int32_t)std::min<int64_t>(NF, 256 / a.TI);
  }
  // a gather whose rows no I axis shares (TI = 1: every row entry serves one
  // product) gains nothing from staging rows: the per-thread / block forms
  // compute the same offsets without the shared-memory round trip
  static const bool tile_ti1 = getenv("SYNO_TILE_TI1") != nullptr;  // A/B switch
  if (!scatter && a.TI == 1 && !tile_ti1) return;
  a.TR = (int32_t)std::max<int64_t>(1, std::min<int64_t>({256 / (a.TI * a.TF), 64, k.R}));
  a.nIb = (int32_t)((NI + a.TI - 1) / a.TI);
  const int64_t budget = 40 * 1024 / 4;  // int32 row entries per chunk
  a.RC = (int32_t)std::max<int64_t>(8, std::min<int64_t>({k.R, budget / ((int64_t)a.n_rt * a.TF) - 1, 1024}));
  // the rows' pitch (RC + 1) must be odd: with lanes along F a warp reads 32
  // rows at one reduce index, and an even pitch such as 320 put all 32 reads
  // in one shared-memory bank (ncu: ~31 conflicts per load)
  if (a.RC % 2 == 1 && a.RC > 8) a.RC -= 1;
  info->ctas = (int64_t)a.nIb * ((NF + a.TF - 1) / a.TF);
  const int64_t want = 148 * 4;
  int64_t S = std::max<int64_t>(1, (want + info->ctas - 1) / info->ctas);
  S = std::min<int64_t>({S, std::max<int64_t>(1, k.R / std::max<int32_t>(a.RC, 32)), 65535});
  const int64_t r_chunk = (k.R + S - 1) / S;
  S = (k.R + r_chunk - 1) / r_chunk;
  info->splits = S;
  info->smem = std::max<size_t>((size_t)a.n_rt * a.TF * (a.RC + 1) * 4, 256 * 8);
  if (scatter) {  // contributions go straight to the fixed-point sums: no finish stage
    ds->tile = info;
    return;
  }
  // finish stage: out[axes] = scale * sum_s acc[s, F, I] * prod(reduce-invariant terms)
  CStage fin;
  fin.axis_ext = cs.axis_ext;
  fin.red_ext = {S};
  fin.scale = cs.scale;
  fin.out = cs.out;
  CTerm acc;
  acc.t.kind = TK_SCRATCH;
  acc.t.extents = {S};
  acc.coords = {c_loop(A)};
  for (int q = 0; q < a.nF; ++q) {
    acc.t.extents.push_back(a.fext[q]);
    acc.coords.push_back(c_loop(a.faxis[q]));
  }
  for (int q = 0; q < a.nI; ++q) {
    acc.t.extents.push_back(a.iext[q]);
    acc.coords.push_back(c_loop(a.iaxis[q]));
  }
  fin.terms.push_back(acc);
  for (int t = 0; t < k.n_terms; ++t)
    if (std::find(rt.begin(), rt.end(), t) == rt.end()) fin.terms.push_back(cs.terms[t]);
  info->finish = std::make_shared<DevStage>();
  build_dev_stage_impl(fin, info->finish.get(), stream, false);
  ds->tile = info;
}

static CE remap_loops(const CE& e, const std::vector<int>& m) {
  if (e->op == COp::Loop) return c_loop(m.at(e->loop));
  if (e->op == COp::Const) return e;
  return c_bin(e->op, remap_loops(e->lhs, m), remap_loops(e->rhs, m));
}

// Scatter pre-reduction (DevStage::pre): with U = axes read by the target or
// by a reduce-dependent term and P = the other axes, the scatter
//     dst[target(U, r)] += scale * prod_{dep}(U, r) * prod_{inv}(U, P)
// summed over P first is
//     g[U] = sum_P prod_{inv}(U, P);  dst[target(U, r)] += scale * g[U] * prod_{dep}(U, r)
// which scatters |P| times fewer points (e.g. a grad-input whose upstream is
// summed over output channels the input never sees).
static bool split_scatter(const CStage& cs, CStage* pre, CStage* main) {
  static const bool off = getenv("SYNO_NO_PREREDUCE") != nullptr;  // A/B switch
  if (off || !cs.scatter) return false;
  const int A = (int)cs.axis_ext.size(), L = cs.nloops();
  std::vector<bool> used(A, false);
  std::vector<bool> rdep(cs.terms.size(), false);
  auto mark = [&](const CTerm& t) {
    for (auto& c : t.coords) {
      std::vector<int> d;
      c_loops(c, &d);
      for (int l : d)
        if (l < A) used[l] = true;
    }
  };
  mark(cs.target);
  for (size_t t = 0; t < cs.terms.size(); ++t) {
    for (auto& c : cs.terms[t].coords) {
      std::vector<int> d;
      c_loops(c, &d);
      for (int l : d) rdep[t] = rdep[t] || l >= A;
    }
    if (rdep[t]) mark(cs.terms[t]);
  }
  std::vector<int> U, P;
  for (int a = 0; a < A; ++a) (used[a] ? U : P).push_back(a);
  if (P.empty()) return false;
  bool any_inv = false;
  for (size_t t = 0; t < cs.terms.size(); ++t) any_inv = any_inv || !rdep[t];
  // loop maps: main = (U, reduces); pre = (U, P)
  std::vector<int> mm(L, -1), pm(L, -1);
  for (size_t q = 0; q < U.size(); ++q) mm[U[q]] = pm[U[q]] = (int)q;
  for (size_t q = 0; q < P.size(); ++q) pm[P[q]] = (int)(U.size() + q);
  for (int l = A; l < L; ++l) mm[l] = (int)U.size() + (l - A);
  *main = CStage();
  main->scatter = true;
  main->out = cs.out;
  main->scale = cs.scale;
  main->red_ext = cs.red_ext;
  for (int a : U) main->axis_ext.push_back(cs.axis_ext[a]);
  auto remap_term = [](const CTerm& t, const std::vector<int>& m) {
    CTerm r = t;
    for (auto& c : r.coords) c = remap_loops(c, m);
    return r;
  };
  if (any_inv) {
    *pre = CStage();
    pre->axis_ext = main->axis_ext;
    for (int a : P) pre->red_ext.push_back(cs.axis_ext[a]);
    for (size_t t = 0; t < cs.terms.size(); ++t)
      if (!rdep[t]) pre->terms.push_back(remap_term(cs.terms[t], pm));
    pre->out.kind = TK_SCRATCH;
    pre->out.extents = main->axis_ext;
    CTerm g;
    g.t.kind = TK_SCRATCH;
    g.t.extents = main->axis_ext;
    for (size_t q = 0; q < U.size(); ++q) g.coords.push_back(c_loop((int)q));
    main->terms.push_back(g);
  } else {
    for (int a : P) main->scale *= (double)cs.axis_ext[a];  // no term reads P: multiplicity
  }
  for (size_t t = 0; t < cs.terms.size(); ++t)
    if (rdep[t]) main->terms.push_back(remap_term(cs.terms[t], mm));
  main->target = remap_term(cs.target, mm);
  return true;
}

// Gather pre-reduction (the reference's rfactor, codegen.py:433-508, applied
// to any gather stage -- gradient stages included): with M a set of terms
// and Q the reduce loops only terms of M read,
//     out[A] = scale * sum_{R \ Q} prod_{t not in M} t * P[loops(M) \ Q],
//     P = sum_Q prod_{t in M} t
// which visits |loops(M) \ Q| * |Q| + |A| * |R \ Q| points instead of
// |A| * |R| (e.g. a weight gradient whose upstream alone reads the output
// channels: 29 G -> 50 M).  Taken when it saves 4x or more.
static bool split_gather(const CStage& cs, CStage* pre, CStage* main) {
  static const bool off = getenv("SYNO_NO_GATHER_PREREDUCE") != nullptr;  // A/B switch
  const int A = (int)cs.axis_ext.size(), L = cs.nloops();
  const int nT = (int)cs.terms.size();
  if (off || cs.scatter || nT < 2 || nT > 30 || L == A) return false;
  // one factored level per stage (a main stage already reads TK_PRE; its own
  // pre stage may factor again)
  for (auto& t : cs.terms)
    if (t.t.kind == TK_PRE) return false;
  std::vector<uint32_t> reads(L, 0);  // terms reading each loop
  for (int t = 0; t < nT; ++t)
    for (auto& c : cs.terms[t].coords) {
      std::vector<int> d;
      c_loops(c, &d);
      for (int l : d) reads[l] |= 1u << t;
    }
  const uint32_t all = (1u << nT) - 1;
  double grid = 1;
  for (int l = 0; l < L; ++l) grid *= (double)cs.ext(l);
  double best = grid / 4.0;
  uint32_t bestM = 0;
  for (int q = A; q < L; ++q) {
    const uint32_t M = reads[q];
    if (!M || M == all) continue;
    double pre_pts = 1, main_pts = 1, psize = 1;
    for (int l = 0; l < L; ++l) {
      const bool inQ = l >= A && reads[l] && (reads[l] & ~M) == 0;
      const bool readM = (reads[l] & M) != 0;
      if (inQ) pre_pts *= (double)cs.ext(l);
      else {
        main_pts *= (double)cs.ext(l);
        if (readM) psize *= (double)cs.ext(l);
      }
    }
    const double cost = psize * pre_pts + main_pts;
    if (cost < best && psize < (double)(1 << 28)) {
      best = cost;
      bestM = M;
    }
  }
  if (!bestM) return false;
  std::vector<int> Ploops, Q, Rrest;
  for (int l = 0; l < L; ++l) {
    const bool inQ = l >= A && reads[l] && (reads[l] & ~bestM) == 0;
    if (inQ) Q.push_back(l);
    else {
      if (reads[l] & bestM) Ploops.push_back(l);
      if (l >= A) Rrest.push_back(l);
    }
  }
  std::vector<int> pm(L, -1), mm(L, -1);
  for (size_t i = 0; i < Ploops.size(); ++i) pm[Ploops[i]] = (int)i;
  for (size_t j = 0; j < Q.size(); ++j) pm[Q[j]] = (int)(Ploops.size() + j);
  for (int a = 0; a < A; ++a) mm[a] = a;
  for (size_t j = 0; j < Rrest.size(); ++j) mm[Rrest[j]] = A + (int)j;
  auto remap_term = [](const CTerm& t, const std::vector<int>& m) {
    CTerm r = t;
    for (auto& c : r.coords) c = remap_loops(c, m);
    return r;
  };
  *pre = CStage();
  for (int l : Ploops) pre->axis_ext.push_back(cs.ext(l));
  for (int l : Q) pre->red_ext.push_back(cs.ext(l));
  for (int t = 0; t < nT; ++t)
    if (bestM >> t & 1) pre->terms.push_back(remap_term(cs.terms[t], pm));
  pre->out.kind = TK_PRE;
  pre->out.extents = pre->axis_ext;
  *main = CStage();
  main->axis_ext = cs.axis_ext;
  for (int l : Rrest) main->red_ext.push_back(cs.ext(l));
  main->out = cs.out;
  main->scale = cs.scale;
  main->dead = cs.dead;
  for (int t = 0; t < nT; ++t)
    if (!(bestM >> t & 1)) main->terms.push_back(remap_term(cs.terms[t], mm));
  CTerm P;
  P.t.kind = TK_PRE;
  P.t.extents = pre->axis_ext;
  for (int l : Ploops) P.coords.push_back(c_loop(mm[l]));
  main->terms.push_back(P);
  return true;
}

static void build_dev_stage_impl(const CStage& cs_in, DevStage* ds, cudaStream_t stream, bool allow_tile) {
  CStage pre_cs, main_cs;
  if (allow_tile && split_gather(cs_in, &pre_cs, &main_cs)) {
    ds->gpre = std::make_shared<DevStage>();
    build_dev_stage_impl(pre_cs, ds->gpre.get(), stream, true);
    ds->gpre_count = pre_cs.out.numel();
    build_dev_stage_impl(main_cs, ds, stream, true);
    return;
  }
  const bool split = allow_tile && split_scatter(cs_in, &pre_cs, &main_cs);
  const CStage& cs = split ? main_cs : cs_in;
  if (split && !pre_cs.terms.empty()) {
    ds->pre = std::make_shared<DevStage>();
    build_dev_stage_impl(pre_cs, ds->pre.get(), stream, true);
  }
  ds->cs = cs;
  KStage& k = ds->k;
  memset(&k, 0, sizeof(KStage));
  if ((int)cs.axis_ext.size() > MAXA) fail(SYNO_E_UNSUPPORTED, "stage has too many axes");
  if ((int)cs.terms.size() > MAXT) fail(SYNO_E_UNSUPPORTED, "stage has too many terms");
  {
    double n = 1;
    for (auto e : cs.axis_ext) n *= (double)e;
    if (n >= 2147483647.0) fail(SYNO_E_UNSUPPORTED, "stage has 2^31 or more outputs");
  }
  k.n_axes = (int)cs.axis_ext.size();
  k.n_terms = (int)cs.terms.size();
  k.out_count = 1;
  for (size_t a = 0; a < cs.axis_ext.size(); ++a) {
    k.axis_ext[a] = cs.axis_ext[a];
    k.out_count *= cs.axis_ext[a];
  }
  k.R = 1;
  for (auto r : cs.red_ext) k.R *= r;
  k.scale = cs.scale;
  std::vector<TabSpec> tabs;
  std::vector<Fixup> fix;
  bool dead = false;
  try {
    for (size_t t = 0; t < cs.terms.size(); ++t) build_kterm(cs, cs.terms[t], &k.terms[t], &tabs, &fix, &dead);
    if (cs.scatter) build_kterm(cs, cs.target, &k.target, &tabs, &fix, &dead);
  } catch (const Error& e) {
    if (e.code != SYNO_E_UNSUPPORTED) throw;
    // table budget exceeded: evaluate the coordinate programs on the fly
    static const bool log = getenv("SYNO_PROG_LOG") != nullptr;
    if (log) fprintf(stderr, "[prog] %s (%s)\n", cs.describe().c_str(), e.what());
    ds->dead = cs.dead;
    build_prog_stage(cs, ds);
    return;
  }
  ds->dead = dead || cs.dead;
  size_t total = 0;
  for (auto& t : tabs) {
    t.offset = total;
    total += (size_t)t.count;
  }
  ds->table_entries = total;
  if (total) {
    cuda_check(cudaMallocAsync((void**)&ds->tables, total * sizeof(int32_t), stream), "cudaMallocAsync(tables)");
    for (auto& t : tabs) launch_k1(t, ds->tables + t.offset, nullptr, stream);
  }
  for (auto& f : fix) *f.field = ds->tables + tabs[f.table].offset;
  if (allow_tile) build_tile(cs, ds, stream);
}

DevPlan::~DevPlan() {
  // in-flight work on any stream may still read the tables
  int cur = -1;
  cudaGetDevice(&cur);
  if (device >= 0 && device != cur) cudaSetDevice(device);
  cudaDeviceSynchronize();
  auto rel = [](std::vector<DevStage>& v) {
    for (auto& s : v) release_dev_stage(s);
  };
  rel(forward);
  rel(grad_x);
  rel(bwd_staged);
  for (auto& g : grad_w) rel(g);
  tc.reset();
  gg.reset();
  for (cudaEvent_t e : {ev_plan, ev_fwd, ev_bwd})
    if (e) cudaEventDestroy(e);
  if (device >= 0 && device != cur && cur >= 0) cudaSetDevice(cur);
}

void wait_built(cudaEvent_t ev, cudaStream_t stream) {
  if (!ev) return;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &st);
  if (st != cudaStreamCaptureStatusNone) return;  // built before the capture on this stream
  cuda_check(cudaStreamWaitEvent(stream, ev, 0), "cudaStreamWaitEvent(plan built)");
}

static cudaEvent_t record_built(cudaStream_t stream) {
  cudaEvent_t ev;
  cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate(built)");
  cuda_check(cudaEventRecord(ev, stream), "cudaEventRecord(built)");
  return ev;
}

// Tables are filled on the building stream; the readiness event orders any
// other stream after them (wait_built) without a host synchronisation.
static void ensure_forward(const Plan& plan, DevPlan& dp, cudaStream_t stream) {
  {
    std::lock_guard<std::mutex> lock(dp.mu);
    if (!dp.have_forward) {
      for (auto& s : plan.forward) {
        dp.forward.emplace_back();
        build_dev_stage(s, &dp.forward.back(), stream);
      }
      dp.ev_fwd = record_built(stream);
      dp.have_forward = true;
    }
  }
  wait_built(dp.ev_fwd, stream);
}

static void ensure_backward(const Plan& plan, DevPlan& dp, cudaStream_t stream) {
  {
    std::lock_guard<std::mutex> lock(dp.mu);
    if (!dp.have_backward) {
      if (!plan.bwd_staged.empty()) {
        for (auto& s : plan.bwd_staged) {
          dp.bwd_staged.emplace_back();
          build_dev_stage(s, &dp.bwd_staged.back(), stream);
        }
      } else {
        for (auto& s : plan.grad_x) {
          dp.grad_x.emplace_back();
          build_dev_stage(s, &dp.grad_x.back(), stream);
        }
        for (auto& gw : plan.grad_w) {
          dp.grad_w.emplace_back();
          for (auto& s : gw) {
            dp.grad_w.back().emplace_back();
            build_dev_stage(s, &dp.grad_w.back().back(), stream);
          }
        }
      }
      dp.ev_bwd = record_built(stream);
      dp.have_backward = true;
    }
  }
  wait_built(dp.ev_bwd, stream);
}

static std::shared_ptr<GatherGemm> gg_build(const Plan& plan, cudaStream_t stream);

bool staged_cheaper(const Plan& plan) {
  static const bool tc_unstaged = getenv("SYNO_TC_UNSTAGED") != nullptr;
  return !tc_unstaged && plan.forward.size() > 1 && !plan.bwd_staged.empty() &&
         (double)plan.flops_staged * 4.0 < (double)plan.flops_unstaged;
}

DevPlan* build_dev_plan(const Plan& plan, cudaStream_t stream) {
  auto dp = std::make_unique<DevPlan>();
  cuda_check(cudaGetDevice(&dp->device), "cudaGetDevice");
  {
    // keep stream-ordered allocations (tables, stage buffers, partials) cached
    static std::atomic<uint64_t> pooled{0};
    const uint64_t bit = 1ull << (dp->device & 63);
    if (!(pooled.fetch_or(bit) & bit)) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dp->device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    }
  }
  // a staged (rfactored) nest with a staged backward that is much cheaper
  // than the unstaged contraction stays on the stage engine: the tensor-core
  // paths compute the unstaged form (e.g. a sampled QKV variant whose staged
  // forward is 0.1 GFLOP against 58 for the dense GEMM).  SYNO_TC_UNSTAGED=1
  // keeps the tensor-core paths for them (A/B switch).
  if (!plan.nest_only && !staged_cheaper(plan)) {
    dp->tc = tc_build(plan, stream);
    if (!dp->tc) dp->gg = gg_build(plan, stream);
  }
  dp->ev_plan = record_built(stream);
  return dp.release();
}

// ---------------------------------------------------------------------------
// Stage kernels
// ---------------------------------------------------------------------------

template <typename T> struct Acc;
template <> struct Acc<float> { using type = float; };
template <> struct Acc<__nv_bfloat16> { using type = float; };
template <> struct Acc<double> { using type = double; };

template <typename TA> __device__ __forceinline__ TA to_acc(float v) { return (TA)v; }
__device__ __forceinline__ float cvt(float v) { return v; }
__device__ __forceinline__ float cvt(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ double cvt(double v) { return v; }

template <typename TO, typename TA> __device__ __forceinline__ TO from_acc(TA v) { return (TO)v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16, float>(float v) { return __float2bfloat16(v); }

template <typename TI, typename TA>
__device__ __forceinline__ TA load_term(const KTerm& T, int64_t off) {
  if (T.kind == 0) return (TA)cvt(__ldg(((const TI*)T.ptr) + off));
  return ((const TA*)T.ptr)[off];
}

__device__ __forceinline__ void term_prep(const KTerm& T, int n_axes, const int32_t* av, int64_t* base, bool* ok,
                                          int32_t* ia) {
  int64_t b = T.base;
  bool good = true;
#pragma unroll
  for (int k = 0; k < MAXA; ++k)
    if (k < n_axes) b += T.lin[k] * av[k];
#pragma unroll
  for (int m = 0; m < MAXTAB; ++m) {
    if (m < T.n_atab) {
      int32_t idx = 0;
#pragma unroll
      for (int k = 0; k < MAXA; ++k)
        if (k < n_axes) idx += T.atab_s[m][k] * av[k];
      int32_t v = __ldg(T.atab[m] + idx);
      good = good && v >= 0;
      b += v;
    }
  }
#pragma unroll
  for (int m = 0; m < MAXMIX; ++m) {
    int32_t idx = 0;
    if (m < T.n_mix) {
#pragma unroll
      for (int k = 0; k < MAXA; ++k)
        if (k < n_axes) idx += T.mtab_s[m][k] * av[k];
    }
    ia[m] = idx;
  }
  *base = b;
  *ok = good;
}

__device__ __forceinline__ bool term_offset(const KTerm& T, int64_t base, bool ok, const int32_t* ia, int64_t r,
                                            int64_t* off) {
  int64_t o = base;
  if (T.rtab) {
    int32_t v = __ldg(T.rtab + r);
    ok = ok && v >= 0;
    o += v;
  }
#pragma unroll
  for (int m = 0; m < MAXMIX; ++m) {
    if (m < T.n_mix) {
      int32_t v = __ldg(T.mtab[m] + ia[m] + __ldg(T.mri[m] + r));
      ok = ok && v >= 0;
      o += v;
    }
  }
  *off = o;
  return ok;
}

// ---------------------------------------------------------------------------
// Deterministic scatter accumulation (reference np.add.at, codegen.py:740-742)
// ---------------------------------------------------------------------------
// Floating-point atomics make the sum's rounding depend on the arrival order,
// so equal inputs could give different low bits run to run (and the search's
// rewards with them).  Integer addition is associative: every contribution is
// rounded ONCE to a fixed-point integer (2^shift units) and added with integer
// atomics, so the result is the same for any order.  The shift is chosen so
// that no partial sum can overflow: |partial| <= fx_mult * prod_t max|term_t|
// (fx_mult = grid points x scale).  fp32 / bf16 use one signed 64-bit word
// (sum < 2^61); f64 a 128-bit (lo, hi) word pair (sum < 2^124), whose carry
// out of the low word is counted exactly once per wrap-around.

template <typename TA> struct FxWide { static constexpr bool value = false; };
template <> struct FxWide<double> { static constexpr bool value = true; };

template <typename TA>
__device__ __forceinline__ int fx_shift(const KStage& S) {
  double b = S.fx_mult;
  for (int i = 0; i < S.fx_n; ++i) b *= S.fx_max[i];
  if (!(b > 0.0) || isinf(b)) return 0;
  int e;
  frexp(b, &e);  // b < 2^e
  const int top = FxWide<TA>::value ? 124 : 61;
  return max(-1000, min(1000, top - e));
}

// The unit 2^sh as a double, computed once per thread: multiplying by an
// exact power of two is the same rounding as ldexp (a library call per
// contribution that dominated the scatter's instruction count).
__device__ __forceinline__ double fx_unit(int sh) { return ldexp(1.0, sh); }

template <typename TA>
__device__ __forceinline__ void fx_add(unsigned long long* fx, int64_t off, double v, double unit) {
  if (!FxWide<TA>::value) {
    atomicAdd(fx + off, (unsigned long long)__double2ll_rn(v * unit));  // round to nearest, as rint
    return;
  }
  const double x = rint(v * unit);
  const double hd = floor(x * 0x1p-64);
  const unsigned long long lo = __double2ull_rn(x - hd * 0x1p64);  // exact, in [0, 2^64)
  const long long hi = __double2ll_rn(hd);
  if (lo) {
    const unsigned long long old = atomicAdd(fx + 2 * off, lo);
    if (old + lo < old) atomicAdd(fx + 2 * off + 1, 1ull);
  }
  if (hi) atomicAdd(fx + 2 * off + 1, (unsigned long long)hi);
}

template <typename TA>
__device__ __forceinline__ double fx_value(const unsigned long long* fx, int64_t i, int sh) {
  if (!FxWide<TA>::value) return ldexp((double)(long long)fx[i], -sh);
  return ldexp((double)(long long)fx[2 * i + 1], 64 - sh) + ldexp((double)fx[2 * i], -sh);
}

struct MaxAbsArgs {
  const void* ptr[MAXT + 1];
  int64_t count[MAXT + 1];
  int32_t acc[MAXT + 1];  // element type: 1 = accumulator dtype, 0 = input dtype
  double* out;            // one max |v| per tensor (zeroed before)
};

// max |v| of each loaded term (blockIdx.y = term): the overflow bound of the
// fixed-point scatter.  atomicMax on the bits of a non-negative double is
// order independent.
template <typename TI, typename TA>
__global__ void __launch_bounds__(256) maxabs_kernel(const __grid_constant__ MaxAbsArgs a) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.y;
  const int64_t n = a.count[t];
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = a.acc[t] ? (double)((const TA*)a.ptr[t])[i] : (double)cvt(((const TI*)a.ptr[t])[i]);
    m = fmax(m, fabs(v));
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, d));
  if ((threadIdx.x & 31) == 0 && m > 0.0)
    atomicMax((unsigned long long*)(a.out + t), (unsigned long long)__double_as_longlong(m));
}

// fixed-point sums -> the scatter's output (accumulator or input dtype)
template <typename TO, typename TA>
__global__ void fx_convert_kernel(const __grid_constant__ KStage S, int64_t count, TO* out) {
  pdl_trigger();
  pdl_wait();
  const int sh = fx_shift<TA>(S);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = from_acc<TO, TA>((TA)fx_value<TA>(S.fx, i, sh));
}

// NT = compile-time bound on the number of terms: fewer live registers and
// higher occupancy for the common 1-3 term stages.
template <typename TI, typename TA, bool SCATTER, int NT>
__global__ void __launch_bounds__(256, NT <= 2 ? 4 : 2) stage_kernel(const __grid_constant__ KStage S) {
  pdl_trigger();
  pdl_wait();
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= S.out_count) return;
  const int64_t r0 = (int64_t)blockIdx.y * S.r_chunk;
  const int64_t r1 = min(S.R, r0 + S.r_chunk);
  int32_t av[MAXA];
  {
    uint32_t rem = (uint32_t)o;  // out_count < 2^31 (checked on the host)
#pragma unroll
    for (int k = MAXA - 1; k >= 0; --k) {
      if (k < S.n_axes) {
        const uint32_t e = (uint32_t)S.axis_ext[k];
        av[k] = (int32_t)(rem % e);
        rem /= e;
      } else {
        av[k] = 0;
      }
    }
  }
  int64_t base[NT];
  bool aok[NT];
  int32_t ia[NT][MAXMIX];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    base[t] = 0;
    aok[t] = false;
    if (t < S.n_terms) term_prep(S.terms[t], S.n_axes, av, &base[t], &aok[t], ia[t]);
  }
  int64_t tbase = 0;
  bool tok = false;
  int32_t tia[MAXMIX];
  if (SCATTER) term_prep(S.target, S.n_axes, av, &tbase, &tok, tia);
  const TA scale = (TA)S.scale;
  const double sh = SCATTER ? fx_unit(fx_shift<TA>(S)) : 1.0;
  TA acc = 0;
  for (int64_t r = r0; r < r1; ++r) {
    TA prod = 1;
    bool ok = true;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      if (t < S.n_terms && ok) {
        const KTerm& T = S.terms[t];
        int64_t off;
        if (!term_offset(T, base[t], aok[t], ia[t], r, &off)) ok = false;
        else if (T.kind != 2) prod *= load_term<TI, TA>(T, off);
      }
    }
    if (SCATTER) {
      int64_t off;
      if (ok && term_offset(S.target, tbase, tok, tia, r, &off)) fx_add<TA>(S.fx, off, (double)(prod * scale), sh);
    } else if (ok) {
      acc += prod;
    }
  }
  if (!SCATTER) {
    if (S.out_acc) ((TA*)S.out)[(int64_t)blockIdx.y * S.out_count * (gridDim.y > 1) + o] = acc * scale;
    else ((TI*)S.out)[o] = from_acc<TI, TA>(acc * scale);
  }
}

// Program fallback (index tables over budget): every coordinate is
// evaluated from its postfix program at every grid point.
__device__ __forceinline__ bool prog_offset(const int64_t* prog, int rec, const int64_t* vals, int64_t* off) {
  const int64_t* r = prog + rec;
  int64_t o = 0;
  bool ok = true;
  for (int64_t d = 0; d < r[0]; ++d) {
    const int64_t* c = r + 1 + 4 * d;
    const int64_t v = eval_prog(prog + c[0], c[1], vals);
    ok = ok && v >= 0 && v < c[2];
    o += v * c[3];
  }
  *off = o;
  return ok;
}

template <typename TI, typename TA, bool SCATTER>
__global__ void __launch_bounds__(128) stage_prog_kernel(const __grid_constant__ KStage S) {
  pdl_trigger();
  pdl_wait();
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= S.out_count) return;
  const int64_t r0 = (int64_t)blockIdx.y * S.r_chunk;
  const int64_t r1 = min(S.R, r0 + S.r_chunk);
  int64_t vals[MAXA + 16];
  {
    int64_t rem = o;
    for (int k = S.n_axes - 1; k >= 0; --k) {
      vals[k] = rem % S.axis_ext[k];
      rem /= S.axis_ext[k];
    }
  }
  const TA scale = (TA)S.scale;
  const double sh = SCATTER ? fx_unit(fx_shift<TA>(S)) : 1.0;
  TA acc = 0;
  for (int64_t r = r0; r < r1; ++r) {
    int64_t rem = r;
    for (int k = S.n_red - 1; k >= 0; --k) {
      vals[S.n_axes + k] = rem % S.red_ext[k];
      rem /= S.red_ext[k];
    }
    TA prod = 1;
    bool ok = true;
    for (int t = 0; t < S.n_terms && ok; ++t) {
      int64_t off;
      if (!prog_offset(S.prog, S.prog_term_off[t], vals, &off)) ok = false;
      else if (S.terms[t].kind != 2) prod *= load_term<TI, TA>(S.terms[t], off);
    }
    if (!ok) continue;
    if (SCATTER) {
      int64_t off;
      if (prog_offset(S.prog, S.prog_term_off[S.n_terms], vals, &off)) fx_add<TA>(S.fx, off, (double)(prod * scale), sh);
    } else {
      acc += prod;
    }
  }
  if (!SCATTER) {
    if (S.out_acc) ((TA*)S.out)[(int64_t)blockIdx.y * S.out_count * (gridDim.y > 1) + o] = acc * scale;
    else ((TI*)S.out)[o] = from_acc<TI, TA>(acc * scale);
  }
}

// Affine form: no reduction and every coordinate a bare iterator (weight
// folds and re-layouts, identity-like gathers): offsets are linear in the
// output digits, so the kernel is a plain strided gather-product.
template <typename TI, typename TA, int NT>
__global__ void __launch_bounds__(256) affine_kernel(const __grid_constant__ KStage S) {
  pdl_trigger();
  pdl_wait();
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= S.out_count) return;
  int64_t off[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) off[t] = t < S.n_terms ? S.terms[t].base : 0;
  uint32_t rem = (uint32_t)o;
#pragma unroll
  for (int k = MAXA - 1; k >= 0; --k) {
    if (k < S.n_axes) {
      const uint32_t e = (uint32_t)S.axis_ext[k];
      const uint32_t d = rem % e;
      rem /= e;
#pragma unroll
      for (int t = 0; t < NT; ++t)
        if (t < S.n_terms) off[t] += S.terms[t].lin[k] * (int64_t)d;
    }
  }
  TA prod = (TA)S.scale;
#pragma unroll
  for (int t = 0; t < NT; ++t)
    if (t < S.n_terms) prod *= load_term<TI, TA>(S.terms[t], off[t]);
  if (S.out_acc) ((TA*)S.out)[o] = prod;
  else ((TI*)S.out)[o] = from_acc<TI, TA>(prod);
}

// K3: block-cooperative form for stages with few outputs and long reductions
// (weight gradients of small weights, pooling to a point): one block per
// output, threads stride the reduce range, warp-shuffle + smem tree reduce.
template <typename TI, typename TA>
__global__ void __launch_bounds__(256) stage_block_kernel(const __grid_constant__ KStage S) {
  pdl_trigger();
  pdl_wait();
  const int64_t o = blockIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * S.r_chunk;
  const int64_t r1 = min(S.R, r0 + S.r_chunk);
  int32_t av[MAXA];
  {
    int64_t rem = o;
#pragma unroll
    for (int k = MAXA - 1; k >= 0; --k) {
      if (k < S.n_axes) {
        int64_t e = S.axis_ext[k];
        av[k] = (int32_t)(rem % e);
        rem /= e;
      } else {
        av[k] = 0;
      }
    }
  }
  int64_t base[MAXT];
  bool aok[MAXT];
  int32_t ia[MAXT][MAXMIX];
#pragma unroll
  for (int t = 0; t < MAXT; ++t) {
    base[t] = 0;
    aok[t] = false;
    if (t < S.n_terms) term_prep(S.terms[t], S.n_axes, av, &base[t], &aok[t], ia[t]);
  }
  TA acc = 0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    TA prod = 1;
    bool ok = true;
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      if (t < S.n_terms && ok) {
        const KTerm& T = S.terms[t];
        int64_t off;
        if (!term_offset(T, base[t], aok[t], ia[t], r, &off)) ok = false;
        else if (T.kind != 2) prod *= load_term<TI, TA>(T, off);
      }
    }
    if (ok) acc += prod;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  __shared__ TA part[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) part[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    acc = lane < (int)(blockDim.x >> 5) ? part[lane] : (TA)0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) {
      const TA v = acc * (TA)S.scale;
      if (S.out_acc) ((TA*)S.out)[(int64_t)blockIdx.y * S.out_count * (gridDim.y > 1) + o] = v;
      else ((TI*)S.out)[o] = from_acc<TI, TA>(v);
    }
  }
}

// Tiled gather form (TileArgs in engine.hpp).  Thread (ti, tf, tr) of CTA
// (ib, fb) owns output (F index fb*TF+tf, I index ib*TI+ti) and every TR-th
// reduce index of each shared-memory chunk.  Per chunk, the CTA first builds
// the offset row of every reduce-dependent term for its TF F-combinations
// (reduce tables + mixed tables indexed by the F digits; -1 = out of range),
// then every thread runs its products reading the rows (one shared load per
// term) plus its own per-thread offset part.  The TR partial sums are added
// in a fixed order: the result is deterministic.
template <typename TI, typename TA, int NT, bool SCATTER>
__global__ void __launch_bounds__(256) stage_tile_kernel(const __grid_constant__ KStage S,
                                                         const __grid_constant__ TileArgs A) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ int32_t srow[];
  const int tid = threadIdx.x;
  const int ti = A.ffast ? (tid / A.TF) % A.TI : tid % A.TI;
  const int tf = A.ffast ? tid % A.TF : (tid / A.TI) % A.TF;
  const int tr = tid / (A.TI * A.TF);
  const int ib = blockIdx.x % A.nIb, fb = blockIdx.x / A.nIb;
  const int i = ib * A.TI + ti, f = fb * A.TF + tf;
  const bool live = i < A.NI && f < A.NF && tr < A.TR;
  int32_t av[MAXA];
#pragma unroll
  for (int k = 0; k < MAXA; ++k) av[k] = 0;
  {
    int rem = live ? i : 0;
    for (int q = A.nI - 1; q >= 0; --q) {
      av[A.iaxis[q]] = rem % A.iext[q];
      rem /= A.iext[q];
    }
    rem = live ? f : 0;
    for (int q = A.nF - 1; q >= 0; --q) {
      av[A.faxis[q]] = rem % A.fext[q];
      rem /= A.fext[q];
    }
  }
  // scatter: the last row is the target's; n_ld terms are loaded per point
  const int n_ld = SCATTER ? A.n_rt - 1 : A.n_rt;
  int64_t base[NT];
  bool aok[NT];
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    base[k] = 0;
    aok[k] = false;
    if (k < n_ld) {
      int32_t ia[MAXMIX];
      term_prep(S.terms[A.rterm[k]], S.n_axes, av, &base[k], &aok[k], ia);
    }
  }
  int64_t tbase = 0;
  bool tok = true;
  TA pre = (TA)S.scale;
  double sh = 1.0;
  if (SCATTER) {
    int32_t ia[MAXMIX];
    term_prep(S.target, S.n_axes, av, &tbase, &tok, ia);
    for (int q = 0; q < A.n_inv && tok; ++q) {
      const KTerm& T = S.terms[A.inv[q]];
      int64_t b0;
      bool ok0;
      term_prep(T, S.n_axes, av, &b0, &ok0, ia);
      if (!ok0) tok = false;
      else if (T.kind != 2) pre *= load_term<TI, TA>(T, b0);
    }
    sh = fx_unit(fx_shift<TA>(S));
  }
  const int64_t r0 = (int64_t)blockIdx.y * S.r_chunk;
  const int64_t r1 = min(S.R, r0 + S.r_chunk);
  const int pitch = A.RC + 1;
  // per-thread view of the loaded terms, hoisted out of the reduce loop:
  // base pointer (term pointer + the thread's offset), dtype and validity
  const void* tp[NT];
  int tk[NT];
  bool any_off = false;
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    tp[k] = nullptr;
    tk[k] = 2;
    if (k < n_ld) {
      const KTerm& T = S.terms[A.rterm[k]];
      tk[k] = T.kind;
      any_off = any_off || !aok[k];
      if (T.kind == 0) tp[k] = static_cast<const TI*>(T.ptr) + base[k];
      else if (T.kind == 1) tp[k] = static_cast<const TA*>(T.ptr) + base[k];
    }
  }
  TA acc = 0;
  // per (row term, F combination): the mixed tables' F-digit offsets, decoded
  // once per CTA (the row loop then needs no divisions by runtime extents)
  __shared__ int32_t fofs[MAXT][MAXMIX][32];
  const bool fofs_ok = A.TF <= 32;
  if (fofs_ok) {
    for (int e = tid; e < A.n_rt * A.TF; e += blockDim.x) {
      const int fl = e % A.TF, k = e / A.TF;
      const KTerm& T = A.rterm[k] < 0 ? S.target : S.terms[A.rterm[k]];
      int32_t fd[MAXA];
      int rem = min(fb * A.TF + fl, A.NF - 1);
      for (int q = A.nF - 1; q >= 0; --q) {
        fd[q] = rem % A.fext[q];
        rem /= A.fext[q];
      }
      for (int m = 0; m < MAXMIX; ++m) {
        int32_t idx = 0;
        if (m < T.n_mix)
          for (int q = 0; q < A.nF; ++q) idx += T.mtab_s[m][A.faxis[q]] * fd[q];
        fofs[k][m][fl] = idx;
      }
    }
  }
  for (int64_t c0 = r0; c0 < r1; c0 += A.RC) {
    const int rc = (int)min((int64_t)A.RC, r1 - c0);
    __syncthreads();
    if (fofs_ok && rc >= 64) {
      // row-major: one (term, F) row at a time, lanes along the reduce index
      for (int row = 0; row < A.n_rt * A.TF; ++row) {
        const int k = row / A.TF, fl = row - k * A.TF;
        const KTerm& T = A.rterm[k] < 0 ? S.target : S.terms[A.rterm[k]];
        const bool fin = fb * A.TF + fl < A.NF;
        for (int rl = tid; rl < rc; rl += blockDim.x) {
          int32_t v = -1;
          if (fin) {
            const int64_t r = c0 + rl;
            bool ok = true;
            int32_t o = 0;
            if (T.rtab) {
              const int32_t x = __ldg(T.rtab + r);
              ok = x >= 0;
              o = x;
            }
            for (int m = 0; m < T.n_mix && ok; ++m) {
              const int32_t x = __ldg(T.mtab[m] + __ldg(T.mri[m] + r) + fofs[k][m][fl]);
              ok = x >= 0;
              o += x;
            }
            v = ok ? o : -1;
          }
          srow[row * pitch + rl] = v;
        }
      }
    } else
    for (int it = tid; it < A.n_rt * A.TF * rc; it += blockDim.x) {
      const int rl = it % rc;
      const int rest = it / rc;
      const int fl = rest % A.TF, k = rest / A.TF;
      const int fg = fb * A.TF + fl;
      int32_t v = -1;
      if (fg < A.NF) {
        const KTerm& T = A.rterm[k] < 0 ? S.target : S.terms[A.rterm[k]];
        const int64_t r = c0 + rl;
        bool ok = true;
        int64_t o = 0;
        if (T.rtab) {
          const int32_t x = __ldg(T.rtab + r);
          ok = x >= 0;
          o = x;
        }
        if (T.n_mix) {
          int32_t fd[MAXA];
          int rem = fg;
          for (int q = A.nF - 1; q >= 0; --q) {
            fd[q] = rem % A.fext[q];
            rem /= A.fext[q];
          }
          for (int m = 0; m < T.n_mix && ok; ++m) {
            int32_t idx = __ldg(T.mri[m] + r);
            for (int q = 0; q < A.nF; ++q) idx += T.mtab_s[m][A.faxis[q]] * fd[q];
            const int32_t x = __ldg(T.mtab[m] + idx);
            ok = x >= 0;
            o += x;
          }
        }
        v = ok ? (int32_t)o : -1;
      }
      srow[(k * A.TF + fl) * pitch + rl] = v;
    }
    __syncthreads();
    if (live && tok && !any_off) {
      for (int rl = tr; rl < rc; rl += A.TR) {
        TA prod = SCATTER ? pre : (TA)1;
        bool ok = true;
#pragma unroll
        for (int k = 0; k < NT; ++k) {
          if (k < n_ld && ok) {
            const int32_t o = srow[(k * A.TF + tf) * pitch + rl];
            if (o < 0) ok = false;
            else if (tk[k] == 0) prod *= (TA)cvt(__ldg(static_cast<const TI*>(tp[k]) + o));
            else if (tk[k] == 1) prod *= static_cast<const TA*>(tp[k])[o];
          }
        }
        if (SCATTER) {
          const int32_t o = srow[(n_ld * A.TF + tf) * pitch + rl];
          if (ok && o >= 0) fx_add<TA>(S.fx, tbase + o, (double)prod, sh);
        } else if (ok) {
          acc += prod;
        }
      }
    }
  }
  if (SCATTER) return;
  // fixed-order combination of the TR partial sums of each output
  __syncthreads();
  TA* red = reinterpret_cast<TA*>(srow);
  red[tid] = acc;
  __syncthreads();
  if (tr == 0 && live) {
    TA s = acc;
    for (int q = 1; q < A.TR; ++q) s += red[tid + q * A.TI * A.TF];
    ((TA*)A.acc)[((int64_t)blockIdx.y * A.NF + f) * A.NI + i] = s;
  }
}

template <typename TO, typename TA>
__global__ void sum_partials(const TA* part, int64_t count, int nsplit, TO* out) {
  pdl_trigger();
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  TA s = 0;
  for (int k = 0; k < nsplit; ++k) s += part[(int64_t)k * count + i];
  out[i] = from_acc<TO, TA>(s);
}

template <typename TO, typename TA>
__global__ void cast_kernel(const TA* in, int64_t count, TO* out) {
  pdl_trigger();
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = from_acc<TO, TA>(in[i]);
}

// ---------------------------------------------------------------------------
// Launch
// ---------------------------------------------------------------------------

static size_t dtype_size(DType dt) { return dt == DT_F64 ? 8 : dt == DT_F32 ? 4 : 2; }
static size_t acc_size(DType dt) { return dt == DT_F64 ? 8 : 4; }

static const void* bind_ptr(const CTensor& t, const Bindings& b) {
  switch (t.kind) {
    case TK_X: return b.x;
    case TK_W: return b.w.at(t.index);
    case TK_STAGE: return b.stages.at(t.index);
    case TK_Y: return b.y;
    case TK_DY: return b.dy;
    case TK_DX: return b.dx;
    case TK_DW: return b.dw.at(t.index);
    case TK_DSTAGE: return b.dstages.at(t.index);
    case TK_SCRATCH:
    case TK_SCRATCH_IN: return b.scratch;
    case TK_PERM: return b.perm;
    case TK_PRE: return b.pre;
    default: return nullptr;
  }
}

template <typename TI, typename TA, bool SCATTER>
static void launch_nt(const KStage& k, dim3 grid, cudaStream_t stream) {
  if (k.prog) {
    dim3 g2((unsigned)((k.out_count + 127) / 128), grid.y);
    launch_k(stage_prog_kernel<TI, TA, SCATTER>, g2, 128, 0, stream, k);
    return;
  }
  if (k.n_terms <= 2) launch_k(stage_kernel<TI, TA, SCATTER, 2>, grid, 256, 0, stream, k);
  else if (k.n_terms <= 4) launch_k(stage_kernel<TI, TA, SCATTER, 4>, grid, 256, 0, stream, k);
  else launch_k(stage_kernel<TI, TA, SCATTER, MAXT>, grid, 256, 0, stream, k);
}

template <typename TI>
static void launch_stage_impl(const DevStage& ds, const Bindings& b, void* out, bool out_acc, cudaStream_t stream,
                              const char** kind);

template <typename TI>
static void launch_stage_t(const DevStage& ds, const Bindings& b, void* out, bool out_acc, cudaStream_t stream) {
  const char* kind = "stage";
  const int id = prof_begin("stage", 2.0 * ds.cs.grid_points(), 0.0, stream);
  launch_stage_impl<TI>(ds, b, out, out_acc, stream, &kind);
  prof_rename(id, kind);
  prof_end(id, stream);
}

template <typename TI>
static void launch_stage_impl(const DevStage& ds, const Bindings& b_in, void* out, bool out_acc, cudaStream_t stream,
                              const char** kind) {
  using TA = typename Acc<TI>::type;
  if (ds.perm_out) {
    // scatter into the permuted target (accumulator precision), then restore
    void* tmp = nullptr;
    cuda_check(cudaMallocAsync(&tmp, (size_t)ds.perm_count * sizeof(TA), stream), "alloc permuted target");
    DevStage inner = ds;
    inner.perm_out.reset();
    launch_stage_impl<TI>(inner, b_in, tmp, true, stream, kind);
    Bindings b2 = b_in;
    b2.scratch = tmp;
    const char* pk = nullptr;
    launch_stage_impl<TI>(*ds.perm_out, b2, out, out_acc, stream, &pk);
    cuda_check(cudaFreeAsync(tmp, stream), "free permuted target");
    return;
  }
  Bindings b = b_in;
  void* perm_buf = nullptr;
  if (ds.perm_in) {
    cuda_check(cudaMallocAsync(&perm_buf, (size_t)ds.perm_count * sizeof(TI), stream), "alloc permuted input");
    const char* pk = nullptr;
    launch_stage_impl<TI>(*ds.perm_in, b_in, perm_buf, false, stream, &pk);
    b.perm = perm_buf;
  }
  struct PermFree {
    void* p;
    cudaStream_t s;
    ~PermFree() {
      if (p) cudaFreeAsync(p, s);
    }
  } perm_free{perm_buf, stream};
  void* gpre_buf = nullptr;
  if (ds.gpre) {
    cuda_check(cudaMallocAsync(&gpre_buf, (size_t)std::max<int64_t>(ds.gpre_count, 1) * sizeof(TA), stream),
               "alloc factored partial sums");
    const char* pk = nullptr;
    launch_stage_impl<TI>(*ds.gpre, b, gpre_buf, true, stream, &pk);
    b.pre = gpre_buf;
  }
  struct PreFree {
    void* p;
    cudaStream_t s;
    ~PreFree() {
      if (p) cudaFreeAsync(p, s);
    }
  } pre_free{gpre_buf, stream};
  KStage k = ds.k;
  for (int t = 0; t < k.n_terms; ++t) {
    k.terms[t].ptr = bind_ptr(ds.cs.terms[t].t, b);
    if (!k.terms[t].ptr && k.terms[t].kind != 2 && !(ds.pre && ds.cs.terms[t].t.kind == TK_SCRATCH))
      fail(SYNO_E_INVALID, "stage input tensor is not bound (kind " + std::to_string(ds.cs.terms[t].t.kind) +
                               ", stage " + ds.cs.describe() + ")");
  }
  const int64_t out_bytes = k.out_count * (int64_t)(out_acc ? sizeof(TA) : sizeof(TI));
  if (ds.dead || k.out_count == 0) {
    if (!ds.cs.scatter && out_bytes) zero_fill(out, out_bytes, stream);
    return;
  }
  bool affine = !ds.cs.scatter && k.R == 1 && !k.prog;
  for (int t = 0; t < k.n_terms && affine; ++t)
    affine = k.terms[t].kind != 2 && k.terms[t].n_atab == 0 && k.terms[t].n_mix == 0 && k.terms[t].rtab == nullptr;
  if (affine) {
    *kind = "stage_affine";
    k.out = out;
    k.out_acc = out_acc;
    const unsigned blocks = (unsigned)((k.out_count + 255) / 256);
    note_launch();
    if (k.n_terms <= 2) launch_k(affine_kernel<TI, TA, 2>, blocks, 256, 0, stream, k);
    else launch_k(affine_kernel<TI, TA, MAXT>, blocks, 256, 0, stream, k);
    cuda_check(cudaGetLastError(), "affine_kernel");
    return;
  }
  if (ds.tile && !ds.cs.scatter && !k.prog) {
    *kind = "stage_tile";
    const TileInfo& ti = *ds.tile;
    TileArgs a = ti.a;
    TA* acc = nullptr;
    cuda_check(cudaMallocAsync((void**)&acc, (size_t)ti.splits * a.NF * a.NI * sizeof(TA), stream), "alloc tile sums");
    a.acc = acc;
    k.r_chunk = (k.R + ti.splits - 1) / ti.splits;
    k.out = nullptr;
    const dim3 grid((unsigned)ti.ctas, (unsigned)ti.splits);
    const unsigned threads = (unsigned)(a.TI * a.TF * a.TR);
    note_launch();
    if (a.n_rt <= 2) launch_k(stage_tile_kernel<TI, TA, 2, false>, grid, threads, ti.smem, stream, k, a);
    else if (a.n_rt <= 4) launch_k(stage_tile_kernel<TI, TA, 4, false>, grid, threads, ti.smem, stream, k, a);
    else launch_k(stage_tile_kernel<TI, TA, MAXT, false>, grid, threads, ti.smem, stream, k, a);
    cuda_check(cudaGetLastError(), "stage_tile_kernel");
    Bindings b2 = b;
    b2.scratch = acc;
    const char* fk = nullptr;
    launch_stage_impl<TI>(*ti.finish, b2, out, out_acc, stream, &fk);
    cuda_check(cudaFreeAsync(acc, stream), "free tile sums");
    return;
  }
  const bool block_mode = !ds.cs.scatter && k.out_count <= 16384 && k.R >= 2048 && !k.prog;
  // Reduce split: enough threads to fill the chip about twice.
  const int64_t want = 148LL * 2048;
  int64_t nsplit = 1;
  if (block_mode) {
    nsplit = std::max<int64_t>(1, std::min<int64_t>({(4 * 148 + k.out_count - 1) / k.out_count, k.R / 2048, 1024}));
  } else if (k.out_count < want && k.R >= 64) {
    nsplit = std::min<int64_t>((want + k.out_count - 1) / k.out_count, k.R / 32);
    nsplit = std::max<int64_t>(1, std::min<int64_t>(nsplit, 4096));
  }
  k.r_chunk = (k.R + nsplit - 1) / nsplit;
  nsplit = (k.R + k.r_chunk - 1) / k.r_chunk;
  if (k.R == 0) { nsplit = 1; k.r_chunk = 0; }
  dim3 grid((unsigned)((k.out_count + 255) / 256), (unsigned)nsplit);
  if (block_mode) {
    *kind = "stage_block_reduce";
    dim3 bgrid((unsigned)k.out_count, (unsigned)nsplit);
    TA* part = nullptr;
    if (nsplit > 1)
      cuda_check(cudaMallocAsync((void**)&part, (size_t)nsplit * k.out_count * sizeof(TA), stream), "alloc partials");
    k.out = nsplit > 1 ? (void*)part : out;
    k.out_acc = nsplit > 1 ? 1 : out_acc;
    note_launch();
    launch_k(stage_block_kernel<TI, TA>, bgrid, 256, 0, stream, k);
    cuda_check(cudaGetLastError(), "stage_block_kernel");
    if (nsplit > 1) {
      unsigned blocks = (unsigned)((k.out_count + 255) / 256);
      note_launch();
      if (out_acc) launch_k(sum_partials<TA, TA>, blocks, 256, 0, stream, part, k.out_count, (int)nsplit, (TA*)out);
      else launch_k(sum_partials<TI, TA>, blocks, 256, 0, stream, part, k.out_count, (int)nsplit, (TI*)out);
      cuda_check(cudaGetLastError(), "sum_partials");
      cuda_check(cudaFreeAsync(part, stream), "free partials");
    }
    return;
  }
  if (ds.cs.scatter) {
    *kind = "stage_scatter";
    void* g = nullptr;
    if (ds.pre) {
      cuda_check(cudaMallocAsync(&g, (size_t)ds.pre->k.out_count * sizeof(TA), stream), "alloc pre-reduction");
      const char* pk = nullptr;
      launch_stage_impl<TI>(*ds.pre, b, g, true, stream, &pk);
      for (int t = 0; t < k.n_terms; ++t)
        if (ds.cs.terms[t].t.kind == TK_SCRATCH) k.terms[t].ptr = g;
    }
    // deterministic fixed-point accumulation (fx_add): zero the integer
    // sums and the bound slots, bound every loaded term, scatter, convert
    const bool wide = sizeof(TA) == 8;
    const int64_t n_out = ds.cs.out.numel();
    MaxAbsArgs ma;
    memset(&ma, 0, sizeof(ma));
    int nl = 0;
    int64_t most = 0;
    for (int t = 0; t < k.n_terms; ++t) {
      if (k.terms[t].kind == 2) continue;
      ma.ptr[nl] = k.terms[t].ptr;
      ma.count[nl] = ds.cs.terms[t].t.numel();
      ma.acc[nl] = k.terms[t].kind == 1;
      most = std::max(most, ma.count[nl]);
      ++nl;
    }
    const size_t fx_bytes = (size_t)n_out * (wide ? 16 : 8);
    uint8_t* buf = nullptr;
    cuda_check(cudaMallocAsync((void**)&buf, fx_bytes + 8 * (MAXT + 1), stream), "alloc scatter sums");
    zero_fill(buf, fx_bytes + 8 * (MAXT + 1), stream);
    ma.out = (double*)(buf + fx_bytes);
    if (nl) {
      note_launch();
      const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((most + 255) / 256, 148 * 4));
      launch_k(maxabs_kernel<TI, TA>, dim3(blocks, nl), 256, 0, stream, ma);
      cuda_check(cudaGetLastError(), "maxabs_kernel");
    }
    k.out = out;
    k.out_acc = 1;
    k.fx = (unsigned long long*)buf;
    k.fx_max = ma.out;
    k.fx_n = nl;
    k.fx_mult = (double)k.out_count * (double)k.R * std::fabs(k.scale);
    note_launch();
    if (ds.tile) {
      *kind = "stage_tile_scatter";
      const TileInfo& ti = *ds.tile;
      k.r_chunk = (k.R + ti.splits - 1) / ti.splits;
      const dim3 tgrid((unsigned)ti.ctas, (unsigned)ti.splits);
      const unsigned threads = (unsigned)(ti.a.TI * ti.a.TF * ti.a.TR);
      if (ti.a.n_rt <= 3) launch_k(stage_tile_kernel<TI, TA, 2, true>, tgrid, threads, ti.smem, stream, k, ti.a);
      else if (ti.a.n_rt <= 5) launch_k(stage_tile_kernel<TI, TA, 4, true>, tgrid, threads, ti.smem, stream, k, ti.a);
      else launch_k(stage_tile_kernel<TI, TA, MAXT, true>, tgrid, threads, ti.smem, stream, k, ti.a);
      cuda_check(cudaGetLastError(), "stage_tile_kernel<scatter>");
    } else {
      launch_nt<TI, TA, true>(k, grid, stream);
      cuda_check(cudaGetLastError(), "stage_kernel<scatter>");
    }
    const unsigned cb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n_out + 255) / 256, 148 * 8));
    note_launch();
    if (out_acc) launch_k(fx_convert_kernel<TA, TA>, cb, 256, 0, stream, k, n_out, (TA*)out);
    else launch_k(fx_convert_kernel<TI, TA>, cb, 256, 0, stream, k, n_out, (TI*)out);
    cuda_check(cudaGetLastError(), "fx_convert_kernel");
    cuda_check(cudaFreeAsync(buf, stream), "free scatter sums");
    if (g) cuda_check(cudaFreeAsync(g, stream), "free pre-reduction");
    return;
  }
  *kind = "stage_gather_reduce";
  if (nsplit == 1) {
    k.out = out;
    k.out_acc = out_acc;
    note_launch();
    launch_nt<TI, TA, false>(k, grid, stream);
    cuda_check(cudaGetLastError(), "stage_kernel");
    return;
  }
  TA* part = nullptr;
  cuda_check(cudaMallocAsync((void**)&part, (size_t)nsplit * k.out_count * sizeof(TA), stream), "alloc partials");
  k.out = part;
  k.out_acc = 1;
  note_launch();
  launch_nt<TI, TA, false>(k, grid, stream);
  cuda_check(cudaGetLastError(), "stage_kernel<split>");
  unsigned blocks = (unsigned)((k.out_count + 255) / 256);
  note_launch();
  if (out_acc) launch_k(sum_partials<TA, TA>, blocks, 256, 0, stream, part, k.out_count, (int)nsplit, (TA*)out);
  else launch_k(sum_partials<TI, TA>, blocks, 256, 0, stream, part, k.out_count, (int)nsplit, (TI*)out);
  cuda_check(cudaGetLastError(), "sum_partials");
  cuda_check(cudaFreeAsync(part, stream), "free partials");
}

void run_stage(DType dt, const DevStage& ds, const Bindings& b, void* out, bool out_acc, cudaStream_t stream) {
  switch (dt) {
    case DT_F32: launch_stage_t<float>(ds, b, out, out_acc, stream); break;
    case DT_BF16: launch_stage_t<__nv_bfloat16>(ds, b, out, out_acc, stream); break;
    case DT_F64: launch_stage_t<double>(ds, b, out, out_acc, stream); break;
    default: fail(SYNO_E_INVALID, "unknown dtype");
  }
}

static void launch_cast(DType dt, const void* acc, int64_t count, void* out, cudaStream_t stream) {
  unsigned blocks = (unsigned)((count + 255) / 256);
  if (!count || dt != DT_BF16) return;
  note_launch();
  launch_k(cast_kernel<__nv_bfloat16, float>, blocks, 256, 0, stream, (const float*)acc, count, (__nv_bfloat16*)out);
  cuda_check(cudaGetLastError(), "cast_kernel");
}

// ---------------------------------------------------------------------------
// Gathered GEMM: a contraction whose operands are arbitrary gathers
// ---------------------------------------------------------------------------
// The reference's `contract` snapshots any target expressions as the weight
// access (pgraph.py:335-352), so a sampled operator is often
//     y[b, n.., m..] = scale * sum_r x[gx(b, m.., r)] * w[gw(n.., r)]
// with windowed / merged / strided index maps that the conv matcher (tc.cu)
// does not take.  Here the two operands are gathered into dense matrices
//     X~[b][r][m] = x[gx(b, m, r)]   (0 out of range)     W~[n][r] = w[gw(n, r)]
// by universal-engine stages (HBM-bound), and the contraction runs on the
// tcgen05 path as a pointwise operator with C_in = |r|, C_out = |n|,
// pixels = |m| -- the same kernels and the same fp32 split-bf16 scheme as the
// config layers.  Backward: the pointwise grad-input / grad-weight give dX~
// and dW~, which scatter back through the same index maps (deterministic
// fixed-point scatter stages).  When w's access is the identity
// (w[n.., r..] in order) W~ is w itself and dW~ is dw.
struct GatherGemm {
  Plan pw;                       // the synthetic pointwise operator
  std::unique_ptr<DevPlan> pdev; // its device plan (tcgen05)
  DevStage gx, gxs;              // X~ = gather(x); dx = scatter(dX~)
  bool w_ident = true;
  bool mr = false;               // QKV-like: X~ = [batch][m][r], y N-contiguous
  DevStage gw, gws;              // W~ = gather(w); dw = scatter(dW~)
  int64_t nx = 0, nw = 0, nxin = 0, nwin = 0;
  ~GatherGemm() {
    release_dev_stage(gx);
    release_dev_stage(gxs);
    release_dev_stage(gw);
    release_dev_stage(gws);
  }
};

static int64_t numel_of(const std::vector<int64_t>& e);
static size_t dtype_size(DType dt);

struct GGShape {
  int tx = -1, tw = -1;
  std::vector<int> Nax, Max;
  int64_t NN = 1, MM = 1, RR = 1;
  bool nfirst = true;
};

// Host-only structural match of the gathered-GEMM form (see GatherGemm).
static bool gg_shape(const Plan& plan, GGShape* out) {
  static const bool off = getenv("SYNO_NO_GATHER_GEMM") != nullptr;  // A/B switch
  const CStage& S = plan.unstaged;
  if (off || S.terms.size() != 2 || plan.w_ext.size() != 1 || S.scale != 1.0 || S.dead) return false;
  GGShape g;
  for (int t = 0; t < 2; ++t) {
    if (S.terms[t].t.kind == TK_X) g.tx = t;
    if (S.terms[t].t.kind == TK_W) g.tw = t;
  }
  if (g.tx < 0 || g.tw < 0) return false;
  const int A = (int)S.axis_ext.size(), L = S.nloops();
  const int B = (int)plan.batch_ext.size();
  if (B != 1) return false;
  auto uses = [&](const CTerm& t, std::vector<bool>* u) {
    u->assign(L, false);
    for (auto& c : t.coords) {
      std::vector<int> d;
      c_loops(c, &d);
      for (int l : d) (*u)[l] = true;
    }
  };
  std::vector<bool> ux, uw;
  uses(S.terms[g.tx], &ux);
  uses(S.terms[g.tw], &uw);
  // x's leading coordinate is the bare batch loop; w never reads the batch
  if (S.terms[g.tx].coords.empty() || S.terms[g.tx].coords[0]->op != COp::Loop ||
      S.terms[g.tx].coords[0]->loop != 0 || uw[0])
    return false;
  for (int a = B; a < A; ++a) {
    if (ux[a] && uw[a]) return false;
    if (uw[a]) g.Nax.push_back(a);
    else if (ux[a]) g.Max.push_back(a);
    else return false;  // broadcast axis: not a GEMM output
  }
  if (g.Nax.empty() || g.Max.empty()) return false;
  // y = [batch][N block][M block] (a pointwise operator, NCHW-like) or
  // y = [batch][M block][N block] (a QKV-like projection, N contiguous)
  bool nlast = true;
  for (size_t q = 0; q < g.Nax.size(); ++q) {
    g.nfirst = g.nfirst && g.Nax[q] == B + (int)q;
    nlast = nlast && g.Nax[q] == A - (int)g.Nax.size() + (int)q;
  }
  if (!g.nfirst && !nlast) return false;
  for (int a : g.Nax) g.NN *= S.axis_ext[a];
  for (int a : g.Max) g.MM *= S.axis_ext[a];
  for (auto r : S.red_ext) g.RR *= r;
  // worth a GEMM, and the gathered operand fits comfortably
  if (g.RR < 64 || g.NN < 16 || g.MM < 64 || (double)plan.batch * g.RR * g.MM > 6.0e8) return false;
  *out = g;
  return true;
}

bool gg_matches(const Plan& plan) {
  GGShape g;
  return gg_shape(plan, &g);
}

static std::shared_ptr<GatherGemm> gg_build(const Plan& plan, cudaStream_t stream) {
  GGShape sh;
  if (!gg_shape(plan, &sh)) return nullptr;
  const CStage& S = plan.unstaged;
  const int A = (int)S.axis_ext.size(), L = S.nloops();
  const int tx = sh.tx, tw = sh.tw;
  const std::vector<int>& Nax = sh.Nax;
  const std::vector<int>& Max = sh.Max;
  const int64_t NN = sh.NN, MM = sh.MM, RR = sh.RR;
  const bool nfirst = sh.nfirst;
  const int64_t batch = plan.batch;
  const int nR = (int)S.red_ext.size();
  auto gg = std::make_shared<GatherGemm>();
  // the synthetic operator: pointwise (C_in = RR, C_out = NN, H x W = MM)
  // or QKV-like (T = MM, E = RR, E3 = NN); W~ = [n][r] in both
  const int64_t Wd = S.axis_ext[Max.back()], Hd = MM / Wd;
  const bool mr = !nfirst;  // X~ = [batch][m][r] (QKV-like) instead of [batch][r][m]
  gg->mr = mr;
  std::string doc = mr ? "operator gathered_gemm\nvar T primary " + std::to_string(MM) + "\nvar E primary " +
                             std::to_string(RR) + "\nvar E3 primary " + std::to_string(NN) + "\nvar B primary " +
                             std::to_string(batch) +
                             "\noutput T E3\ninput T E\nbatch B\nsteps op{reduce(E); contract[1:weight,2:both]}\n"
                       : "operator gathered_gemm\nvar C_out primary " + std::to_string(NN) + "\nvar C_in primary " +
                             std::to_string(RR) + "\nvar H primary " + std::to_string(Hd) + "\nvar W primary " +
                             std::to_string(Wd) + "\nvar N primary " + std::to_string(batch) +
                             "\noutput C_out H W\ninput C_in H W\nbatch N\nsteps op{reduce(C_in); contract[0:weight,3:both]}\n";
  try {
    Graph g = parse_operator(doc);
    Assignment env = g.spec->assignment();
    LoopNest un = build_loop_nest(g, env);
    gg->pw = build_plan(un, un, g.spec->batch_dims, env);
  } catch (const Error&) {
    return nullptr;
  }
  gg->pdev.reset(build_dev_plan(gg->pw, stream));
  if (!gg->pdev->tc) return nullptr;
  auto remap = [](const CTerm& t, const std::vector<int>& m) {
    CTerm r = t;
    for (auto& c : r.coords) c = remap_loops(c, m);
    return r;
  };
  // X~ = [batch][r..][m..] (or [batch][m..][r..]): a gather stage, no reduce
  {
    const int nM = (int)Max.size();
    std::vector<int> m(L, -1);
    m[0] = 0;
    for (int j = 0; j < nR; ++j) m[A + j] = mr ? 1 + nM + j : 1 + j;
    for (int q = 0; q < nM; ++q) m[Max[q]] = mr ? 1 + q : 1 + nR + q;
    CStage g;
    g.axis_ext.push_back(batch);
    if (!mr)
      for (auto r : S.red_ext) g.axis_ext.push_back(r);
    for (int a : Max) g.axis_ext.push_back(S.axis_ext[a]);
    if (mr)
      for (auto r : S.red_ext) g.axis_ext.push_back(r);
    g.terms.push_back(remap(S.terms[tx], m));
    g.out.kind = TK_SCRATCH;
    g.out.extents = g.axis_ext;
    simplify_stage(&g);
    build_dev_stage(g, &gg->gx, stream);
    gg->nx = g.out.numel();
    // dx[gx(b, m, r)] += dX~[b][r][m]: scatter over (batch, M) x reduces
    std::vector<int> ms(L, -1);
    ms[0] = 0;
    for (size_t q = 0; q < Max.size(); ++q) ms[Max[q]] = 1 + (int)q;
    for (int j = 0; j < nR; ++j) ms[A + j] = 1 + (int)Max.size() + j;
    CStage sc;
    sc.axis_ext.push_back(batch);
    for (int a : Max) sc.axis_ext.push_back(S.axis_ext[a]);
    sc.red_ext = S.red_ext;
    CTerm d;
    d.t.kind = TK_SCRATCH_IN;  // dX~ comes from the tensor-core path in the operator's dtype
    d.t.extents = g.axis_ext;
    d.coords.push_back(c_loop(0));
    if (!mr)
      for (int j = 0; j < nR; ++j) d.coords.push_back(c_loop(1 + nM + j));
    for (int q = 0; q < nM; ++q) d.coords.push_back(c_loop(1 + q));
    if (mr)
      for (int j = 0; j < nR; ++j) d.coords.push_back(c_loop(1 + nM + j));
    sc.terms.push_back(d);
    sc.scatter = true;
    sc.target = remap(S.terms[tx], ms);
    sc.target.t.kind = TK_DX;
    sc.out = sc.target.t;
    simplify_stage(&sc);
    build_dev_stage(sc, &gg->gxs, stream);
    gg->nxin = numel_of(plan.x_ext);
  }
  // W~ = [n..][r..]
  {
    const CTerm& wt = S.terms[tw];
    bool ident = wt.coords.size() == Nax.size() + (size_t)nR;
    for (size_t q = 0; ident && q < wt.coords.size(); ++q) {
      const int want = q < Nax.size() ? Nax[q] : A + (int)(q - Nax.size());
      ident = wt.coords[q]->op == COp::Loop && wt.coords[q]->loop == want &&
              wt.t.extents[q] == S.ext(want);
    }
    gg->w_ident = ident;
    gg->nw = NN * RR;
    gg->nwin = numel_of(plan.w_ext[0]);
    if (!ident) {
      std::vector<int> m(L, -1);
      for (size_t q = 0; q < Nax.size(); ++q) m[Nax[q]] = (int)q;
      for (int j = 0; j < nR; ++j) m[A + j] = (int)Nax.size() + j;
      CStage g;
      for (int a : Nax) g.axis_ext.push_back(S.axis_ext[a]);
      for (auto r : S.red_ext) g.axis_ext.push_back(r);
      g.terms.push_back(remap(wt, m));
      g.out.kind = TK_SCRATCH;
      g.out.extents = g.axis_ext;
      simplify_stage(&g);
      build_dev_stage(g, &gg->gw, stream);
      std::vector<int> ms(L, -1);
      for (size_t q = 0; q < Nax.size(); ++q) ms[Nax[q]] = (int)q;
      for (int j = 0; j < nR; ++j) ms[A + j] = (int)Nax.size() + j;
      CStage sc;
      for (int a : Nax) sc.axis_ext.push_back(S.axis_ext[a]);
      for (auto r : S.red_ext) sc.red_ext.push_back(r);
      CTerm d;
      d.t.kind = TK_SCRATCH_IN;
      d.t.extents = g.axis_ext;
      for (size_t q = 0; q < g.axis_ext.size(); ++q) d.coords.push_back(c_loop((int)q));
      // as a scatter over (N) x reduces: dW~[n][r] -> dw[gw(n, r)]
      sc.terms.push_back(d);
      sc.scatter = true;
      sc.target = remap(wt, ms);
      sc.target.t.kind = TK_DW;
      sc.target.t.index = 0;
      sc.out = sc.target.t;
      simplify_stage(&sc);
      build_dev_stage(sc, &gg->gws, stream);
    }
  }
  return gg;
}

static void run_grad(DType dt, const DevStage& ds, const Bindings& b, void* out, int64_t count, cudaStream_t stream);
static int64_t numel_of(const std::vector<int64_t>& e);

static bool gg_forward(GatherGemm& gg, DType dt, const Bindings& b, cudaStream_t stream) {
  if (dt != DT_F32 && dt != DT_BF16) return false;
  const size_t es = dtype_size(dt);
  void *xt = nullptr, *wt = nullptr;
  cuda_check(cudaMallocAsync(&xt, gg.nx * es, stream), "alloc gathered x");
  run_stage(dt, gg.gx, b, xt, false, stream);
  if (!gg.w_ident) {
    cuda_check(cudaMallocAsync(&wt, gg.nw * es, stream), "alloc gathered w");
    run_stage(dt, gg.gw, b, wt, false, stream);
  }
  Bindings pb;
  pb.x = xt;
  pb.w = {gg.w_ident ? b.w.at(0) : wt};
  pb.y = b.y;
  const bool ok = tc_forward(*gg.pdev->tc, dt, pb, stream);
  cuda_check(cudaFreeAsync(xt, stream), "free gathered x");
  if (wt) cuda_check(cudaFreeAsync(wt, stream), "free gathered w");
  if (!ok) fail(SYNO_E_INVALID, "gathered GEMM: tensor-core forward refused its own plan");
  return true;
}

static bool gg_backward(GatherGemm& gg, DType dt, const Bindings& b, cudaStream_t stream) {
  if (dt != DT_F32 && dt != DT_BF16) return false;
  const size_t es = dtype_size(dt);
  const bool want_w = !b.dw.empty() && b.dw[0];
  void *xt = nullptr, *wt = nullptr, *dxt = nullptr, *dwt = nullptr;
  cuda_check(cudaMallocAsync(&xt, gg.nx * es, stream), "alloc gathered x");
  run_stage(dt, gg.gx, b, xt, false, stream);
  if (!gg.w_ident) {
    cuda_check(cudaMallocAsync(&wt, gg.nw * es, stream), "alloc gathered w");
    run_stage(dt, gg.gw, b, wt, false, stream);
  }
  if (b.dx) cuda_check(cudaMallocAsync(&dxt, gg.nx * es, stream), "alloc gathered dx");
  if (want_w && !gg.w_ident) cuda_check(cudaMallocAsync(&dwt, gg.nw * es, stream), "alloc gathered dw");
  Bindings pb;
  pb.x = xt;
  pb.w = {gg.w_ident ? b.w.at(0) : wt};
  pb.dy = b.dy;
  pb.dx = dxt;
  pb.dw = {want_w ? (gg.w_ident ? b.dw[0] : dwt) : nullptr};
  const bool ok = tc_backward(*gg.pdev->tc, dt, pb, stream);
  if (!ok) fail(SYNO_E_INVALID, "gathered GEMM: tensor-core backward refused its own plan");
  if (b.dx) {
    Bindings sb = b;
    sb.scratch = dxt;
    run_grad(dt, gg.gxs, sb, b.dx, gg.nxin, stream);
  }
  if (dwt) {
    Bindings sb = b;
    sb.scratch = dwt;
    run_grad(dt, gg.gws, sb, b.dw[0], gg.nwin, stream);
  }
  for (void* p : {xt, wt, dxt, dwt})
    if (p) cuda_check(cudaFreeAsync(p, stream), "free gathered operand");
  return true;
}

void run_forward(const Plan& plan, DevPlan& dp, DType dt, const Bindings& b_in, cudaStream_t stream) {
  wait_built(dp.ev_plan, stream);
  // Tensor-core path first: it computes the unstaged contraction, which the
  // staged nest equals by construction (codegen.py:605-608).
  if (dp.tc && tc_forward(*dp.tc, dt, b_in, stream)) return;
  if (dp.gg && gg_forward(*dp.gg, dt, b_in, stream)) return;
  ensure_forward(plan, dp, stream);
  Bindings b = b_in;
  b.stages.assign(plan.stage_ext.size(), nullptr);
  std::vector<void*> owned;
  for (size_t k = 0; k < plan.stage_ext.size(); ++k) {
    int64_t n = 1;
    for (auto e : plan.stage_ext[k]) n *= e;
    void* p = nullptr;
    cuda_check(cudaMallocAsync(&p, std::max<int64_t>(n, 1) * acc_size(dt), stream), "alloc stage buffer");
    b.stages[k] = p;
    owned.push_back(p);
  }
  for (auto& ds : dp.forward) {
    bool to_stage = ds.cs.out.kind == TK_STAGE;
    void* out = to_stage ? b.stages[ds.cs.out.index] : b.y;
    run_stage(dt, ds, b, out, to_stage, stream);
  }
  for (void* p : owned) cuda_check(cudaFreeAsync(p, stream), "free stage buffer");
}

static void run_grad(DType dt, const DevStage& ds, const Bindings& b, void* out, int64_t count, cudaStream_t stream) {
  if (!out) return;
  if (!ds.cs.scatter) {
    run_stage(dt, ds, b, out, false, stream);
    return;
  }
  const size_t asz = acc_size(dt);
  if (dt != DT_BF16) {
    zero_fill(out, count * asz, stream);
    if (!ds.dead) run_stage(dt, ds, b, out, true, stream);
    return;
  }
  void* acc = nullptr;
  cuda_check(cudaMallocAsync(&acc, std::max<int64_t>(count, 1) * asz, stream), "alloc grad acc");
  zero_fill(acc, count * asz, stream);
  if (!ds.dead) run_stage(dt, ds, b, acc, true, stream);
  launch_cast(dt, acc, count, out, stream);
  cuda_check(cudaFreeAsync(acc, stream), "free grad acc");
}

static int64_t numel_of(const std::vector<int64_t>& e) {
  int64_t n = 1;
  for (auto v : e) n *= v;
  return n;
}

// Reverse-mode through the rfactored stages (Plan::bwd_staged): recompute
// the forward intermediates, then run each gradient stage into dx, dw_j or
// the gradient buffer of an intermediate.
static void run_backward_staged(const Plan& plan, DevPlan& dp, DType dt, const Bindings& b_in, cudaStream_t stream) {
  ensure_forward(plan, dp, stream);
  ensure_backward(plan, dp, stream);
  Bindings b = b_in;
  const size_t nst = plan.stage_ext.size();
  std::vector<void*> owned;
  auto acc_alloc = [&](int64_t n) {
    void* p = nullptr;
    cuda_check(cudaMallocAsync(&p, std::max<int64_t>(n, 1) * acc_size(dt), stream), "alloc stage buffer");
    owned.push_back(p);
    return p;
  };
  b.stages.assign(nst, nullptr);
  b.dstages.assign(nst, nullptr);
  for (size_t k = 0; k < nst; ++k) {
    b.stages[k] = acc_alloc(numel_of(plan.stage_ext[k]));
    b.dstages[k] = acc_alloc(numel_of(plan.stage_ext[k]));
  }
  for (auto& ds : dp.forward) {
    if (ds.cs.out.kind != TK_STAGE) continue;  // the output y is not needed
    run_stage(dt, ds, b, b.stages[ds.cs.out.index], true, stream);
  }
  for (auto& ds : dp.bwd_staged) {
    const CTensor& o = ds.cs.out;
    if (o.kind == TK_DX) {
      run_grad(dt, ds, b, b.dx, numel_of(plan.x_ext), stream);
    } else if (o.kind == TK_DW) {
      run_grad(dt, ds, b, o.index < (int)b.dw.size() ? b.dw[o.index] : nullptr, numel_of(plan.w_ext.at(o.index)),
               stream);
    } else {
      void* out = b.dstages.at(o.index);
      if (ds.cs.scatter) {
        zero_fill(out, numel_of(o.extents) * acc_size(dt), stream);
        if (!ds.dead) run_stage(dt, ds, b, out, true, stream);
      } else {
        run_stage(dt, ds, b, out, true, stream);
      }
    }
  }
  for (void* p : owned) cuda_check(cudaFreeAsync(p, stream), "free stage buffer");
}

void run_backward(const Plan& plan, DevPlan& dp, DType dt, const Bindings& b, cudaStream_t stream) {
  wait_built(dp.ev_plan, stream);
  if (dp.tc && tc_backward(*dp.tc, dt, b, stream)) return;
  if (dp.gg && gg_backward(*dp.gg, dt, b, stream)) return;
  if (!plan.bwd_staged.empty()) {
    run_backward_staged(plan, dp, dt, b, stream);
    return;
  }
  ensure_backward(plan, dp, stream);
  int64_t nx = 1;
  for (auto e : plan.x_ext) nx *= e;
  run_grad(dt, dp.grad_x.at(0), b, b.dx, nx, stream);
  for (size_t j = 0; j < plan.w_ext.size(); ++j) {
    int64_t nw = 1;
    for (auto e : plan.w_ext[j]) nw *= e;
    run_grad(dt, dp.grad_w.at(j).at(0), b, j < b.dw.size() ? b.dw[j] : nullptr, nw, stream);
  }
}

}  // namespace syno
