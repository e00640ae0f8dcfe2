// extern "C" boundary (include/syno.h).
#include "../../include/syno.h"

#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>

#include "engine.hpp"
#include "tc.hpp"

using namespace syno;

struct syno_op {
  Graph graph;
  Assignment env;
  bool staged = false;
  bool replay_only = false;
  bool nest_handle = false;  // syno_compile_nest: built from loop-nest text, not from steps
  LoopNest unstaged, staged_nest;
  Plan plan;
  std::mutex mu;
  std::map<int, std::unique_ptr<DevPlan>> dev;
};

static thread_local std::string g_last_error;

template <typename F>
static int guarded(F&& f) {
  try {
    f();
    return SYNO_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SYNO_E_INVALID;
  }
}

static Assignment parse_assignment(const char* kv) {
  Assignment a;
  std::string s(kv);
  for (char& c : s)
    if (c == ',' || c == ';') c = ' ';
  std::istringstream in(s);
  std::string item;
  while (in >> item) {
    size_t eq = item.find('=');
    if (eq == std::string::npos || eq == 0) fail(SYNO_E_INVALID, "bad assignment item '" + item + "'");
    try {
      a[item.substr(0, eq)] = std::stoll(item.substr(eq + 1));
    } catch (const std::exception&) {
      fail(SYNO_E_INVALID, "bad assignment value in '" + item + "'");
    }
  }
  return a;
}

static int put_text(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap) {
    size_t n = std::min(cap - 1, s.size());
    memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return SYNO_OK;
}

static DevPlan& dev_plan(syno_op* op, cudaStream_t stream) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(op->mu);
  auto it = op->dev.find(dev);
  if (it != op->dev.end()) return *it->second;
  DevPlan* p = build_dev_plan(op->plan, stream);
  op->dev[dev].reset(p);
  return *p;
}

extern "C" {

int syno_compile(const char* doc, const char* assignment_kv, int flags, syno_op_t* out) {
  return guarded([&] {
    if (!doc || !out) fail(SYNO_E_INVALID, "null argument");
    auto op = std::make_unique<syno_op>();
    op->graph = parse_operator(doc);
    op->env = assignment_kv ? parse_assignment(assignment_kv) : op->graph.spec->assignment();
    op->staged = flags & SYNO_STAGED;
    op->replay_only = flags & SYNO_REPLAY_ONLY;
    if (op->replay_only) {
      *out = op.release();
      return;
    }
    op->unstaged = build_loop_nest(op->graph, op->env);
    LoopNest st = rfactor(op->unstaged);
    op->staged_nest = st;
    op->plan = build_plan(op->unstaged, op->staged ? st : op->unstaged, op->graph.spec->batch_dims, op->env);
    op->plan.flops_staged = nest_flops(st) * op->plan.batch;
    *out = op.release();
  });
}

int syno_compile_nest(const char* spec_document, const char* nest_text, const char* assignment_kv, int flags,
                      syno_op_t* out) {
  return guarded([&] {
    if (!spec_document || !nest_text || !out) fail(SYNO_E_INVALID, "null argument");
    if (flags) fail(SYNO_E_INVALID, "syno_compile_nest takes no flags");
    std::string doc = spec_document;
    if (doc.find("\nsteps ") == std::string::npos && doc.compare(0, 6, "steps ") != 0) {
      if (!doc.empty() && doc.back() != '\n') doc += "\n";
      doc += "steps op{}\n";
    }
    auto op = std::make_unique<syno_op>();
    op->graph = parse_operator(doc);
    op->env = assignment_kv ? parse_assignment(assignment_kv) : op->graph.spec->assignment();
    LoopNest nest = parse_loop_nest(nest_text, *op->graph.spec, op->env);
    if (nest.stages.empty()) fail(SYNO_E_PARSE, "loop nest has no stages");
    // executable nests name declared tensors only (run_nest would fail later)
    auto declared = [&](const std::string& name) {
      for (auto& t : nest.tensors)
        if (t.name == name) return true;
      return false;
    };
    for (auto& st : nest.stages) {
      if (!declared(st.tensor)) fail(SYNO_E_PARSE, "stage writes undeclared tensor '" + st.tensor + "'");
      for (auto& t : st.terms)
        if (!declared(t.tensor)) fail(SYNO_E_PARSE, "term reads undeclared tensor '" + t.tensor + "'");
    }
    if (!declared("x") || !declared("y")) fail(SYNO_E_PARSE, "loop nest declares no input x / output y");
    op->nest_handle = true;
    op->unstaged = nest;
    op->staged_nest = nest;
    // run_nest (codegen.py:549-572) has no batch; a single-stage nest is an
    // unstaged operator and gets the full plan (backward, tensor cores)
    const bool single = nest.stages.size() == 1;
    op->plan = build_plan(nest, nest, {}, op->env, single);
    *out = op.release();
  });
}

static void check_weights(syno_op* op, const void* const* w, int n_w) {
  if (op->replay_only) fail(SYNO_E_INVALID, "handle was compiled with SYNO_REPLAY_ONLY");
  if (n_w != (int)op->plan.w_ext.size())
    fail(SYNO_E_SHAPE, op->graph.spec->name + ": expected " + std::to_string(op->plan.w_ext.size()) +
                           " weight tensors, got " + std::to_string(n_w));
  for (int j = 0; j < n_w; ++j)
    if (!w[j]) fail(SYNO_E_INVALID, "null weight pointer");
}

int syno_forward(syno_op_t op, int dtype, const void* x, const void* const* w, int n_w, void* y, void* stream) {
  return guarded([&] {
    if (!op || !x || !y || (n_w && !w)) fail(SYNO_E_INVALID, "null argument");
    if (dtype < 0 || dtype > 2) fail(SYNO_E_INVALID, "unknown dtype");
    check_weights(op, w, n_w);
    cudaStream_t s = (cudaStream_t)stream;
    DevPlan& dp = dev_plan(op, s);
    Bindings b;
    b.x = x;
    for (int j = 0; j < n_w; ++j) b.w.push_back(w[j]);
    b.y = y;
    run_forward(op->plan, dp, (DType)dtype, b, s);
  });
}

int syno_backward_ex(syno_op_t op, int dtype, const void* x, const void* const* w, int n_w, const void* dy,
                     void* dx, void* const* dw, int flags, void* stream) {
  return guarded([&] {
    if (!op || !x || !dy || (n_w && !w)) fail(SYNO_E_INVALID, "null argument");
    if (dtype < 0 || dtype > 2) fail(SYNO_E_INVALID, "unknown dtype");
    if (flags & ~(SYNO_BWD_X_UNCHANGED | SYNO_BWD_W_UNCHANGED)) fail(SYNO_E_INVALID, "unknown backward flag");
    check_weights(op, w, n_w);
    cudaStream_t s = (cudaStream_t)stream;
    DevPlan& dp = dev_plan(op, s);
    Bindings b;
    b.x = x;
    for (int j = 0; j < n_w; ++j) b.w.push_back(w[j]);
    b.dy = dy;
    b.dx = dx;
    for (int j = 0; j < n_w; ++j) b.dw.push_back(dw ? dw[j] : nullptr);
    if (op->plan.nest_only)
      fail(SYNO_E_UNSUPPORTED, "a parsed loop nest with several stages runs forward only (codegen.run_nest)");
    b.x_unchanged = (flags & SYNO_BWD_X_UNCHANGED) != 0;
    b.w_unchanged = (flags & SYNO_BWD_W_UNCHANGED) != 0;
    run_backward(op->plan, dp, (DType)dtype, b, s);
  });
}

int syno_backward(syno_op_t op, int dtype, const void* x, const void* const* w, int n_w, const void* dy, void* dx,
                  void* const* dw, void* stream) {
  return syno_backward_ex(op, dtype, x, w, n_w, dy, dx, dw, 0, stream);
}

int syno_query(syno_op_t op, syno_info* info) {
  return guarded([&] {
    if (!op || !info) fail(SYNO_E_INVALID, "null argument");
    memset(info, 0, sizeof(*info));
    std::vector<int> perm;
    info->complete = op->nest_handle ? 1 : match_input(op->graph, &perm);
    if (op->replay_only) {
      info->replay_only = 1;
      info->n_weights = (int)op->graph.weights.size();
      return;
    }
    const Plan& p = op->plan;
    if (p.x_ext.size() > SYNO_MAX_RANK || p.y_ext.size() > SYNO_MAX_RANK || p.w_ext.size() > SYNO_MAX_WEIGHTS)
      fail(SYNO_E_UNSUPPORTED, "operator rank exceeds the query struct");
    info->n_weights = (int)p.w_ext.size();
    info->batch_rank = (int)p.batch_ext.size();
    info->x_rank = (int)p.x_ext.size();
    info->y_rank = (int)p.y_ext.size();
    for (size_t k = 0; k < p.x_ext.size(); ++k) info->x_shape[k] = p.x_ext[k];
    for (size_t k = 0; k < p.y_ext.size(); ++k) info->y_shape[k] = p.y_ext[k];
    int64_t params = 0;
    for (size_t j = 0; j < p.w_ext.size(); ++j) {
      if (p.w_ext[j].size() > SYNO_MAX_RANK) fail(SYNO_E_UNSUPPORTED, "weight rank exceeds the query struct");
      info->w_rank[j] = (int)p.w_ext[j].size();
      int64_t n = 1;
      for (size_t k = 0; k < p.w_ext[j].size(); ++k) {
        info->w_shape[j][k] = p.w_ext[j][k];
        n *= p.w_ext[j][k];
      }
      params += n;
      info->grad_w_scatter[j] = p.nest_only ? 0 : p.grad_w.at(j).at(0).scatter;
    }
    info->params = params;
    info->flops_unstaged = p.flops_unstaged;
    info->flops_staged = p.flops_staged;
    info->n_forward_stages = (int)p.forward.size();
    info->grad_x_scatter = p.nest_only ? 0 : p.grad_x.at(0).scatter;
    double g = 1;
    for (auto e : p.unstaged.axis_ext) g *= (double)e;
    for (auto e : op->unstaged.stages[0].reduces) g *= (double)e.extent;
    info->index_grid = (int64_t)g;
    info->tc_path = p.nest_only || staged_cheaper(p) ? 0 : tc_matches(p) ? 1 : gg_matches(p) ? 2 : 0;
  });
}

int syno_emit_loop_nest(syno_op_t op, int staged, char* buf, size_t cap, size_t* len) {
  int rc = guarded([&] {
    if (!op) fail(SYNO_E_INVALID, "null argument");
  });
  if (rc) return rc;
  if (op->replay_only) { g_last_error = "handle was compiled with SYNO_REPLAY_ONLY"; return SYNO_E_INVALID; }
  return put_text(emit_loop_nest(staged ? op->staged_nest : op->unstaged), buf, cap, len);
}

int syno_print_operator(syno_op_t op, char* buf, size_t cap, size_t* len) {
  if (!op) { g_last_error = "null argument"; return SYNO_E_INVALID; }
  return put_text(print_operator(op->graph), buf, cap, len);
}

int syno_describe_plan(syno_op_t op, char* buf, size_t cap, size_t* len) {
  if (!op) { g_last_error = "null argument"; return SYNO_E_INVALID; }
  if (op->replay_only) { g_last_error = "handle was compiled with SYNO_REPLAY_ONLY"; return SYNO_E_INVALID; }
  std::string s;
  for (auto& st : op->plan.forward) s += "forward: " + st.describe() + "\n";
  for (auto& st : op->plan.grad_x) s += "grad_x: " + st.describe() + "\n";
  for (size_t j = 0; j < op->plan.grad_w.size(); ++j)
    for (auto& st : op->plan.grad_w[j]) s += "grad_w" + std::to_string(j) + ": " + st.describe() + "\n";
  for (auto& st : op->plan.bwd_staged) s += "staged_bwd: " + st.describe() + "\n";
  return put_text(s, buf, cap, len);
}

int syno_index_map(syno_op_t op, int term, int coord, int64_t* out_dev, void* stream) {
  return guarded([&] {
    if (!op || !out_dev) fail(SYNO_E_INVALID, "null argument");
    if (op->replay_only) fail(SYNO_E_INVALID, "handle was compiled with SYNO_REPLAY_ONLY");
    // The unstaged stage keeps every reduce (no folding) for this hook.
    LoopNest& n = op->unstaged;
    CStage s;
    for (auto e : op->plan.batch_ext) s.axis_ext.push_back(e);
    std::map<std::string, int> loop_of;
    for (auto& a : n.stages[0].axes) {
      loop_of[a.name] = (int)s.axis_ext.size();
      s.axis_ext.push_back(a.extent);
    }
    for (auto& r : n.stages[0].reduces) {
      loop_of[r.name] = (int)(s.axis_ext.size() + s.red_ext.size());
      s.red_ext.push_back(r.extent);
    }
    if (term < 0 || term >= (int)n.stages[0].terms.size()) fail(SYNO_E_INVALID, "term out of range");
    const Access& acc = n.stages[0].terms[term];
    if (coord < 0 || coord >= (int)acc.exprs.size()) fail(SYNO_E_INVALID, "coordinate out of range");
    // Convert the one expression; batch loops are not referenced by it.
    std::function<CE(const E&)> conv = [&](const E& e) -> CE {
      switch (e->op) {
        case Op::Iter: return c_loop(loop_of.at(e->name));
        case Op::Const: return c_const(e->value);
        case Op::SizeRef: return c_const(eval_size(e->size, n.env));
        default: break;
      }
      COp o = e->op == Op::Add ? COp::Add : e->op == Op::Sub ? COp::Sub : e->op == Op::Mul ? COp::Mul
              : e->op == Op::FloorDiv ? COp::FloorDiv : COp::Mod;
      return c_bin(o, conv(e->lhs), conv(e->rhs));
    };
    CTerm t;
    t.coords.push_back(conv(acc.exprs[coord]));
    s.terms.push_back(t);
    eval_coordinate_grid(s, 0, 0, out_dev, (cudaStream_t)stream);
  });
}

int syno_graph_distance(syno_op_t op, double* out) {
  return guarded([&] {
    if (!op || !out) fail(SYNO_E_INVALID, "null argument");
    *out = graph_distance(op->graph);
  });
}

int syno_capi_set_error(const char* msg) {
  g_last_error = msg ? msg : "";
  return 0;
}

void syno_destroy(syno_op_t op) { delete op; }

const char* syno_last_error(void) { return g_last_error.c_str(); }

const char* syno_version(void) { return "syno-b200 0.1 (sm_100a)"; }

uint64_t syno_launch_count(void) { return launch_count(); }

void syno_profile_begin(void) { prof_enable(true); }

int syno_profile_end(syno_kernel_stat* out, int cap, int* n) {
  return guarded([&] {
    auto stats = prof_collect();
    prof_enable(false);
    if (n) *n = (int)stats.size();
    for (int i = 0; i < (int)stats.size() && i < cap && out; ++i) {
      memset(&out[i], 0, sizeof(out[i]));
      strncpy(out[i].name, stats[i].name.c_str(), sizeof(out[i].name) - 1);
      out[i].launches = stats[i].launches;
      out[i].ms = stats[i].ms;
      out[i].flops = stats[i].flops;
      out[i].bytes = stats[i].bytes;
    }
  });
}

}  // extern "C"

extern "C" {

int syno_tensor_write(const char* path, int rank, const int64_t* dims, const double* data) {
  return guarded([&] {
    if (!path || rank < 0 || (rank && !dims)) fail(SYNO_E_INVALID, "null argument");
    int64_t count = 1;
    for (int k = 0; k < rank; ++k) {
      if (dims[k] < 0) fail(SYNO_E_VALUE, "negative tensor dimension");
      count *= dims[k];
    }
    if (count && !data) fail(SYNO_E_INVALID, "null payload");
    std::unique_ptr<FILE, int (*)(FILE*)> f(fopen(path, "wb"), fclose);
    if (!f) fail(SYNO_E_INVALID, std::string("cannot open ") + path);
    // the format is little-endian; this library only builds for little-endian hosts
    const int64_t r = rank;
    bool ok = fwrite(&r, 8, 1, f.get()) == 1;
    if (rank) ok = ok && fwrite(dims, 8, (size_t)rank, f.get()) == (size_t)rank;
    if (count) ok = ok && fwrite(data, 8, (size_t)count, f.get()) == (size_t)count;
    if (!ok) fail(SYNO_E_INVALID, std::string("short write to ") + path);
  });
}

int syno_tensor_read(const char* path, int* rank, int64_t* dims, double* data, int64_t cap, int64_t* count) {
  return guarded([&] {
    if (!path || !rank || !count) fail(SYNO_E_INVALID, "null argument");
    std::unique_ptr<FILE, int (*)(FILE*)> f(fopen(path, "rb"), fclose);
    if (!f) fail(SYNO_E_INVALID, std::string("cannot open ") + path);
    fseek(f.get(), 0, SEEK_END);
    const long size = ftell(f.get());
    fseek(f.get(), 0, SEEK_SET);
    if (size < 8) fail(SYNO_E_SHAPE, "tensor file too short for a header");
    int64_t r = 0;
    if (fread(&r, 8, 1, f.get()) != 1) fail(SYNO_E_SHAPE, "tensor file too short for a header");
    if (r < 0 || size < 8 + 8 * r) fail(SYNO_E_SHAPE, "tensor file header truncated");
    if (r > SYNO_MAX_RANK) fail(SYNO_E_UNSUPPORTED, "tensor rank exceeds SYNO_MAX_RANK");
    int64_t d[SYNO_MAX_RANK];
    if (r && fread(d, 8, (size_t)r, f.get()) != (size_t)r) fail(SYNO_E_SHAPE, "tensor file header truncated");
    int64_t n = 1;
    for (int64_t k = 0; k < r; ++k) n *= d[k];
    const long payload = size - 8 - 8 * r;
    if (payload != 8 * n)
      fail(SYNO_E_SHAPE, "tensor payload holds " + std::to_string(payload / 8) + " values, header says " +
                             std::to_string(n));
    *rank = (int)r;
    *count = n;
    if (dims)
      for (int64_t k = 0; k < r; ++k) dims[k] = d[k];
    if (data) {
      if (cap < n) fail(SYNO_E_INVALID, "payload buffer too small");
      if (n && fread(data, 8, (size_t)n, f.get()) != (size_t)n) fail(SYNO_E_SHAPE, "tensor payload truncated");
    }
  });
}

}  // extern "C"
