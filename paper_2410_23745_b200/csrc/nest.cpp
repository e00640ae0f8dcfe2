// Loop-nest lowering, staging and emission (see nest.hpp).
#include "nest.hpp"

#include <algorithm>

namespace syno {

const TensorDecl& LoopNest::tensor(const std::string& n) const {
  for (auto& t : tensors)
    if (t.name == n) return t;
  fail(SYNO_E_KEY, "'" + n + "'");
}

static std::string sanitize(const std::string& text) {
  std::string out;
  for (char c : text)
    if (isalnum((unsigned char)c) || c == '_') out += c;
  return out.empty() ? "d" : out;
}

// codegen._display_names (codegen.py:251-294)
static std::map<std::string, std::string> display_names(const Graph& graph) {
  const Spec& spec = *graph.spec;
  std::map<std::string, std::string> names;
  std::map<std::string, int> taken;
  auto claim = [&](const std::string& base) {
    int n = ++taken[base];
    return n == 1 ? base : base + "_" + std::to_string(n);
  };
  for (size_t k = 0; k < spec.output_dims.size(); ++k)
    names["i" + std::to_string(k)] = claim("i_" + sanitize(spec.output_dims[k].str()));

  std::map<std::string, std::string> window_axis;
  Graph g = graph_root(graph.spec);
  for (auto& step : graph.steps) {
    if (step.kind == "unfold") {
      const Dim& data = g.dim_by_ident(step.targets[0]);
      const Dim& window = g.dim_by_ident(step.targets[1]);
      std::vector<E> frees, spatial;
      free_iterators(data.expr, &frees);
      for (auto& it : frees)
        if (!it->name.empty() && it->name[0] == 'i') spatial.push_back(it);
      if (window.expr->op == Op::Iter && spatial.size() == 1 && !window_axis.count(window.expr->name))
        window_axis[window.expr->name] = sanitize(spatial[0]->size.str());
    }
    g = graph_apply(g, step);
  }
  for (auto& it : graph.reduce_iters) {
    std::string base = "r_" + sanitize(it->size.str());
    auto w = window_axis.find(it->name);
    if (w != window_axis.end()) base += "_" + w->second;
    names[it->name] = claim(base);
  }
  return names;
}

static SizeLike sym(const Size& s) {
  SizeLike r;
  r.sym = s;
  return r;
}

LoopNest build_loop_nest(const Graph& graph, const Assignment& env) {
  const Spec& spec = *graph.spec;
  std::vector<int> perm;
  if (!match_input(graph, &perm)) fail(SYNO_E_SHAPE, spec.name + ": frontier does not match the input shape");
  auto names = display_names(graph);
  LoopNest nest;
  nest.name = spec.name;
  nest.env = env;
  Access x{"x", {}};
  for (int p : perm) x.exprs.push_back(rename_iters(graph.dims[p].expr, names));
  std::vector<Access> terms{x};
  TensorDecl xd{"x", "input", {}, {}};
  for (auto& s : spec.input_dims) {
    xd.sizes.push_back(sym(s));
    xd.extents.push_back(eval_size(s, env));
  }
  nest.tensors.push_back(xd);
  for (size_t j = 0; j < graph.weights.size(); ++j) {
    const Weight& w = graph.weights[j];
    Access a{"w" + std::to_string(j), {}};
    for (auto& e : w.exprs) a.exprs.push_back(rename_iters(e, names));
    terms.push_back(a);
    TensorDecl wd{"w" + std::to_string(j), "weight", {}, {}};
    for (auto& s : w.sizes) {
      wd.sizes.push_back(sym(s));
      wd.extents.push_back(eval_size(s, env));
    }
    nest.tensors.push_back(wd);
  }
  TensorDecl yd{"y", "output", {}, {}};
  for (auto& s : spec.output_dims) {
    yd.sizes.push_back(sym(s));
    yd.extents.push_back(eval_size(s, env));
  }
  nest.tensors.push_back(yd);
  Stage st;
  st.tensor = "y";
  for (size_t k = 0; k < spec.output_dims.size(); ++k)
    st.axes.push_back({names["i" + std::to_string(k)], sym(spec.output_dims[k]), eval_size(spec.output_dims[k], env)});
  for (auto& it : graph.reduce_iters) st.reduces.push_back({names[it->name], sym(it->size), eval_size(it->size, env)});
  st.terms = terms;
  nest.stages.push_back(st);
  return nest;
}

// Saturating at INT64_MAX: the reference computes with Python big ints, so a
// staging whose cost overflows must compare as (very) expensive, never wrap.
int64_t nest_flops(const LoopNest& nest) {
  const __int128 cap = (__int128)INT64_MAX;
  __int128 total = 0;
  for (auto& s : nest.stages) {
    __int128 n = 2;
    for (auto& a : s.axes) n = std::min(cap, n * (__int128)a.extent);
    for (auto& r : s.reduces) n = std::min(cap, n * (__int128)r.extent);
    total = std::min(cap, total + n);
  }
  return (int64_t)total;
}

static E shift_expr(const E& e, int64_t off) {
  if (off > 0) return mk_bin(Op::Add, e, mk_const(off));
  if (off < 0) return mk_bin(Op::Sub, e, mk_const(-off));
  return e;
}

struct Placeholder {
  E sub;
  E it;
  int64_t lo;
};

using Ranges = std::map<std::string, std::pair<int64_t, int64_t>>;

// codegen._carve (codegen.py:390-430); returns nullptr for "None".
static E carve(const E& e, const std::string& rname, std::vector<Placeholder>* ph, const Ranges& ranges,
               const Assignment& env, int* counter) {
  std::vector<E> frees;
  free_iterators(e, &frees);
  bool has_r = false;
  for (auto& f : frees) has_r = has_r || f->name == rname;
  if (!has_r) {
    if (frees.empty()) return e;
    for (auto& p : *ph)
      if (expr_eq(p.sub, e)) return shift_expr(p.it, p.lo);
    int64_t lo, hi;
    if (!expr_bounds(e, ranges, env, &lo, &hi)) return nullptr;
    E it = mk_iter("u" + std::to_string((*counter)++), Size{});
    ph->push_back({e, it, lo});
    return shift_expr(it, lo);
  }
  if (e->op == Op::Iter) return e;
  E a = carve(e->lhs, rname, ph, ranges, env, counter);
  E b = carve(e->rhs, rname, ph, ranges, env, counter);
  if (!a || !b) return nullptr;
  return mk_bin(e->op, a, b);
}

// codegen._factor_once (codegen.py:433-487)
static bool factor_once(const LoopNest& nest, const Axis& raxis, LoopNest* out) {
  const Stage& fin = nest.stages.back();
  const Assignment& env = nest.env;
  Ranges ranges;
  for (auto& a : fin.axes) ranges[a.name] = {0, a.extent - 1};
  for (auto& a : fin.reduces) ranges[a.name] = {0, a.extent - 1};
  std::vector<Access> with_r, without_r;
  for (auto& t : fin.terms) {
    bool touched = false;
    for (auto& e : t.exprs) touched = touched || mentions(e, raxis.name);
    (touched ? with_r : without_r).push_back(t);
  }
  if (with_r.empty()) return false;
  int maxu = -1;
  for (auto& s : nest.stages) {
    auto scan = [&](const std::vector<Axis>& v) {
      for (auto& a : v) {
        const std::string& n = a.name;
        if (n.size() >= 2 && n[0] == 'u' &&
            std::all_of(n.begin() + 1, n.end(), [](char c) { return c >= '0' && c <= '9'; }))
          maxu = std::max(maxu, std::stoi(n.substr(1)));
      }
    };
    scan(s.axes);
    scan(s.reduces);
  }
  int counter = maxu + 1;
  std::vector<Placeholder> ph;
  std::vector<Access> carved;
  for (auto& t : with_r) {
    Access a{t.tensor, {}};
    for (auto& e : t.exprs) {
      E ce = carve(e, raxis.name, &ph, ranges, env, &counter);
      if (!ce) return false;
      a.exprs.push_back(ce);
    }
    carved.push_back(a);
  }
  int stage_no = 0;
  for (auto& t : nest.tensors) stage_no += t.role == "stage";
  std::string name = "t" + std::to_string(stage_no);
  Stage mid;
  mid.tensor = name;
  std::vector<E> outer;
  TensorDecl decl{name, "stage", {}, {}};
  for (auto& p : ph) {
    int64_t lo, hi;
    expr_bounds(p.sub, ranges, env, &lo, &hi);
    int64_t ext = hi - p.lo + 1;
    SizeLike sl;
    sl.is_int = true;
    sl.ival = ext;
    mid.axes.push_back({p.it->name, sl, ext});
    outer.push_back(shift_expr(p.sub, -p.lo));
    decl.sizes.push_back(sl);
    decl.extents.push_back(ext);
  }
  mid.reduces.push_back(raxis);
  mid.terms = carved;
  Stage last;
  last.tensor = fin.tensor;
  last.axes = fin.axes;
  for (auto& r : fin.reduces)
    if (r.name != raxis.name) last.reduces.push_back(r);
  last.terms = without_r;
  last.terms.push_back({name, outer});
  *out = nest;
  out->tensors.insert(out->tensors.end() - 1, decl);
  out->stages.pop_back();
  out->stages.push_back(mid);
  out->stages.push_back(last);
  return true;
}

LoopNest rfactor(const LoopNest& in) {
  LoopNest nest = in;
  while (true) {
    bool have = false;
    LoopNest best;
    int64_t best_cost = nest_flops(nest);
    for (auto& r : nest.stages.back().reduces) {
      LoopNest cand;
      if (factor_once(nest, r, &cand)) {
        int64_t c = nest_flops(cand);
        if (c < best_cost) {
          best = cand;
          best_cost = c;
          have = true;
        }
      }
    }
    if (!have) return nest;
    nest = best;
  }
}

std::string emit_loop_nest(const LoopNest& nest) {
  std::string out = "nest " + nest.name + "\n";
  for (auto& t : nest.tensors) {
    std::string sizes;
    for (size_t k = 0; k < t.sizes.size(); ++k) sizes += (k ? ", " : "") + t.sizes[k].str();
    if (t.role == "weight") out += "tensor " + t.name + " = weight " + t.name.substr(1) + " [" + sizes + "]\n";
    else out += "tensor " + t.name + " = " + t.role + "[" + sizes + "]\n";
  }
  for (auto& st : nest.stages) {
    std::string pad;
    for (auto& a : st.axes) {
      out += pad + "for " + a.name + " in " + a.size.str() + ":\n";
      pad += "  ";
    }
    std::string target = st.tensor;
    if (!st.axes.empty()) {
      target += "[";
      for (size_t k = 0; k < st.axes.size(); ++k) target += (k ? ", " : "") + st.axes[k].name;
      target += "]";
    }
    std::string terms;
    for (size_t k = 0; k < st.terms.size(); ++k) {
      const Access& t = st.terms[k];
      if (k) terms += " * ";
      if (t.exprs.empty()) {
        terms += t.tensor;
      } else {
        terms += t.tensor + "[";
        for (size_t j = 0; j < t.exprs.size(); ++j) terms += (j ? ", " : "") + render_expr(t.exprs[j], true);
        terms += "]";
      }
    }
    if (!st.reduces.empty()) {
      out += pad + "acc = 0\n";
      std::string inner = pad;
      for (auto& r : st.reduces) {
        out += inner + "for " + r.name + " in " + r.size.str() + ":\n";
        inner += "  ";
      }
      out += inner + "acc += " + terms + "\n";
      out += pad + target + " = acc\n";
    } else {
      out += pad + target + " = " + terms + "\n";
    }
  }
  return out;
}

}  // namespace syno
