// Concrete plan construction and backward-stage derivation (see plan.hpp).
#include "plan.hpp"

#include <algorithm>
#include <functional>
#include <map>
#include <set>
#include <sstream>

namespace syno {

CE c_loop(int l) {
  auto n = std::make_shared<CNode>();
  n->op = COp::Loop; n->loop = l;
  return n;
}
CE c_const(int64_t v) {
  auto n = std::make_shared<CNode>();
  n->op = COp::Const; n->value = v;
  return n;
}
CE c_bin(COp op, CE a, CE b) {
  if (a->op == COp::Const && b->op == COp::Const) {  // constant folding (Python semantics)
    int64_t x = a->value, y = b->value;
    switch (op) {
      case COp::Add: return c_const(x + y);
      case COp::Sub: return c_const(x - y);
      case COp::Mul: return c_const(x * y);
      case COp::FloorDiv: return c_const(py_floordiv(x, y));
      case COp::Mod: return c_const(py_mod(x, y));
      default: break;
    }
  }
  auto n = std::make_shared<CNode>();
  n->op = op; n->lhs = std::move(a); n->rhs = std::move(b);
  return n;
}

static void loops_into(const CE& e, std::set<int>* s) {
  if (e->op == COp::Loop) s->insert(e->loop);
  else if (e->op != COp::Const) { loops_into(e->lhs, s); loops_into(e->rhs, s); }
}
void c_loops(const CE& e, std::vector<int>* out) {
  std::set<int> s;
  loops_into(e, &s);
  out->assign(s.begin(), s.end());
}

int64_t c_eval(const CE& e, const int64_t* v) {
  switch (e->op) {
    case COp::Loop: return v[e->loop];
    case COp::Const: return e->value;
    default: break;
  }
  int64_t a = c_eval(e->lhs, v), b = c_eval(e->rhs, v);
  switch (e->op) {
    case COp::Add: return a + b;
    case COp::Sub: return a - b;
    case COp::Mul: return a * b;
    case COp::FloorDiv: return py_floordiv(a, b);
    default: return py_mod(a, b);
  }
}

std::string c_render(const CE& e) {
  switch (e->op) {
    case COp::Loop: return "L" + std::to_string(e->loop);
    case COp::Const: return std::to_string(e->value);
    default: break;
  }
  const char* s = e->op == COp::Add ? "+" : e->op == COp::Sub ? "-" : e->op == COp::Mul ? "*" : e->op == COp::FloorDiv ? "//" : "%";
  return "(" + c_render(e->lhs) + s + c_render(e->rhs) + ")";
}

double CStage::grid_points() const {
  double g = 1;
  for (auto e : axis_ext) g *= (double)e;
  for (auto e : red_ext) g *= (double)e;
  return g;
}

std::string CStage::describe() const {
  std::ostringstream o;
  static const char* kn[] = {"x", "w", "t", "y", "dy", "dx", "dw", "phantom", "dt", "acc", "op"};
  o << (scatter ? "scatter" : "gather") << " out=" << kn[out.kind] << out.index << " axes=[";
  for (size_t k = 0; k < axis_ext.size(); ++k) o << (k ? "," : "") << axis_ext[k];
  o << "] reduces=[";
  for (size_t k = 0; k < red_ext.size(); ++k) o << (k ? "," : "") << red_ext[k];
  o << "] scale=" << scale << " terms:";
  auto term = [&](const CTerm& t) {
    o << " " << kn[t.t.kind] << t.t.index << "[";
    for (size_t k = 0; k < t.coords.size(); ++k) o << (k ? "," : "") << c_render(t.coords[k]);
    o << "]";
  };
  for (auto& t : terms) term(t);
  if (scatter) { o << " target:"; term(target); }
  return o.str();
}

// ---------------------------------------------------------------------------

static CE to_concrete(const E& e, const std::map<std::string, int>& loop_of, const Assignment& env) {
  switch (e->op) {
    case Op::Iter: {
      auto it = loop_of.find(e->name);
      if (it == loop_of.end()) fail(SYNO_E_GRAPH, "iterator " + e->name + " is not a loop of its stage");
      return c_loop(it->second);
    }
    case Op::Const: return c_const(e->value);
    case Op::SizeRef: return c_const(eval_size(e->size, env));
    case Op::Add: return c_bin(COp::Add, to_concrete(e->lhs, loop_of, env), to_concrete(e->rhs, loop_of, env));
    case Op::Sub: return c_bin(COp::Sub, to_concrete(e->lhs, loop_of, env), to_concrete(e->rhs, loop_of, env));
    case Op::Mul: return c_bin(COp::Mul, to_concrete(e->lhs, loop_of, env), to_concrete(e->rhs, loop_of, env));
    case Op::FloorDiv: return c_bin(COp::FloorDiv, to_concrete(e->lhs, loop_of, env), to_concrete(e->rhs, loop_of, env));
    default: return c_bin(COp::Mod, to_concrete(e->lhs, loop_of, env), to_concrete(e->rhs, loop_of, env));
  }
}

// Reduces no term reads only multiply the sum by their extent.
static void fold_unread_reduces(CStage* s) {
  std::set<int> read;
  auto scan = [&](const CTerm& t) {
    for (auto& c : t.coords) loops_into(c, &read);
  };
  for (auto& t : s->terms) scan(t);
  // a reduce no term and no target coordinate reads repeats identical
  // contributions: for a gather sum and for a scatter alike it is a factor
  if (s->scatter) scan(s->target);
  int A = (int)s->axis_ext.size();
  std::vector<int64_t> keep;
  std::map<int, int> remap;
  for (int l = 0; l < A; ++l) remap[l] = l;
  for (size_t r = 0; r < s->red_ext.size(); ++r) {
    int l = A + (int)r;
    if (read.count(l)) {
      remap[l] = A + (int)keep.size();
      keep.push_back(s->red_ext[r]);
    } else {
      s->scale *= (double)s->red_ext[r];
    }
  }
  if (keep.size() == s->red_ext.size()) return;
  std::function<CE(const CE&)> rn = [&](const CE& e) -> CE {
    if (e->op == COp::Loop) return c_loop(remap.at(e->loop));
    if (e->op == COp::Const) return e;
    return c_bin(e->op, rn(e->lhs), rn(e->rhs));
  };
  for (auto& t : s->terms)
    for (auto& c : t.coords) c = rn(c);
  if (s->scatter)
    for (auto& c : s->target.coords) c = rn(c);
  s->red_ext = keep;
}

static CE subst(const CE& e, int l, const CE& by) {
  if (e->op == COp::Loop) return e->loop == l ? by : e;
  if (e->op == COp::Const) return e;
  CE a = subst(e->lhs, l, by), b = subst(e->rhs, l, by);
  if (a == e->lhs && b == e->rhs) return e;
  return c_bin(e->op, a, b);
}

static int count_loop(const CE& e, int l) {
  if (e->op == COp::Loop) return e->loop == l;
  if (e->op == COp::Const) return 0;
  return count_loop(e->lhs, l) + count_loop(e->rhs, l);
}

// True when e = sign*l + rest through Add/Sub nodes only.
static bool additive_path(const CE& e, int l) {
  if (e->op == COp::Loop) return e->loop == l;
  if (e->op == COp::Add || e->op == COp::Sub) {
    if (count_loop(e->lhs, l)) return additive_path(e->lhs, l);
    return additive_path(e->rhs, l);
  }
  return false;
}

// Split e = sign*l + rest.
static void linearize(const CE& e, int l, int* sign, CE* rest) {
  if (e->op == COp::Loop) { *sign = 1; *rest = c_const(0); return; }
  bool left = count_loop(e->lhs, l) > 0;
  int s;
  CE r;
  if (left) {
    linearize(e->lhs, l, &s, &r);
    *sign = s;
    *rest = c_bin(e->op, r, e->rhs);
  } else {
    linearize(e->rhs, l, &s, &r);
    *sign = e->op == COp::Sub ? -s : s;
    *rest = c_bin(e->op, e->lhs, r);
  }
}

static CStage remap_stage_loops(CStage s, const std::map<int, int>& m) {
  std::function<CE(const CE&)> rn = [&](const CE& e) -> CE {
    if (e->op == COp::Loop) return c_loop(m.at(e->loop));
    if (e->op == COp::Const) return e;
    return c_bin(e->op, rn(e->lhs), rn(e->rhs));
  };
  for (auto& t : s.terms)
    for (auto& c : t.coords) c = rn(c);
  return s;
}

// Gradient of <dy, out> with respect to term j of the unstaged stage S.
CStage derive_gradient(const CStage& S, int j, const CTensor& grad) {
  CTensor up;
  up.kind = TK_DY;
  up.extents = S.out.extents;
  return derive_gradient(S, j, grad, up);
}

CStage derive_gradient(const CStage& S, int j, const CTensor& grad, const CTensor& upstream) {
  const int L = S.nloops();
  const int A = (int)S.axis_ext.size();
  const CTerm& tj = S.terms[j];
  const int D = (int)tj.coords.size();
  CTerm up;
  up.t = upstream;
  for (int a = 0; a < A; ++a) up.coords.push_back(c_loop(a));

  // --- scatter form: the reference algorithm (codegen.py:727-742) ---------
  CStage sc;
  sc.axis_ext = S.axis_ext;
  sc.red_ext = S.red_ext;
  sc.terms.push_back(up);
  for (size_t t = 0; t < S.terms.size(); ++t)
    if ((int)t != j) sc.terms.push_back(S.terms[t]);
  sc.scatter = true;
  sc.target = tj;
  sc.target.t = grad;
  sc.out = grad;
  sc.scale = S.scale;
  double scatter_cost = S.grid_points();

  // --- gather form: solve the target coordinates for loop iterators -------
  // loops 0..L-1 are the original loops; L+d is the new axis for coordinate d.
  std::vector<CE> vals(L);           // current value of every original loop
  for (int l = 0; l < L; ++l) vals[l] = c_loop(l);
  std::vector<bool> solved(L, false);
  std::vector<std::pair<CE, int64_t>> checks;  // (expr, extent): 0 <= expr < extent
  for (int d = 0; d < D; ++d) {
    CE e = tj.coords[d];
    for (int l = 0; l < L; ++l)
      if (solved[l]) e = subst(e, l, vals[l]);
    CE vd = c_loop(L + d);
    int best = -1;
    for (int l = 0; l < L; ++l) {
      if (solved[l] || count_loop(e, l) != 1 || !additive_path(e, l)) continue;
      if (best < 0 || S.ext(l) > S.ext(best)) best = l;
    }
    if (best < 0) {
      checks.push_back({c_bin(COp::Sub, e, vd), 1});  // e == v_d
      continue;
    }
    int sign;
    CE rest;
    linearize(e, best, &sign, &rest);
    bool zero_rest = rest->op == COp::Const && rest->value == 0;
    CE sol = sign > 0 ? (zero_rest ? vd : c_bin(COp::Sub, vd, rest)) : c_bin(COp::Sub, rest, vd);
    for (int l = 0; l < L; ++l)
      if (solved[l]) vals[l] = subst(vals[l], best, sol);
    for (auto& c : checks) c.first = subst(c.first, best, sol);
    vals[best] = sol;
    solved[best] = true;
    bool exact = rest->op == COp::Const && rest->value == 0 && sign > 0 && grad.extents[d] <= S.ext(best);
    if (!exact) checks.push_back({sol, S.ext(best)});
  }
  double gather_cost = 1;
  for (auto e : grad.extents) gather_cost *= (double)e;
  std::vector<int> unsolved;
  for (int l = 0; l < L; ++l)
    if (!solved[l]) {
      unsolved.push_back(l);
      gather_cost *= (double)S.ext(l);
    }
  if (gather_cost > 4.0 * scatter_cost) return sc;

  CStage g;
  g.axis_ext = grad.extents;
  for (int l : unsolved) g.red_ext.push_back(S.ext(l));
  g.out = grad;
  g.scale = S.scale;
  auto rewrite = [&](const CE& e) {
    CE r = e;
    for (int l = 0; l < L; ++l)
      if (solved[l]) r = subst(r, l, vals[l]);
    return r;
  };
  CTerm gu = up;
  for (auto& c : gu.coords) c = rewrite(c);
  g.terms.push_back(gu);
  for (size_t t = 0; t < S.terms.size(); ++t) {
    if ((int)t == j) continue;
    CTerm ct = S.terms[t];
    for (auto& c : ct.coords) c = rewrite(c);
    g.terms.push_back(ct);
  }
  for (auto& c : checks) {
    CTerm ph;
    ph.t.kind = TK_PHANTOM;
    ph.t.extents = {c.second};
    ph.coords = {c.first};
    g.terms.push_back(ph);
  }
  std::map<int, int> m;
  for (int d = 0; d < D; ++d) m[L + d] = d;
  for (size_t k = 0; k < unsolved.size(); ++k) m[unsolved[k]] = D + (int)k;
  g = remap_stage_loops(g, m);
  fold_unread_reduces(&g);
  return g;
}

Plan build_plan(const LoopNest& unstaged, const LoopNest& staged, const std::vector<Size>& batch_dims,
                const Assignment& env, bool derive_backward) {
  Plan p;
  for (auto& s : batch_dims) {
    p.batch_ext.push_back(eval_size(s, env));
    p.batch *= p.batch_ext.back();
  }
  const int B = (int)p.batch_ext.size();
  auto prefixed = [&](const std::vector<int64_t>& e) {
    std::vector<int64_t> r = p.batch_ext;
    r.insert(r.end(), e.begin(), e.end());
    return r;
  };
  p.x_ext = prefixed(unstaged.tensor("x").extents);
  p.y_ext = prefixed(unstaged.tensor("y").extents);
  for (auto& t : unstaged.tensors)
    if (t.role == "weight") p.w_ext.push_back(t.extents);
  p.flops_unstaged = nest_flops(unstaged) * p.batch;
  p.flops_staged = nest_flops(staged) * p.batch;

  auto convert = [&](const LoopNest& nest, std::vector<CStage>* out, std::vector<std::vector<int64_t>>* stage_ext) {
    std::vector<bool> stage_data;
    for (auto& st : nest.stages) {
      bool data = false;
      for (auto& t : st.terms) {
        if (t.tensor == "x") data = true;
        if (t.tensor[0] == 't') data = data || stage_data.at(std::stoi(t.tensor.substr(1)));
      }
      CStage cs;
      std::map<std::string, int> loop_of;
      int nb = data ? B : 0;
      for (int b = 0; b < nb; ++b) cs.axis_ext.push_back(p.batch_ext[b]);
      for (auto& a : st.axes) {
        loop_of[a.name] = (int)cs.axis_ext.size();
        cs.axis_ext.push_back(a.extent);
      }
      for (auto& r : st.reduces) {
        loop_of[r.name] = (int)(cs.axis_ext.size() + cs.red_ext.size());
        cs.red_ext.push_back(r.extent);
      }
      for (auto& t : st.terms) {
        CTerm ct;
        bool tdata = false;
        if (t.tensor == "x") {
          ct.t.kind = TK_X;
          ct.t.extents = p.x_ext;
          tdata = true;
        } else if (t.tensor[0] == 'w') {
          ct.t.kind = TK_W;
          ct.t.index = std::stoi(t.tensor.substr(1));
          ct.t.extents = p.w_ext.at(ct.t.index);
        } else {
          ct.t.kind = TK_STAGE;
          ct.t.index = std::stoi(t.tensor.substr(1));
          ct.t.extents = stage_ext->at(ct.t.index);
          tdata = stage_data.at(ct.t.index);
        }
        if (tdata)
          for (int b = 0; b < B; ++b) ct.coords.push_back(c_loop(b));
        for (auto& e : t.exprs) ct.coords.push_back(to_concrete(e, loop_of, nest.env));
        cs.terms.push_back(ct);
      }
      if (st.tensor == "y") {
        cs.out.kind = TK_Y;
        cs.out.extents = p.y_ext;
      } else {
        cs.out.kind = TK_STAGE;
        cs.out.index = (int)stage_ext->size();
        cs.out.extents = cs.axis_ext;
        stage_ext->push_back(cs.axis_ext);
      }
      stage_data.push_back(data);
      fold_unread_reduces(&cs);
      out->push_back(cs);
    }
  };
  std::vector<CStage> un;
  std::vector<std::vector<int64_t>> un_ext;
  convert(unstaged, &un, &un_ext);
  p.unstaged = un.at(0);
  convert(staged, &p.forward, &p.stage_ext);

  if (!derive_backward) {
    p.nest_only = true;
    for (auto& st : p.forward) {
      simplify_stage(&st);
      fold_unread_reduces(&st);
    }
    return p;
  }
  // Backward always differentiates the unstaged nest, as the reference does
  // (codegen.py:680-681).  Gradients of reduces folded into `scale` keep it.
  CStage S = un.at(0);
  CTensor gx;
  gx.kind = TK_DX;
  gx.extents = p.x_ext;
  p.grad_x.push_back(derive_gradient(S, 0, gx));
  for (size_t j = 0; j < p.w_ext.size(); ++j) {
    CTensor gw;
    gw.kind = TK_DW;
    gw.index = (int)j;
    gw.extents = p.w_ext[j];
    p.grad_w.push_back({derive_gradient(S, (int)j + 1, gw)});
  }

  // Staged backward: reverse-mode through the rfactored stages when every
  // tensor is read by exactly one term (no gradient accumulation needed).
  if (p.forward.size() > 1 && &staged != &unstaged) {
    std::map<std::pair<int, int>, int> reads;  // (kind, index) -> count
    for (auto& st : p.forward)
      for (auto& t : st.terms) ++reads[{t.t.kind, t.t.index}];
    bool unique = true;
    for (auto& kv : reads) unique = unique && kv.second == 1 && kv.first.first != TK_PHANTOM;
    const int S = (int)p.forward.size();
    for (int k = 0; k + 1 < S && unique; ++k) unique = reads.count({TK_STAGE, k}) == 1;
    if (unique) {
      for (int k = S - 1; k >= 0; --k) {
        const CStage& F = p.forward[k];
        CTensor up;
        if (k == S - 1) {
          up.kind = TK_DY;
        } else {
          up.kind = TK_DSTAGE;
          up.index = k;
        }
        up.extents = F.out.extents;
        for (size_t j = 0; j < F.terms.size(); ++j) {
          const CTensor& t = F.terms[j].t;
          CTensor g;
          g.extents = t.extents;
          if (t.kind == TK_X) {
            g.kind = TK_DX;
          } else if (t.kind == TK_W) {
            g.kind = TK_DW;
            g.index = t.index;
          } else {
            g.kind = TK_DSTAGE;
            g.index = t.index;
          }
          p.bwd_staged.push_back(derive_gradient(F, (int)j, g, up));
        }
      }
    }
  }
  // the engine's stages get simplified coordinates (smaller index tables);
  // `unstaged` keeps the reference's form for the tensor-core matcher
  // (simplification can remove a reduce from every coordinate: fold it again)
  auto simp = [](CStage& st) {
    simplify_stage(&st);
    fold_unread_reduces(&st);
  };
  for (auto& st : p.forward) simp(st);
  for (auto& st : p.grad_x) simp(st);
  for (auto& gw : p.grad_w)
    for (auto& st : gw) simp(st);
  for (auto& st : p.bwd_staged) simp(st);
  return p;
}

}  // namespace syno
