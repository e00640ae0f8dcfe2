// Quasi-affine simplification of concrete coordinate expressions.
//
// Every coordinate the reference builds (pgraph.py:326-403) is a tree of
// + - * and floor division / modulo by evaluated sizes.  The reference
// evaluates the tree as written for every grid point (codegen.py:153-176).
// The device engine tabulates coordinates over the loops they depend on, so
// fewer dependencies mean smaller tables and loops that separate into an
// axis part and a reduce part.  The rewrite is exact over the loop ranges
// (Python floor semantics, positive divisors):
//
//   (B*Q + R) // B == Q + R // B        (B*Q + R) % B == R % B
//   R // B == k and R % B == R - k*B    when every R in range lies in [kB, kB+B)
//   (R // A) // B == R // (A*B)         (R % A) % B == R % B   when B | A
//
// with R's range from interval arithmetic over the loop extents.  Values
// are unchanged for every loop assignment inside the extents, so the
// index maps stay bit-exact to the reference's (tests/test_lowering.py,
// tests/test_gpu_parity.py compare the raw values).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <functional>
#include <map>

#include "plan.hpp"

namespace syno {

namespace {

struct Range {
  int64_t lo = 0, hi = 0;
  bool known = true;
};

struct Lin {
  int64_t c0 = 0;
  std::vector<std::pair<int64_t, CE>> terms;  // coefficient x atom (Loop, FloorDiv, Mod or opaque)
};

struct Ctx {
  const std::vector<int64_t>* ext;
  std::map<std::string, Range> memo;
};

Range range_of(const CE& e, Ctx& cx);

Range lin_range(const Lin& l, Ctx& cx) {
  Range r{l.c0, l.c0, true};
  for (auto& [c, a] : l.terms) {
    Range ar = range_of(a, cx);
    if (!ar.known) return Range{0, 0, false};
    // |values| stay far below 2^62 for the sizes an operator can have
    int64_t x = c * ar.lo, y = c * ar.hi;
    r.lo += std::min(x, y);
    r.hi += std::max(x, y);
  }
  return r;
}

Range range_of(const CE& e, Ctx& cx) {
  switch (e->op) {
    case COp::Loop: return Range{0, (*cx.ext)[e->loop] - 1, true};
    case COp::Const: return Range{e->value, e->value, true};
    default: break;
  }
  const std::string key = c_render(e);
  auto it = cx.memo.find(key);
  if (it != cx.memo.end()) return it->second;
  Range a = range_of(e->lhs, cx), b = range_of(e->rhs, cx), r{0, 0, false};
  if (a.known && b.known) {
    switch (e->op) {
      case COp::Add: r = Range{a.lo + b.lo, a.hi + b.hi, true}; break;
      case COp::Sub: r = Range{a.lo - b.hi, a.hi - b.lo, true}; break;
      case COp::Mul: {
        int64_t p[4] = {a.lo * b.lo, a.lo * b.hi, a.hi * b.lo, a.hi * b.hi};
        r = Range{*std::min_element(p, p + 4), *std::max_element(p, p + 4), true};
        break;
      }
      case COp::FloorDiv:
        if (b.lo == b.hi && b.lo > 0) r = Range{py_floordiv(a.lo, b.lo), py_floordiv(a.hi, b.lo), true};
        break;
      case COp::Mod:
        if (b.lo == b.hi && b.lo > 0) {
          if (py_floordiv(a.lo, b.lo) == py_floordiv(a.hi, b.lo)) r = Range{py_mod(a.lo, b.lo), py_mod(a.hi, b.lo), true};
          else r = Range{0, b.lo - 1, true};
        }
        break;
      default: break;
    }
  }
  cx.memo[key] = r;
  return r;
}

void add_term(Lin* l, int64_t c, const CE& a) {
  if (c == 0) return;
  const std::string key = c_render(a);
  for (auto& t : l->terms)
    if (c_render(t.second) == key) {
      t.first += c;
      return;
    }
  l->terms.push_back({c, a});
}

void lin_add(Lin* dst, const Lin& src, int64_t scale) {
  dst->c0 += scale * src.c0;
  for (auto& [c, a] : src.terms) add_term(dst, scale * c, a);
  dst->terms.erase(std::remove_if(dst->terms.begin(), dst->terms.end(),
                                  [](const std::pair<int64_t, CE>& t) { return t.first == 0; }),
                   dst->terms.end());
}

CE from_lin(const Lin& l) {
  // loops first (by index), then the nonlinear atoms, constant last
  std::vector<std::pair<int64_t, CE>> t = l.terms;
  std::stable_sort(t.begin(), t.end(), [](const std::pair<int64_t, CE>& a, const std::pair<int64_t, CE>& b) {
    bool la = a.second->op == COp::Loop, lb = b.second->op == COp::Loop;
    if (la != lb) return la;
    if (la) return a.second->loop < b.second->loop;
    return false;
  });
  CE acc;
  for (auto& [c, a] : t) {
    CE term = c == 1 ? a : c_bin(COp::Mul, c_const(c), a);
    if (!acc) acc = term;
    else acc = c_bin(COp::Add, acc, term);
  }
  if (!acc) return c_const(l.c0);
  if (l.c0 > 0) acc = c_bin(COp::Add, acc, c_const(l.c0));
  if (l.c0 < 0) acc = c_bin(COp::Sub, acc, c_const(-l.c0));
  return acc;
}

Lin to_lin(const CE& e, Ctx& cx);

Lin atom(const CE& a) {
  Lin l;
  l.terms.push_back({1, a});
  return l;
}

// e // B and e % B for a constant B > 0.
Lin divmod(const Lin& e, int64_t B, bool is_div, Ctx& cx) {
  Lin keep, rest;
  rest.c0 = py_mod(e.c0, B);
  keep.c0 = py_floordiv(e.c0, B);
  for (auto& [c, a] : e.terms) {
    if (c % B == 0) add_term(&keep, c / B, a);
    else add_term(&rest, c, a);
  }
  Range r = lin_range(rest, cx);
  if (r.known && py_floordiv(r.lo, B) == py_floordiv(r.hi, B)) {
    const int64_t k = py_floordiv(r.lo, B);
    if (is_div) {
      keep.c0 += k;
      return keep;
    }
    rest.c0 -= k * B;
    return rest;
  }
  if (!is_div) {
    // (R % A) % B == R % B when B divides A
    if (rest.c0 == 0 && rest.terms.size() == 1 && rest.terms[0].first == 1 && rest.terms[0].second->op == COp::Mod) {
      const CE& m = rest.terms[0].second;
      if (m->rhs->op == COp::Const && m->rhs->value % B == 0) return atom(c_bin(COp::Mod, m->lhs, c_const(B)));
    }
    return atom(c_bin(COp::Mod, from_lin(rest), c_const(B)));
  }
  Lin out = keep;
  // (R // A) // B == R // (A*B)
  if (rest.c0 == 0 && rest.terms.size() == 1 && rest.terms[0].first == 1 &&
      rest.terms[0].second->op == COp::FloorDiv && rest.terms[0].second->rhs->op == COp::Const &&
      rest.terms[0].second->rhs->value > 0) {
    const CE& d = rest.terms[0].second;
    add_term(&out, 1, c_bin(COp::FloorDiv, d->lhs, c_const(d->rhs->value * B)));
    return out;
  }
  add_term(&out, 1, c_bin(COp::FloorDiv, from_lin(rest), c_const(B)));
  return out;
}

Lin to_lin(const CE& e, Ctx& cx) {
  switch (e->op) {
    case COp::Loop: return atom(e);
    case COp::Const: {
      Lin l;
      l.c0 = e->value;
      return l;
    }
    case COp::Add:
    case COp::Sub: {
      Lin l = to_lin(e->lhs, cx);
      lin_add(&l, to_lin(e->rhs, cx), e->op == COp::Add ? 1 : -1);
      return l;
    }
    case COp::Mul: {
      Lin a = to_lin(e->lhs, cx), b = to_lin(e->rhs, cx);
      if (a.terms.empty()) std::swap(a, b);
      if (b.terms.empty()) {
        Lin l;
        lin_add(&l, a, b.c0);
        return l;
      }
      return atom(c_bin(COp::Mul, from_lin(a), from_lin(b)));  // opaque product
    }
    case COp::FloorDiv:
    case COp::Mod: {
      Lin a = to_lin(e->lhs, cx), b = to_lin(e->rhs, cx);
      if (b.terms.empty() && b.c0 > 0) return divmod(a, b.c0, e->op == COp::FloorDiv, cx);
      return atom(c_bin(e->op, from_lin(a), from_lin(b)));  // non-constant or non-positive divisor: as written
    }
  }
  return atom(e);
}

}  // namespace

CE c_simplify(const CE& e, const std::vector<int64_t>& loop_ext) {
  Ctx cx{&loop_ext, {}};
  return from_lin(to_lin(e, cx));
}

void c_sum_parts(const CE& e, int64_t* c0, std::vector<std::pair<int64_t, CE>>* parts) {
  Ctx cx{nullptr, {}};
  Lin l;
  // a structural walk (no range analysis: ext is not needed)
  std::function<void(const CE&, int64_t)> walk = [&](const CE& x, int64_t k) {
    if (x->op == COp::Const) { l.c0 += k * x->value; return; }
    if (x->op == COp::Add || x->op == COp::Sub) {
      walk(x->lhs, k);
      walk(x->rhs, x->op == COp::Add ? k : -k);
      return;
    }
    if (x->op == COp::Mul && x->lhs->op == COp::Const) { walk(x->rhs, k * x->lhs->value); return; }
    if (x->op == COp::Mul && x->rhs->op == COp::Const) { walk(x->lhs, k * x->rhs->value); return; }
    add_term(&l, k, x);
  };
  walk(e, 1);
  (void)cx;
  *c0 = l.c0;
  *parts = l.terms;
}

bool c_range(const CE& e, const std::vector<int64_t>& loop_ext, int64_t* lo, int64_t* hi) {
  Ctx cx{&loop_ext, {}};
  Range r = range_of(e, cx);
  *lo = r.lo;
  *hi = r.hi;
  return r.known;
}

// SYNO_CHECK_SIMPLIFY=1 (tests): compare every rewritten coordinate with the
// original at the loop-range corners and at pseudo-random grid points.
static void check_same(const CE& a, const CE& b, const std::vector<int64_t>& ext) {
  const int L = (int)ext.size();
  std::vector<int64_t> v(L);
  uint64_t st = 0x9E3779B97F4A7C15ull;
  for (int it = 0; it < 4096 + 2; ++it) {
    for (int l = 0; l < L; ++l) {
      if (it == 0) v[l] = 0;
      else if (it == 1) v[l] = ext[l] - 1;
      else {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        v[l] = (int64_t)((st >> 33) % (uint64_t)ext[l]);
      }
    }
    if (c_eval(a, v.data()) != c_eval(b, v.data()))
      fail(SYNO_E_GRAPH, "coordinate simplification changed a value: " + c_render(a) + " vs " + c_render(b));
  }
}

void simplify_stage(CStage* s) {
  static const bool check = getenv("SYNO_CHECK_SIMPLIFY") != nullptr;
  std::vector<int64_t> ext(s->axis_ext);
  ext.insert(ext.end(), s->red_ext.begin(), s->red_ext.end());
  auto one = [&](CE& c) {
    CE r = c_simplify(c, ext);
    if (check) check_same(c, r, ext);
    c = r;
  };
  for (auto& t : s->terms)
    for (auto& c : t.coords) one(c);
  if (s->scatter)
    for (auto& c : s->target.coords) one(c);
}

}  // namespace syno
