// Symbolic sizes and coordinate expressions (see symbolic.hpp).
#include "symbolic.hpp"

#include <algorithm>
#include <functional>
#include <sstream>

namespace syno {

static std::string trim(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && isspace((unsigned char)s[a])) ++a;
  while (b > a && isspace((unsigned char)s[b - 1])) --b;
  return s.substr(a, b - a);
}

std::string Size::str() const {
  if (p.empty()) return "1";
  std::string out;
  for (size_t k = 0; k < p.size(); ++k) {
    if (k) out += "*";
    out += p[k].name;
    if (p[k].exp != 1) out += "^" + std::to_string(p[k].exp);
  }
  return out;
}

Size size_from_powers(const std::map<std::string, std::pair<bool, int>>& acc) {
  Size s;  // std::map iterates in name order, matching the reference's sort
  for (auto& kv : acc) {
    if (kv.second.second == 0) continue;
    if (kv.second.first && kv.second.second < 0)
      fail(SYNO_E_VALUE, "primary " + kv.first + " with negative exponent " + std::to_string(kv.second.second));
    s.p.push_back({kv.first, kv.second.first, kv.second.second});
  }
  return s;
}

static std::map<std::string, std::pair<bool, int>> to_acc(const Size& a) {
  std::map<std::string, std::pair<bool, int>> acc;
  for (auto& q : a.p) acc[q.name] = {q.primary, q.exp};
  return acc;
}

Size size_mul(const Size& a, const Size& b) {
  auto acc = to_acc(a);
  for (auto& q : b.p) {
    auto it = acc.find(q.name);
    if (it == acc.end()) acc[q.name] = {q.primary, q.exp};
    else it->second.second += q.exp;
  }
  return size_from_powers(acc);
}

bool size_div(const Size& a, const Size& b, Size* out) {
  auto acc = to_acc(a);
  for (auto& q : b.p) {
    auto it = acc.find(q.name);
    if (it == acc.end()) acc[q.name] = {q.primary, -q.exp};
    else it->second.second -= q.exp;
  }
  for (auto& kv : acc)
    if (kv.second.first && kv.second.second < 0) return false;
  *out = size_from_powers(acc);
  return true;
}

static int64_t ipow(int64_t v, int e) {
  int64_t r = 1;
  for (int k = 0; k < e; ++k) r *= v;
  return r;
}

int64_t eval_size(const Size& s, const Assignment& env) {
  int64_t num = 1, den = 1;
  for (auto& q : s.p) {
    auto it = env.find(q.name);
    if (it == env.end()) fail(SYNO_E_KEY, "'" + q.name + "'");
    int64_t val = it->second;
    if (val < 1) fail(SYNO_E_VALUE, "assignment for " + q.name + " must be >= 1, got " + std::to_string(val));
    if (q.exp > 0) num *= ipow(val, q.exp);
    else den *= ipow(val, -q.exp);
  }
  if (num % den != 0) fail(SYNO_E_NONINTEGRAL, s.str() + " is not integral under the assignment");
  return num / den;
}

static bool parse_py_int(const std::string& raw, int64_t* v) {
  std::string t = trim(raw);
  if (t.empty()) return false;
  size_t k = 0;
  bool neg = false;
  if (t[0] == '+' || t[0] == '-') { neg = t[0] == '-'; k = 1; }
  if (k >= t.size()) return false;
  int64_t acc = 0;
  for (; k < t.size(); ++k) {
    char c = t[k];
    if (c == '_') continue;
    if (c < '0' || c > '9') return false;
    acc = acc * 10 + (c - '0');
  }
  *v = neg ? -acc : acc;
  return true;
}

Size parse_size(const std::string& text_in, const std::map<std::string, Var>& vars) {
  std::string text = trim(text_in);
  if (text == "1") return Size{};
  std::map<std::string, std::pair<bool, int>> acc;
  size_t start = 0;
  while (true) {
    size_t star = text.find('*', start);
    std::string factor = trim(text.substr(start, star == std::string::npos ? std::string::npos : star - start));
    size_t caret = factor.find('^');
    std::string name = trim(factor.substr(0, caret));
    auto it = vars.find(name);
    if (it == vars.end()) fail(SYNO_E_VALUE, "unknown size variable '" + name + "' in '" + text + "'");
    int64_t exp = 1;
    if (caret != std::string::npos && caret + 1 < factor.size()) {
      if (!parse_py_int(factor.substr(caret + 1), &exp))
        fail(SYNO_E_VALUE, "invalid literal for int() in '" + text + "'");
    }
    auto& slot = acc[name];
    slot.first = it->second.primary;
    slot.second += (int)exp;
    if (star == std::string::npos) break;
    start = star + 1;
  }
  return size_from_powers(acc);
}

// ---------------------------------------------------------------------------

E mk_iter(const std::string& name, const Size& size) {
  auto e = std::make_shared<Expr>();
  e->op = Op::Iter; e->name = name; e->size = size;
  return e;
}
E mk_const(int64_t v) {
  auto e = std::make_shared<Expr>();
  e->op = Op::Const; e->value = v;
  return e;
}
E mk_sizeref(const Size& s) {
  auto e = std::make_shared<Expr>();
  e->op = Op::SizeRef; e->size = s;
  return e;
}
E mk_bin(Op op, E a, E b) {
  auto e = std::make_shared<Expr>();
  e->op = op; e->lhs = std::move(a); e->rhs = std::move(b);
  return e;
}

bool is_binary(Op op) { return op >= Op::Add; }

bool expr_eq(const E& a, const E& b) {
  if (a.get() == b.get()) return true;
  if (a->op != b->op) return false;
  switch (a->op) {
    case Op::Iter: return a->name == b->name && a->size == b->size;
    case Op::Const: return a->value == b->value;
    case Op::SizeRef: return a->size == b->size;
    default: return expr_eq(a->lhs, b->lhs) && expr_eq(a->rhs, b->rhs);
  }
}

size_t expr_hash(const E& a) {
  std::hash<std::string> hs;
  size_t h = (size_t)a->op * 0x9e3779b97f4a7c15ULL;
  switch (a->op) {
    case Op::Iter: return h ^ hs(a->name) ^ (hs(a->size.str()) << 1);
    case Op::Const: return h ^ std::hash<int64_t>()(a->value);
    case Op::SizeRef: return h ^ hs(a->size.str());
    default: return h ^ (expr_hash(a->lhs) * 31 + expr_hash(a->rhs) * 131);
  }
}

void free_iterators(const E& e, std::vector<E>* out) {
  if (e->op == Op::Iter) {
    for (auto& x : *out)
      if (x->name == e->name) return;
    out->push_back(e);
  } else if (is_binary(e->op)) {
    free_iterators(e->lhs, out);
    free_iterators(e->rhs, out);
  }
}

bool mentions(const E& e, const std::string& name) {
  if (e->op == Op::Iter) return e->name == name;
  if (is_binary(e->op)) return mentions(e->lhs, name) || mentions(e->rhs, name);
  return false;
}

static int prec_of(const E& e) {
  switch (e->op) {
    case Op::Add: case Op::Sub: return 1;
    case Op::Mul: case Op::FloorDiv: case Op::Mod: return 2;
    case Op::SizeRef: return e->size.p.size() > 1 ? 2 : 3;
    default: return 3;
  }
}

static void render_into(const E& e, bool spaced, std::string* out);

static void wrap(const E& c, int min_prec, bool spaced, std::string* out) {
  bool par = prec_of(c) < min_prec;
  if (par) *out += "(";
  render_into(c, spaced, out);
  if (par) *out += ")";
}

static void render_into(const E& e, bool spaced, std::string* out) {
  const char* sym = nullptr;
  int p = 0;
  switch (e->op) {
    case Op::Iter: *out += e->name; return;
    case Op::Const: *out += std::to_string(e->value); return;
    case Op::SizeRef: *out += e->size.str(); return;
    case Op::Add: sym = "+"; p = 1; break;
    case Op::Sub: sym = "-"; p = 1; break;
    case Op::Mul: sym = "*"; p = 2; break;
    case Op::FloorDiv: sym = "/"; p = 2; break;
    case Op::Mod: sym = "%"; p = 2; break;
  }
  wrap(e->lhs, p, spaced, out);
  if (spaced) *out += " ";
  *out += sym;
  if (spaced) *out += " ";
  wrap(e->rhs, p + 1, spaced, out);
}

std::string render_expr(const E& e, bool spaced) {
  std::string s;
  render_into(e, spaced, &s);
  return s;
}

int64_t eval_expr(const E& e, const std::map<std::string, int64_t>& iters, const Assignment& env) {
  switch (e->op) {
    case Op::Iter: {
      auto it = iters.find(e->name);
      if (it == iters.end()) fail(SYNO_E_KEY, "'" + e->name + "'");
      return it->second;
    }
    case Op::Const: return e->value;
    case Op::SizeRef: return eval_size(e->size, env);
    default: break;
  }
  int64_t a = eval_expr(e->lhs, iters, env), b = eval_expr(e->rhs, iters, env);
  switch (e->op) {
    case Op::Add: return a + b;
    case Op::Sub: return a - b;
    case Op::Mul: return a * b;
    case Op::FloorDiv: return py_floordiv(a, b);
    default: return py_mod(a, b);
  }
}

bool expr_bounds(const E& e, const std::map<std::string, std::pair<int64_t, int64_t>>& ranges,
                 const Assignment& env, int64_t* lo, int64_t* hi) {
  switch (e->op) {
    case Op::Iter: {
      auto it = ranges.find(e->name);
      if (it == ranges.end()) return false;
      *lo = it->second.first; *hi = it->second.second;
      return true;
    }
    case Op::Const: *lo = *hi = e->value; return true;
    case Op::SizeRef: *lo = *hi = eval_size(e->size, env); return true;
    default: break;
  }
  // Interval endpoints saturate at +-2^62 (the reference uses Python big
  // ints); saturated extents only ever make a staging look more expensive.
  auto sat = [](__int128 v) -> int64_t {
    const __int128 lim = (__int128)1 << 62;
    return (int64_t)(v > lim ? lim : v < -lim ? -lim : v);
  };
  int64_t alo, ahi, blo, bhi;
  if (!expr_bounds(e->lhs, ranges, env, &alo, &ahi)) return false;
  if (!expr_bounds(e->rhs, ranges, env, &blo, &bhi)) return false;
  switch (e->op) {
    case Op::Add: *lo = sat((__int128)alo + blo); *hi = sat((__int128)ahi + bhi); return true;
    case Op::Sub: *lo = sat((__int128)alo - bhi); *hi = sat((__int128)ahi - blo); return true;
    case Op::Mul: {
      int64_t c[4] = {sat((__int128)alo * blo), sat((__int128)alo * bhi), sat((__int128)ahi * blo),
                      sat((__int128)ahi * bhi)};
      *lo = *std::min_element(c, c + 4); *hi = *std::max_element(c, c + 4);
      return true;
    }
    case Op::FloorDiv: {
      if (blo <= 0) return false;
      int64_t c[4] = {py_floordiv(alo, blo), py_floordiv(alo, bhi), py_floordiv(ahi, blo), py_floordiv(ahi, bhi)};
      *lo = *std::min_element(c, c + 4); *hi = *std::max_element(c, c + 4);
      return true;
    }
    default: {  // Mod
      if (blo <= 0) return false;
      if (blo == bhi && py_floordiv(alo, blo) == py_floordiv(ahi, blo)) {
        *lo = py_mod(alo, blo); *hi = py_mod(ahi, blo);
        return true;
      }
      *lo = 0; *hi = bhi - 1;
      return true;
    }
  }
}

E rename_iters(const E& e, const std::map<std::string, std::string>& names) {
  switch (e->op) {
    case Op::Iter: {
      auto it = names.find(e->name);
      return it == names.end() ? e : mk_iter(it->second, e->size);
    }
    case Op::Const: case Op::SizeRef: return e;
    default: return mk_bin(e->op, rename_iters(e->lhs, names), rename_iters(e->rhs, names));
  }
}

}  // namespace syno
