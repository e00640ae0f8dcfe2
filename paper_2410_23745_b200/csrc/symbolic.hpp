// Symbolic sizes and integer coordinate expressions.
//
// Restates the semantics of the reference's symexpr module
// (/root/reference/pkg/src/opsmith/symexpr.py): sizes are monomials over
// named variables (symexpr.py:35-66), coordinate expressions are small
// integer ASTs with PYTHON floor-division / modulo semantics
// (symexpr.py:9-12, 242-245).  Everything here is host code; the device
// side evaluates the same ASTs after they are compiled to postfix
// bytecode (plan.hpp).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/syno.h"

namespace syno {

// Status codes are the C ABI's (include/syno.h), one per reference exception family.


struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

// Python semantics for // and % on int64 (numpy int64 semantics for a zero divisor).
inline int64_t py_floordiv(int64_t a, int64_t b) {
  if (b == 0) return 0;
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
inline int64_t py_mod(int64_t a, int64_t b) {
  if (b == 0) return 0;
  int64_t r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) r += b;
  return r;
}

struct Var {
  std::string name;
  bool primary = true;
};

struct Pow {
  std::string name;
  bool primary;
  int exp;
  bool operator==(const Pow& o) const { return name == o.name && primary == o.primary && exp == o.exp; }
};

// A product of variable powers, sorted by name (symexpr.py:35-66).
struct Size {
  std::vector<Pow> p;
  bool operator==(const Size& o) const { return p == o.p; }
  bool operator!=(const Size& o) const { return !(p == o.p); }
  bool is_one() const { return p.empty(); }
  std::string str() const;
};

using Assignment = std::map<std::string, int64_t>;

Size size_from_powers(const std::map<std::string, std::pair<bool, int>>& acc);  // drops zeros, validates
Size size_mul(const Size& a, const Size& b);
bool size_div(const Size& a, const Size& b, Size* out);  // false when a primary would go negative
int64_t eval_size(const Size& s, const Assignment& env);
Size parse_size(const std::string& text, const std::map<std::string, Var>& vars);

// ---------------------------------------------------------------------------
// Coordinate expressions
// ---------------------------------------------------------------------------

enum class Op : uint8_t { Iter, Const, SizeRef, Add, Sub, Mul, FloorDiv, Mod };

struct Expr;
using E = std::shared_ptr<const Expr>;

struct Expr {
  Op op;
  std::string name;  // Iter
  Size size;         // Iter (its domain) / SizeRef
  int64_t value = 0; // Const
  E lhs, rhs;
};

E mk_iter(const std::string& name, const Size& size);
E mk_const(int64_t v);
E mk_sizeref(const Size& s);
E mk_bin(Op op, E a, E b);

bool is_binary(Op op);
bool expr_eq(const E& a, const E& b);   // structural equality (domains are not part of it)
size_t expr_hash(const E& a);

// Iterator names in traversal order (lhs first), first occurrence wins (symexpr.py:249-264).
void free_iterators(const E& e, std::vector<E>* out);
bool mentions(const E& e, const std::string& iter_name);

std::string render_expr(const E& e, bool spaced);
int64_t eval_expr(const E& e, const std::map<std::string, int64_t>& iters, const Assignment& env);

// Interval analysis, codegen._bounds (codegen.py:179-220).  Returns false for "None".
bool expr_bounds(const E& e, const std::map<std::string, std::pair<int64_t, int64_t>>& ranges,
                 const Assignment& env, int64_t* lo, int64_t* hi);

E rename_iters(const E& e, const std::map<std::string, std::string>& names);

}  // namespace syno
