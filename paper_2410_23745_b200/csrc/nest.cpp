// Loop-nest lowering, staging and emission (see nest.hpp).
#include "nest.hpp"

#include <algorithm>
#include <cstring>

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



// ---------------------------------------------------------------------------
// parse_loop_nest (codegen.py:846-943) with the coordinate parser
// symexpr.parse_expr (symexpr.py:421-485) and its tokenizer (symexpr.py:502-531).
// Failures are SYNO_E_PARSE (LoopNestParseError / ExprParseError, both
// ValueErrors in the reference).
// ---------------------------------------------------------------------------

namespace {

[[noreturn]] void nest_error(const std::string& msg) { fail(SYNO_E_PARSE, msg); }

bool is_word(char c) { return isalnum((unsigned char)c) || c == '_'; }

bool all_digits(const std::string& s) {
  if (s.empty()) return false;
  for (char c : s)
    if (!isdigit((unsigned char)c)) return false;
  return true;
}

std::string strip(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && isspace((unsigned char)s[a])) ++a;
  while (b > a && isspace((unsigned char)s[b - 1])) --b;
  return s.substr(a, b - a);
}

std::vector<std::string> tokenize(const std::string& text) {  // symexpr._tokenize
  std::vector<std::string> tokens;
  size_t i = 0;
  while (i < text.size()) {
    const char c = text[i];
    if (isspace((unsigned char)c)) {
      ++i;
    } else if (std::string("+-*/%()^#").find(c) != std::string::npos) {
      if (c == '-' && !tokens.empty() && tokens.back() == "^") {
        size_t j = i + 1;
        while (j < text.size() && isdigit((unsigned char)text[j])) ++j;
        tokens.push_back(text.substr(i, j - i));
        i = j;
      } else {
        tokens.push_back(std::string(1, c));
        ++i;
      }
    } else if (is_word(c)) {
      size_t j = i;
      while (j < text.size() && is_word(text[j])) ++j;
      tokens.push_back(text.substr(i, j - i));
      i = j;
    } else {
      nest_error(std::string("bad character '") + c + "' in '" + text + "'");
    }
  }
  return tokens;
}

struct ExprParser {  // symexpr.parse_expr
  const std::string& text;
  std::vector<std::string> tokens;
  size_t pos = 0;
  const std::map<std::string, E>& iters;
  const std::map<std::string, Var>& vars;

  const std::string* peek() const { return pos < tokens.size() ? &tokens[pos] : nullptr; }
  std::string take() {
    if (pos >= tokens.size()) nest_error("unexpected end of input in '" + text + "'");
    return tokens[pos++];
  }
  static bool is_size(const E& e) { return e->op == Op::SizeRef; }
  E size_of(const std::string& name, int exp) {
    const Var& v = vars.at(name);
    std::map<std::string, std::pair<bool, int>> acc;
    acc[name] = {v.primary, exp};
    return mk_sizeref(size_from_powers(acc));
  }
  E atom() {
    std::string tok = take();
    if (tok == "(") {
      E inner = sum();
      if (take() != ")") nest_error("missing ')' in '" + text + "'");
      return inner;
    }
    std::string digits = tok;
    while (!digits.empty() && digits[0] == '-') digits.erase(0, 1);
    if (all_digits(digits)) {
      try {
        return mk_const(std::stoll(tok));
      } catch (const std::exception&) {
        nest_error("bad integer '" + tok + "' in '" + text + "'");
      }
    }
    int exp = 1;
    if (peek() && *peek() == "^") {
      take();
      std::string e = take();
      try {
        size_t used = 0;
        exp = std::stoi(e, &used);
        if (used != e.size()) throw std::invalid_argument(e);
      } catch (const std::exception&) {
        nest_error("bad exponent '" + e + "' in '" + text + "'");
      }
    }
    if (vars.count(tok) && exp != 1) return size_of(tok, exp);
    auto it = iters.find(tok);
    if (it != iters.end()) return it->second;
    if (vars.count(tok)) return size_of(tok, 1);
    nest_error("unknown name '" + tok + "' in '" + text + "'");
  }
  E product() {
    E node = atom();
    while (peek() && (*peek() == "*" || *peek() == "/" || *peek() == "%")) {
      const std::string op = take();
      E rhs = atom();
      if (op == "*" && is_size(node) && is_size(rhs)) node = mk_sizeref(size_mul(node->size, rhs->size));
      else if (op == "*") node = mk_bin(Op::Mul, node, rhs);
      else if (op == "/") node = mk_bin(Op::FloorDiv, node, rhs);
      else node = mk_bin(Op::Mod, node, rhs);
    }
    return node;
  }
  E sum() {
    E node = product();
    while (peek() && (*peek() == "+" || *peek() == "-")) {
      const std::string op = take();
      E rhs = product();
      node = mk_bin(op == "+" ? Op::Add : Op::Sub, node, rhs);
    }
    return node;
  }
  E parse() {
    tokens = tokenize(text);
    E r = sum();
    if (pos != tokens.size()) nest_error("trailing tokens in '" + text + "'");
    return r;
  }
};

SizeLike parse_sizelike(const std::string& raw, const std::map<std::string, Var>& vars) {
  SizeLike s;
  if (all_digits(raw)) {
    s.is_int = true;
    s.ival = std::stoll(raw);
  } else {
    try {
      s.sym = parse_size(raw, vars);
    } catch (const Error& e) {
      nest_error(e.what());
    }
  }
  return s;
}

int64_t extent_of(const SizeLike& s, const Assignment& env) { return s.is_int ? s.ival : eval_size(s.sym, env); }

// codegen._parse_terms: split on " * " outside index brackets.
std::vector<Access> parse_terms(const std::string& text, const std::map<std::string, E>& iters,
                                const std::map<std::string, Var>& vars) {
  std::vector<std::string> parts;
  int depth = 0;
  size_t start = 0;
  for (size_t k = 0; k < text.size(); ++k) {
    if (text[k] == '[') ++depth;
    else if (text[k] == ']') --depth;
    else if (depth == 0 && text.compare(k, 3, " * ") == 0) {
      parts.push_back(text.substr(start, k - start));
      start = k + 3;
      k += 2;
    }
  }
  parts.push_back(text.substr(start));
  std::vector<Access> terms;
  for (auto& raw : parts) {
    const std::string part = strip(raw);
    size_t name_end = 0;
    while (name_end < part.size() && is_word(part[name_end])) ++name_end;
    Access a;
    a.tensor = part.substr(0, name_end);
    if (name_end == 0) nest_error("bad term: '" + part + "'");
    if (name_end == part.size()) {
      terms.push_back(a);
      continue;
    }
    if (part[name_end] != '[' || part.back() != ']' ||
        part.find(']', name_end) != part.size() - 1)
      nest_error("bad term: '" + part + "'");
    const std::string inner = part.substr(name_end + 1, part.size() - name_end - 2);
    size_t s0 = 0;
    while (true) {
      size_t comma = inner.find(',', s0);
      std::string e = strip(inner.substr(s0, comma == std::string::npos ? std::string::npos : comma - s0));
      if (!e.empty()) a.exprs.push_back(ExprParser{e, {}, 0, iters, vars}.parse());
      if (comma == std::string::npos) break;
      s0 = comma + 1;
    }
    terms.push_back(a);
  }
  return terms;
}

// "<tensor>" or "<tensor>[...]" followed by " = <rest>"; false when the line has another shape.
bool split_target(const std::string& line, std::string* tensor, std::string* rest) {
  size_t k = 0;
  while (k < line.size() && is_word(line[k])) ++k;
  if (k == 0) return false;
  *tensor = line.substr(0, k);
  if (k < line.size() && line[k] == '[') {
    size_t close = line.find(']', k);
    if (close == std::string::npos || line.find('[', k + 1) < close) return false;
    k = close + 1;
  }
  if (line.compare(k, 3, " = ") != 0) return false;
  *rest = line.substr(k + 3);
  return !rest->empty();
}

}  // namespace

LoopNest parse_loop_nest(const std::string& text, const Spec& spec, const Assignment& env) {
  const auto vars = spec.var_map();
  std::vector<std::string> lines;
  {
    size_t s0 = 0;
    while (s0 <= text.size()) {
      size_t nl = text.find('\n', s0);
      std::string ln = text.substr(s0, nl == std::string::npos ? std::string::npos : nl - s0);
      if (!ln.empty() && ln.back() == '\r') ln.pop_back();
      if (!strip(ln).empty()) lines.push_back(ln);
      if (nl == std::string::npos) break;
      s0 = nl + 1;
    }
  }
  if (lines.empty() || lines[0].compare(0, 5, "nest ") != 0) nest_error("missing nest header");
  LoopNest nest;
  nest.name = strip(lines[0].substr(5));
  nest.env = env;
  size_t pos = 1;
  while (pos < lines.size() && lines[pos].compare(0, 7, "tensor ") == 0) {
    // ^tensor (\w+) = (input|output|stage|weight)(?: (\d+))? ?\[([^\]]*)\]$
    const std::string& ln = lines[pos];
    size_t k = 7;
    size_t n0 = k;
    while (k < ln.size() && is_word(ln[k])) ++k;
    TensorDecl t;
    t.name = ln.substr(n0, k - n0);
    bool ok = !t.name.empty() && ln.compare(k, 3, " = ") == 0;
    k += 3;
    if (ok) {
      ok = false;
      for (const char* role : {"input", "output", "stage", "weight"})
        if (ln.compare(k, strlen(role), role) == 0) {
          t.role = role;
          k += strlen(role);
          ok = true;
          break;
        }
    }
    if (ok && k < ln.size() && ln[k] == ' ' && k + 1 < ln.size() && isdigit((unsigned char)ln[k + 1])) {
      ++k;
      while (k < ln.size() && isdigit((unsigned char)ln[k])) ++k;
    }
    if (ok && k < ln.size() && ln[k] == ' ') ++k;
    ok = ok && k < ln.size() && ln[k] == '[' && ln.back() == ']' && ln.find(']', k) == ln.size() - 1;
    if (!ok) nest_error("bad tensor line: '" + ln + "'");
    const std::string raw = ln.substr(k + 1, ln.size() - k - 2);
    size_t s0 = 0;
    while (true) {
      size_t comma = raw.find(',', s0);
      std::string piece = strip(raw.substr(s0, comma == std::string::npos ? std::string::npos : comma - s0));
      if (!piece.empty()) {
        t.sizes.push_back(parse_sizelike(piece, vars));
        t.extents.push_back(extent_of(t.sizes.back(), env));
      }
      if (comma == std::string::npos) break;
      s0 = comma + 1;
    }
    nest.tensors.push_back(t);
    ++pos;
  }

  while (pos < lines.size()) {
    Stage st;
    std::map<std::string, E> iters;
    // `for <name> in <size>:` (codegen._FOR_RE); false when the line is not one
    auto read_for = [&](const std::string& line, Axis* axis) {
      const std::string s = strip(line);
      if (s.compare(0, 4, "for ") != 0 || s.back() != ':') return false;
      size_t k = 4;
      while (k < s.size() && is_word(s[k])) ++k;
      if (k == 4 || s.compare(k, 4, " in ") != 0) return false;
      const std::string name = s.substr(4, k - 4);
      const std::string raw = strip(s.substr(k + 4, s.size() - k - 5));
      if (raw.empty() || raw.find(':') != std::string::npos) return false;
      axis->name = name;
      axis->size = parse_sizelike(raw, vars);
      axis->extent = extent_of(axis->size, env);
      iters[name] = mk_iter(name, axis->size.is_int ? Size{} : axis->size.sym);
      return true;
    };
    while (pos < lines.size()) {
      Axis a;
      if (!read_for(lines[pos], &a)) break;
      const std::string body = pos + 1 < lines.size() ? strip(lines[pos + 1]) : "";
      st.axes.push_back(a);
      ++pos;
      if (body == "acc = 0") break;
    }
    if (pos >= lines.size()) nest_error("unexpected end of loop nest");
    std::string stripped = strip(lines[pos]);
    std::string tensor, rest;
    if (stripped == "acc = 0") {
      ++pos;
      while (pos < lines.size()) {
        Axis a;
        if (!read_for(lines[pos], &a)) break;
        st.reduces.push_back(a);
        ++pos;
      }
      if (pos >= lines.size()) nest_error("unexpected end of loop nest");
      stripped = strip(lines[pos]);
      if (stripped.compare(0, 7, "acc += ") != 0) nest_error("expected accumulation, got '" + stripped + "'");
      st.terms = parse_terms(stripped.substr(7), iters, vars);
      ++pos;
      if (pos >= lines.size()) nest_error("unexpected end of loop nest");
      stripped = strip(lines[pos]);
      if (!split_target(stripped, &tensor, &rest) || rest != "acc")
        nest_error("expected store, got '" + stripped + "'");
      ++pos;
    } else {
      if (!split_target(stripped, &tensor, &rest)) nest_error("expected assignment, got '" + stripped + "'");
      st.terms = parse_terms(rest, iters, vars);
      ++pos;
    }
    st.tensor = tensor;
    nest.stages.push_back(st);
  }
  return nest;
}

}  // namespace syno
