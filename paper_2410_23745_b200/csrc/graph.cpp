// pGraph replay and the operator text forms (see graph.hpp).
#include "graph.hpp"

#include <regex>
#include <set>
#include <sstream>

namespace syno {

static std::string strip(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && isspace((unsigned char)s[a])) ++a;
  while (b > a && isspace((unsigned char)s[b - 1])) --b;
  return s.substr(a, b - a);
}

static std::vector<std::string> split_on(const std::string& s, char sep) {
  std::vector<std::string> out;
  size_t start = 0;
  while (true) {
    size_t k = s.find(sep, start);
    out.push_back(s.substr(start, k == std::string::npos ? std::string::npos : k - start));
    if (k == std::string::npos) break;
    start = k + 1;
  }
  return out;
}

static std::vector<std::string> split_ws(const std::string& s) {
  std::vector<std::string> out;
  std::istringstream in(s);
  std::string tok;
  while (in >> tok) out.push_back(tok);
  return out;
}

std::map<std::string, Var> Spec::var_map() const {
  std::map<std::string, Var> m;
  for (auto& v : vars) m[v.name] = v;
  return m;
}

Assignment Spec::assignment() const {
  Assignment a;
  for (auto& kv : reference) a[kv.first] = kv.second;
  return a;
}

const Dim& Graph::dim_by_ident(int ident) const {
  for (auto& d : dims)
    if (d.ident == ident) return d;
  fail(SYNO_E_GRAPH, "no frontier dim with ident " + std::to_string(ident));
}

Graph graph_root(std::shared_ptr<const Spec> spec) {
  Graph g;
  g.spec = spec;
  for (size_t k = 0; k < spec->output_dims.size(); ++k) {
    Dim d;
    d.ident = (int)k;
    d.size = spec->output_dims[k];
    d.expr = mk_iter("i" + std::to_string(k), d.size);
    d.origin = "root";
    d.origin_step = -1;
    d.origin_pos = (int)k;
    g.dims.push_back(d);
  }
  g.next_id = (int)spec->output_dims.size();
  return g;
}

static bool reduce_pure(const E& e, const std::vector<E>& reduce_iters) {
  std::vector<E> fr;
  free_iterators(e, &fr);
  if (fr.empty()) return false;
  for (auto& it : fr) {
    bool found = false;
    for (auto& r : reduce_iters) found = found || r->name == it->name;
    if (!found) return false;
  }
  return true;
}

struct Produced {
  Size size;
  E expr;
  bool strided;
};

// pgraph._advance (pgraph.py:274-323)
static Graph advance(const Graph& g, const Step& step, const std::vector<Dim>& consumed,
                     const std::vector<Produced>& produced_specs, const std::vector<Weight>* weights,
                     E new_reduce) {
  Graph n;
  n.spec = g.spec;
  int step_index = (int)g.steps.size();
  n.reduce_iters = g.reduce_iters;
  if (new_reduce) n.reduce_iters.push_back(new_reduce);
  std::vector<Dim> produced;
  int ident = g.next_id;
  for (size_t pos = 0; pos < produced_specs.size(); ++pos) {
    Dim d;
    d.ident = ident++;
    d.size = produced_specs[pos].size;
    d.expr = produced_specs[pos].expr;
    d.origin = step.kind;
    d.origin_step = step_index;
    d.origin_pos = (int)pos;
    d.strided = produced_specs[pos].strided;
    d.reduce_pure = reduce_pure(d.expr, n.reduce_iters);
    produced.push_back(d);
  }
  std::set<int> consumed_ids;
  for (auto& d : consumed) consumed_ids.insert(d.ident);
  for (auto& d : g.dims)
    if (!consumed_ids.count(d.ident)) n.dims.push_back(d);
  for (auto& d : produced) n.dims.push_back(d);
  Step rec = step;
  rec.produced.clear();
  for (auto& d : produced) rec.produced.push_back(d.ident);
  n.weights = weights ? *weights : g.weights;
  n.steps = g.steps;
  n.steps.push_back(rec);
  n.in_reduction = g.in_reduction && step.kind == "reduce";
  n.after_contract = step.kind == "contract";
  n.next_id = ident;
  return n;
}

static std::vector<Dim> take_targets(const Graph& g, const Step& step, size_t arity,
                                     std::vector<bool> strided_ok = {}) {
  if (step.targets.size() != arity)
    fail(SYNO_E_GRAPH, step.kind + " takes " + std::to_string(arity) + " targets, got " +
                           std::to_string(step.targets.size()));
  std::set<int> uniq(step.targets.begin(), step.targets.end());
  if (uniq.size() != step.targets.size()) fail(SYNO_E_GRAPH, step.kind + " targets repeat");
  std::vector<Dim> dims;
  for (int t : step.targets) dims.push_back(g.dim_by_ident(t));
  if (strided_ok.empty()) strided_ok.assign(arity, false);
  for (size_t k = 0; k < dims.size(); ++k)
    if (dims[k].strided && !strided_ok[k])
      fail(SYNO_E_GRAPH, "strided dim " + std::to_string(dims[k].ident) + " may only be the data operand of unfold");
  return dims;
}

Graph graph_apply(const Graph& g, const Step& step_in) {
  static const std::set<std::string> kinds = {"reduce", "contract", "split", "merge",
                                              "shift", "expand", "unfold", "stride"};
  const std::string& kind = step_in.kind;
  if (!kinds.count(kind)) fail(SYNO_E_GRAPH, "unknown primitive '" + kind + "'");
  Step step = step_in;
  if (kind == "reduce") {  // pgraph.py:326-332
    if (!g.in_reduction) fail(SYNO_E_GRAPH, "reduce after the reduction stage ended");
    if (!step.has_param) fail(SYNO_E_GRAPH, "reduce needs a size parameter");
    if (!step.targets.empty()) fail(SYNO_E_GRAPH, "reduce takes no targets");
    E it = mk_iter("r" + std::to_string(g.reduce_iters.size()), step.param);
    return advance(g, step, {}, {{step.param, it, false}}, nullptr, it);
  }
  if (kind == "contract" && g.after_contract) fail(SYNO_E_GRAPH, "contraction directly after a contraction");
  if (kind == "contract") {  // pgraph.py:335-352
    if (step.targets.empty()) fail(SYNO_E_GRAPH, "contract needs at least one target");
    if (step.modes.size() != step.targets.size()) fail(SYNO_E_GRAPH, "contract needs one mode per target");
    for (auto& m : step.modes)
      if (m != "both" && m != "weight") fail(SYNO_E_GRAPH, "bad contract modes");
    auto dims = take_targets(g, step, step.targets.size());
    Weight w;
    std::vector<Produced> prod;
    for (size_t k = 0; k < dims.size(); ++k) {
      w.sizes.push_back(dims[k].size);
      w.exprs.push_back(dims[k].expr);
      if (step.modes[k] == "both") prod.push_back({dims[k].size, dims[k].expr, false});
    }
    std::vector<Weight> ws = g.weights;
    ws.push_back(w);
    return advance(g, step, dims, prod, &ws, nullptr);
  }
  if (kind == "split") {  // pgraph.py:355-362
    auto dims = take_targets(g, step, 2);
    const Dim &hi = dims[0], &lo = dims[1];
    Size coeff = lo.size;
    E expr = mk_bin(Op::Add, mk_bin(Op::Mul, mk_sizeref(coeff), hi.expr), lo.expr);
    if (step.has_param && step.param != coeff)
      fail(SYNO_E_GRAPH, "split coefficient mismatch: " + step.param.str() + " vs " + coeff.str());
    step.has_param = true;
    step.param = coeff;
    return advance(g, step, dims, {{size_mul(hi.size, coeff), expr, false}}, nullptr, nullptr);
  }
  if (kind == "merge") {  // pgraph.py:365-376
    auto dims = take_targets(g, step, 1);
    if (!step.has_param) fail(SYNO_E_GRAPH, "merge needs a size parameter");
    Size quot;
    if (!size_div(dims[0].size, step.param, &quot))
      fail(SYNO_E_GRAPH, step.param.str() + " does not divide " + dims[0].size.str());
    E q = mk_bin(Op::FloorDiv, dims[0].expr, mk_sizeref(step.param));
    E r = mk_bin(Op::Mod, dims[0].expr, mk_sizeref(step.param));
    return advance(g, step, dims, {{quot, q, false}, {step.param, r, false}}, nullptr, nullptr);
  }
  if (kind == "shift") {  // pgraph.py:379-382
    auto dims = take_targets(g, step, 1);
    E e = mk_bin(Op::Mod, mk_bin(Op::Add, dims[0].expr, mk_const(1)), mk_sizeref(dims[0].size));
    return advance(g, step, dims, {{dims[0].size, e, false}}, nullptr, nullptr);
  }
  if (kind == "expand") {  // pgraph.py:385-387
    auto dims = take_targets(g, step, 1);
    return advance(g, step, dims, {}, nullptr, nullptr);
  }
  if (kind == "unfold") {  // pgraph.py:390-394
    auto dims = take_targets(g, step, 2, {true, false});
    E off = mk_bin(Op::FloorDiv, mk_sizeref(dims[1].size), mk_const(2));
    E e = mk_bin(Op::Sub, mk_bin(Op::Add, dims[0].expr, dims[1].expr), off);
    return advance(g, step, dims, {{dims[0].size, e, false}}, nullptr, nullptr);
  }
  // stride, pgraph.py:397-403
  auto dims = take_targets(g, step, 1);
  if (!step.has_param) fail(SYNO_E_GRAPH, "stride needs a size parameter");
  Size sz = size_mul(step.param, dims[0].size);
  E e = mk_bin(Op::Mul, mk_sizeref(step.param), dims[0].expr);
  return advance(g, step, dims, {{sz, e, true}}, nullptr, nullptr);
}

bool match_input(const Graph& g, std::vector<int>* perm) {
  const auto& in = g.spec->input_dims;
  if (g.dims.size() != in.size()) return false;
  for (auto& d : g.dims)
    if (d.strided) return false;
  std::vector<bool> used(g.dims.size(), false);
  perm->clear();
  for (auto& size : in) {
    bool ok = false;
    for (size_t k = 0; k < g.dims.size(); ++k) {
      if (!used[k] && g.dims[k].size == size) {
        used[k] = true;
        perm->push_back((int)k);
        ok = true;
        break;
      }
    }
    if (!ok) return false;
  }
  return true;
}

// _STEP_RE = ^(?P<kind>[a-z]+)(?:\((?P<param>[^)]*)\))?(?:\[(?P<targets>[^\]]*)\])?$
static bool match_step(const std::string& part, std::string* kind, bool* has_param, std::string* param,
                       bool* has_targets, std::string* targets) {
  size_t k = 0;
  while (k < part.size() && part[k] >= 'a' && part[k] <= 'z') ++k;
  if (k == 0) return false;
  *kind = part.substr(0, k);
  *has_param = false;
  *has_targets = false;
  if (k < part.size() && part[k] == '(') {
    size_t close = part.find(')', k + 1);
    if (close == std::string::npos) return false;
    *param = part.substr(k + 1, close - k - 1);
    *has_param = true;
    k = close + 1;
  }
  if (k < part.size() && part[k] == '[') {
    size_t close = part.find(']', k + 1);
    if (close == std::string::npos) return false;
    *targets = part.substr(k + 1, close - k - 1);
    *has_targets = true;
    k = close + 1;
  }
  return k == part.size();
}

static int parse_target_int(const std::string& raw, const std::string& part) {
  std::string t = strip(raw);
  size_t k = 0;
  bool neg = false;
  if (!t.empty() && (t[0] == '-' || t[0] == '+')) { neg = t[0] == '-'; k = 1; }
  if (k >= t.size()) fail(SYNO_E_VALUE, "invalid literal for int(): '" + raw + "' in " + part);
  long v = 0;
  for (; k < t.size(); ++k) {
    if (t[k] < '0' || t[k] > '9') fail(SYNO_E_VALUE, "invalid literal for int(): '" + raw + "' in " + part);
    v = v * 10 + (t[k] - '0');
  }
  return (int)(neg ? -v : v);
}

Graph parse_steps(const std::string& text_in, std::shared_ptr<const Spec> spec) {
  std::string text = strip(text_in);
  if (!(text.size() >= 4 && text.compare(0, 3, "op{") == 0 && text.back() == '}'))
    fail(SYNO_E_PARSE, "expected op{...}, got '" + text.substr(0, 40) + "'");
  std::string body = strip(text.substr(3, text.size() - 4));
  Graph g = graph_root(spec);
  if (body.empty()) return g;
  auto vm = spec->var_map();
  for (auto raw : split_on(body, ';')) {
    std::string part = strip(raw);
    std::string kind, param, targets;
    bool has_param, has_targets;
    if (!match_step(part, &kind, &has_param, &param, &has_targets, &targets))
      fail(SYNO_E_PARSE, "bad step '" + part + "'");
    Step st;
    st.kind = kind;
    if (has_param && !param.empty()) {
      st.has_param = true;
      st.param = parse_size(param, vm);
    }
    if (has_targets && !targets.empty()) {
      for (auto item : split_on(targets, ',')) {
        item = strip(item);
        if (kind == "contract") {
          auto pair = split_on(item, ':');
          if (pair.size() != 2) fail(SYNO_E_PARSE, "bad contract targets '" + part + "'");
          st.targets.push_back(parse_target_int(pair[0], part));
          st.modes.push_back(pair[1]);
        } else {
          st.targets.push_back(parse_target_int(item, part));
        }
      }
    }
    try {
      g = graph_apply(g, st);
    } catch (const Error& err) {
      if (err.code == SYNO_E_GRAPH) fail(SYNO_E_PARSE, "cannot replay '" + part + "': " + err.what());
      throw;
    }
  }
  return g;
}

std::string print_steps(const Graph& g) {
  std::string out = "op{";
  for (size_t k = 0; k < g.steps.size(); ++k) {
    const Step& st = g.steps[k];
    if (k) out += "; ";
    if (st.kind == "reduce") {
      out += "reduce(" + st.param.str() + ")";
    } else if (st.kind == "contract") {
      out += "contract[";
      for (size_t j = 0; j < st.targets.size(); ++j) {
        if (j) out += ",";
        out += std::to_string(st.targets[j]) + ":" + st.modes[j];
      }
      out += "]";
    } else if (st.kind == "merge" || st.kind == "stride") {
      out += st.kind + "(" + st.param.str() + ")[" + std::to_string(st.targets[0]) + "]";
    } else {
      out += st.kind + "[";
      for (size_t j = 0; j < st.targets.size(); ++j) {
        if (j) out += ",";
        out += std::to_string(st.targets[j]);
      }
      out += "]";
    }
  }
  return out + "}";
}

std::string print_operator(const Graph& g) {
  const Spec& s = *g.spec;
  auto ref = s.assignment();
  std::string out = "operator " + s.name + "\n";
  for (auto& v : s.vars)
    out += "var " + v.name + (v.primary ? " primary " : " coefficient ") + std::to_string(ref[v.name]) + "\n";
  auto join = [](const std::vector<Size>& dims) {
    std::string r;
    for (size_t k = 0; k < dims.size(); ++k) r += (k ? " " : "") + dims[k].str();
    return r;
  };
  out += "output " + join(s.output_dims) + "\n";
  out += "input " + join(s.input_dims) + "\n";
  if (!s.batch_dims.empty()) out += "batch " + join(s.batch_dims) + "\n";
  out += "steps " + print_steps(g) + "\n";
  std::vector<int> perm;
  if (match_input(g, &perm)) {
    out += "perm";
    for (int p : perm) out += " " + std::to_string(p);
    out += "\n";
  }
  return out;
}

Graph parse_operator(const std::string& doc) {
  auto spec = std::make_shared<Spec>();
  bool have_name = false, have_steps = false, have_perm = false;
  std::string steps_text, perm_text;
  std::map<std::string, std::string> shapes;
  std::istringstream in(doc);
  std::string raw;
  while (std::getline(in, raw)) {
    std::string line = strip(raw);
    if (line.empty() || line[0] == '#') continue;
    size_t sp = line.find(' ');
    std::string head = line.substr(0, sp);
    std::string rest = sp == std::string::npos ? "" : line.substr(sp + 1);
    if (head == "operator") {
      spec->name = strip(rest);
      have_name = true;
    } else if (head == "var") {
      auto f = split_ws(rest);
      if (f.size() != 3 || (f[1] != "primary" && f[1] != "coefficient"))
        fail(SYNO_E_PARSE, "bad variable line '" + line + "'");
      spec->vars.push_back({f[0], f[1] == "primary"});
      try {
        size_t used = 0;
        long long v = std::stoll(f[2], &used);
        if (used != f[2].size()) throw std::invalid_argument("x");
        spec->reference.push_back({f[0], v});
      } catch (const std::exception&) {
        fail(SYNO_E_PARSE, "bad reference value in '" + line + "'");
      }
    } else if (head == "output" || head == "input" || head == "batch") {
      shapes[head] = rest;
    } else if (head == "steps") {
      steps_text = strip(rest);
      have_steps = true;
    } else if (head == "perm") {
      perm_text = rest;
      have_perm = true;
    } else {
      fail(SYNO_E_PARSE, "unknown line '" + line + "'");
    }
  }
  if (!have_name || !have_steps) fail(SYNO_E_PARSE, "document needs operator and steps lines");
  if (!shapes.count("output") || !shapes.count("input")) fail(SYNO_E_PARSE, "document needs output and input lines");
  auto vm = spec->var_map();
  auto shape = [&](const std::string& key) {
    std::vector<Size> out;
    if (!shapes.count(key)) return out;
    for (auto& tok : split_ws(shapes[key])) out.push_back(parse_size(tok, vm));
    return out;
  };
  spec->output_dims = shape("output");
  spec->input_dims = shape("input");
  spec->batch_dims = shape("batch");
  Graph g = parse_steps(steps_text, spec);
  if (have_perm) {
    std::vector<int> want;
    for (auto& t : split_ws(perm_text)) want.push_back(parse_target_int(t, perm_text));
    std::vector<int> got;
    if (!match_input(g, &got) || got != want) fail(SYNO_E_PARSE, "document permutation does not match");
  }
  return g;
}

}  // namespace syno
