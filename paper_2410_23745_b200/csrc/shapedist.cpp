// Admissible distance from a partial graph's frontier to its input shape,
// restating /root/reference/pkg/src/opsmith/shapedist.py (the search-side
// hot spot, ~73% of MCTS CPU time in the reference).
//
// The algorithm is the reference's: the frontier dims and the input dims are
// partitioned into reshape groups, each group is priced by its cheapest
// reading (_group_options, shapedist.py:144-232) and the partition cost is
// minimised by a memoised recursion that pins the first remaining input (or
// dim) into the group under construction (_search, shapedist.py:280-333).
// Sizes are monomials over caller-chosen variable ids; the result does not
// depend on which ids name which variables, so every caller shares one memo.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/syno.h"
#include "graph.hpp"

namespace syno {
namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

using Powers = std::vector<std::pair<int, int>>;  // (variable id, exponent), sorted by id, no zeros

struct Desc {  // shapedist.DimDesc (shapedist.py:55-61)
  Powers pw;
  bool pure = false, strided = false;
  bool operator<(const Desc& o) const {
    if (pw != o.pw) return pw < o.pw;
    if (pure != o.pure) return pure < o.pure;
    return strided < o.strided;
  }
};

using Ids = std::vector<int>;
using Cost = std::pair<double, double>;  // (plain, any): shapedist.py:150-152

struct Solver {
  std::mutex mu;
  std::map<Desc, int> desc_ids;
  std::vector<Desc> descs;
  std::map<Powers, int> size_ids;
  std::vector<Powers> sizes;
  std::unordered_map<std::string, Cost> opt_memo, memo;

  int intern_desc(const Desc& d) {  // shapedist.py:114-124
    auto it = desc_ids.find(d);
    if (it != desc_ids.end()) return it->second;
    int i = (int)descs.size();
    desc_ids.emplace(d, i);
    descs.push_back(d);
    return i;
  }
  int intern_size(const Powers& p) {  // shapedist.py:127-134
    auto it = size_ids.find(p);
    if (it != size_ids.end()) return it->second;
    int i = (int)sizes.size();
    size_ids.emplace(p, i);
    sizes.push_back(p);
    return i;
  }

  static std::string key(const Ids& a, const Ids& b, bool may_reduce) {
    std::string k;
    const int na = (int)a.size();
    k.reserve(4 * (a.size() + b.size()) + 5);
    k.append(reinterpret_cast<const char*>(&na), sizeof(int));
    k.append(reinterpret_cast<const char*>(a.data()), a.size() * sizeof(int));
    k.append(reinterpret_cast<const char*>(b.data()), b.size() * sizeof(int));
    k.push_back(may_reduce ? '1' : '0');
    return k;
  }

  // _group_options (shapedist.py:144-232): the cheapest readings of one group.
  Cost group_options(const Ids& sub, const Ids& rhs, bool may_reduce) {
    const std::string k = key(sub, rhs, may_reduce);
    auto hit = opt_memo.find(k);
    if (hit != opt_memo.end()) return hit->second;
    Ids strided, normal;
    for (int i : sub) (descs[i].strided ? strided : normal).push_back(i);
    const int strided_n = (int)strided.size(), n_normal = (int)normal.size(), n_rhs = (int)rhs.size();
    std::map<int, int> base;  // -rhs content + strided content
    for (int i : rhs)
      for (auto& ve : sizes[i]) base[ve.first] -= ve.second;
    for (int i : strided)
      for (auto& ve : descs[i].pw) base[ve.first] += ve.second;
    bool strided_all_pure = true;
    for (int i : strided) strided_all_pure = strided_all_pure && descs[i].pure;
    double min_plain = kInf, min_any = kInf;
    // Every subset of the normal dims is a window choice; the minimum does
    // not depend on the enumeration order the reference uses.
    for (uint32_t windows = 0; windows < (1u << n_normal); ++windows) {
      std::map<int, int> q = base;
      int kept_normal = 0, w_pure = 0, wk = 0;
      bool kept_all_pure = true;
      for (int k2 = 0; k2 < n_normal; ++k2) {
        const Desc& d = descs[normal[k2]];
        if (windows >> k2 & 1) {
          ++wk;
          w_pure += d.pure;
        } else {
          ++kept_normal;
          kept_all_pure = kept_all_pure && d.pure;
          for (auto& ve : d.pw) q[ve.first] += ve.second;
        }
      }
      const int kept_n = strided_n + kept_normal;
      bool neg = false, pos = false;
      for (auto& ve : q) {
        neg = neg || ve.second < 0;
        pos = pos || ve.second > 0;
      }
      const int w_plain = wk - w_pure;
      const bool carve_pure = (kept_normal > 0 || strided_n > 0) && kept_all_pure && strided_all_pure;
      for (int repairs = 0; repairs < 2; ++repairs) {
        if (repairs && (!neg || kept_n == 0)) continue;
        int created = 0;
        if (neg && !repairs) {
          if (!may_reduce) continue;
          created = 1;
        }
        const int carve = pos ? 1 : 0;
        const int pure_items = w_pure + (carve_pure ? carve : 0);
        const int plain_items = w_plain + (carve_pure ? 0 : carve);
        const int slots = strided_n + repairs;
        int pure_left = pure_items - slots;
        const int slots_left = pure_left < 0 ? -pure_left : 0;
        if (pure_left < 0) pure_left = 0;
        const int plain_left = std::max(plain_items - slots_left, 0);
        double cost = strided_n + 2 * repairs + created + std::max(kept_n + created - 1, 0) +
                      std::max(n_rhs + carve - 1, 0) + pure_left;
        if (cost < min_any) min_any = cost;
        if (plain_left) cost += 1;
        if (cost < min_plain) min_plain = cost;
      }
    }
    Cost r{min_plain, min_any};
    opt_memo.emplace(k, r);
    return r;
  }

  // The first-group candidates in the reference's order (_splits, shapedist.py:253-277):
  // the first remaining input (or, once inputs run out, the first remaining dim) is pinned.
  template <typename F>
  static void for_splits(const Ids& dims, const Ids& tgts, F&& f) {
    Ids pinned, d_pool;
    std::vector<std::pair<Ids, Ids>> t_choices;
    if (!tgts.empty()) {
      const int n = (int)tgts.size() - 1;
      for (uint32_t m = 0; m < (1u << n); ++m) {
        Ids rhs{tgts[0]}, rem;
        for (int i = 0; i < n; ++i) (m >> i & 1 ? rhs : rem).push_back(tgts[i + 1]);
        t_choices.emplace_back(std::move(rhs), std::move(rem));
      }
      d_pool = dims;
    } else {
      t_choices.emplace_back();
      pinned.assign(dims.begin(), dims.begin() + 1);
      d_pool.assign(dims.begin() + 1, dims.end());
    }
    const int nd = (int)d_pool.size();
    for (uint32_t m = 0; m < (1u << nd); ++m) {
      Ids sub = pinned, rem_d;
      for (int i = 0; i < nd; ++i) (m >> i & 1 ? sub : rem_d).push_back(d_pool[i]);
      for (auto& tc : t_choices)
        if (!f(sub, tc.first, rem_d, tc.second)) return;
    }
  }

  // _search (shapedist.py:280-333)
  Cost search(const Ids& dims, const Ids& tgts, bool may_reduce) {
    const std::string k = key(dims, tgts, may_reduce);
    auto hit = memo.find(k);
    if (hit != memo.end()) return hit->second;
    if (dims.empty() && tgts.empty()) {
      memo.emplace(k, Cost{0, 0});
      return {0, 0};
    }
    double best_plain = kInf, best_any = kInf;
    for_splits(dims, tgts, [&](const Ids& sub, const Ids& rhs, const Ids& rem_d, const Ids& rem_t) {
      const Cost g = group_options(sub, rhs, may_reduce);
      if (g.second == kInf) return true;
      const Cost t = search(rem_d, rem_t, may_reduce);
      best_plain = std::min(best_plain, g.first + t.first);
      best_any = std::min(best_any, g.second + std::min(t.second, t.first));
      return true;
    });
    Cost r{best_plain, best_any};
    memo.emplace(k, r);
    return r;
  }

  // _witness (shapedist.py:336-362): one optimal grouping, walking the memoised costs.
  void witness(const Ids& dims, const Ids& tgts, bool may_reduce, bool flexible,
               std::vector<std::pair<Ids, Ids>>* groups) {
    if (dims.empty() && tgts.empty()) return;
    const Cost all = search(dims, tgts, may_reduce);
    const double want = flexible ? all.second : all.first;
    bool found = false;
    Ids nd, nt;
    for_splits(dims, tgts, [&](const Ids& sub, const Ids& rhs, const Ids& rem_d, const Ids& rem_t) {
      const Cost g = group_options(sub, rhs, may_reduce);
      const double head = flexible ? g.second : g.first;
      if (head == kInf) return true;
      const Cost t = search(rem_d, rem_t, may_reduce);
      const double tail = flexible ? std::min(t.first, t.second) : t.first;
      if (head + tail != want) return true;
      groups->emplace_back(sub, rhs);
      nd = rem_d;
      nt = rem_t;
      found = true;
      return false;
    });
    if (!found) fail(SYNO_E_INVALID, "shape distance: optimal cost has no matching grouping");
    witness(nd, nt, may_reduce, flexible, groups);
  }

  void clear() {  // shapedist.clear_cache (shapedist.py:423-433)
    memo.clear();
    opt_memo.clear();
    desc_ids.clear();
    descs.clear();
    size_ids.clear();
    sizes.clear();
  }
};

Solver& solver() {
  static Solver s;
  return s;
}

Powers read_powers(const int32_t* nterms, const int32_t* terms, int k, size_t* cursor) {
  std::map<int, int> acc;
  for (int t = 0; t < nterms[k]; ++t) {
    const int v = terms[2 * (*cursor)], e = terms[2 * (*cursor) + 1];
    ++*cursor;
    if (v < 0) fail(SYNO_E_INVALID, "shape distance: negative variable id");
    acc[v] += e;
  }
  Powers p;
  for (auto& ve : acc)
    if (ve.second) p.push_back(ve);
  return p;
}

struct Result {
  double distance = kInf;
  std::vector<int> dim_group, tgt_group;
  int n_groups = 0;
};

// explain_distance / shape_distance (shapedist.py:377-412) on descriptors.
Result distance(const std::vector<Desc>& current, const std::vector<Powers>& inputs, bool may_reduce,
                bool want_groups) {
  Solver& s = solver();
  std::lock_guard<std::mutex> lock(s.mu);
  std::vector<int> cur_ids, tgt_ids;
  for (auto& d : current) cur_ids.push_back(s.intern_desc(d));
  for (auto& p : inputs) tgt_ids.push_back(s.intern_size(p));
  Ids dims = cur_ids, tgts = tgt_ids;  // multiset-canonical keys (shapedist.py:365-374)
  std::sort(dims.begin(), dims.end());
  std::sort(tgts.begin(), tgts.end());
  const Cost c = s.search(dims, tgts, may_reduce);
  Result r;
  const bool flexible = !(c.first <= c.second + 1);
  r.distance = flexible ? c.second + 1 : c.first;
  if (!want_groups || r.distance == kInf) return r;
  std::vector<std::pair<Ids, Ids>> groups;
  s.witness(dims, tgts, may_reduce, flexible, &groups);
  r.dim_group.assign(current.size(), -1);
  r.tgt_group.assign(inputs.size(), -1);
  for (size_t g = 0; g < groups.size(); ++g) {
    for (int id : groups[g].first)
      for (size_t i = 0; i < cur_ids.size(); ++i)
        if (cur_ids[i] == id && r.dim_group[i] < 0) {
          r.dim_group[i] = (int)g;
          break;
        }
    for (int id : groups[g].second)
      for (size_t i = 0; i < tgt_ids.size(); ++i)
        if (tgt_ids[i] == id && r.tgt_group[i] < 0) {
          r.tgt_group[i] = (int)g;
          break;
        }
  }
  r.n_groups = (int)groups.size();
  return r;
}

Powers powers_of(const Size& size, std::map<std::string, int>* var_ids) {
  Powers p;
  for (auto& pw : size.p) {
    auto it = var_ids->emplace(pw.name, (int)var_ids->size()).first;
    p.emplace_back(it->second, pw.exp);
  }
  std::sort(p.begin(), p.end());
  return p;
}

}  // namespace

// graph_distance (shapedist.py:415-420) on a replayed graph.
double graph_distance(const Graph& g) {
  std::map<std::string, int> var_ids;
  std::vector<Desc> cur;
  for (auto& d : g.dims) cur.push_back(Desc{powers_of(d.size, &var_ids), d.reduce_pure, d.strided});
  std::vector<Powers> inputs;
  for (auto& s : g.spec->input_dims) inputs.push_back(powers_of(s, &var_ids));
  return distance(cur, inputs, g.in_reduction, false).distance;
}

}  // namespace syno

using namespace syno;

extern "C" int syno_capi_set_error(const char* msg);  // capi.cpp

extern "C" {

int syno_shape_distance(int n_dims, const int32_t* dim_nterms, const int32_t* dim_terms, const uint8_t* dim_flags,
                        int n_inputs, const int32_t* in_nterms, const int32_t* in_terms, int may_reduce,
                        double* out, int32_t* dim_group, int32_t* in_group, int32_t* n_groups) {
  try {
    if (!out || n_dims < 0 || n_inputs < 0 || (n_dims && (!dim_nterms || !dim_flags)) || (n_inputs && !in_nterms))
      fail(SYNO_E_INVALID, "null argument");
    if (n_dims > 24 || n_inputs > 24) fail(SYNO_E_UNSUPPORTED, "shape distance: more than 24 dims");
    std::vector<Desc> cur;
    size_t cursor = 0;
    for (int k = 0; k < n_dims; ++k) {
      if (dim_nterms[k] < 0 || (dim_nterms[k] && !dim_terms)) fail(SYNO_E_INVALID, "bad term count");
      Desc d;
      d.pw = read_powers(dim_nterms, dim_terms, k, &cursor);
      d.pure = dim_flags[k] & 1;
      d.strided = dim_flags[k] & 2;
      cur.push_back(d);
    }
    std::vector<Powers> inputs;
    cursor = 0;
    for (int k = 0; k < n_inputs; ++k) {
      if (in_nterms[k] < 0 || (in_nterms[k] && !in_terms)) fail(SYNO_E_INVALID, "bad term count");
      inputs.push_back(read_powers(in_nterms, in_terms, k, &cursor));
    }
    const bool want = dim_group || in_group || n_groups;
    Result r = distance(cur, inputs, may_reduce != 0, want);
    *out = r.distance;
    if (n_groups) *n_groups = r.n_groups;
    for (int k = 0; dim_group && k < n_dims; ++k) dim_group[k] = r.dim_group.empty() ? -1 : r.dim_group[k];
    for (int k = 0; in_group && k < n_inputs; ++k) in_group[k] = r.tgt_group.empty() ? -1 : r.tgt_group[k];
    return SYNO_OK;
  } catch (const Error& e) {
    syno_capi_set_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    syno_capi_set_error(e.what());
    return SYNO_E_INVALID;
  }
}

void syno_shape_distance_clear_cache(void) {
  Solver& s = solver();
  std::lock_guard<std::mutex> lock(s.mu);
  s.clear();
}

}  // extern "C"
