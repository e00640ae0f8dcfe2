// Primitive graphs (pGraphs): replay of the reference's operator-construction
// API, /root/reference/pkg/src/opsmith/pgraph.py.  Only the replay half is
// restated (root/apply/match_input and the two text forms); legal-move
// enumeration is search-side and out of scope.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "symbolic.hpp"

namespace syno {

struct Spec {  // pgraph.ProblemSpec (pgraph.py:127-158), search knobs omitted
  std::string name;
  std::vector<Var> vars;
  std::vector<std::pair<std::string, int64_t>> reference;
  std::vector<Size> output_dims, input_dims, batch_dims;
  std::map<std::string, Var> var_map() const;
  Assignment assignment() const;
};

struct Dim {  // pgraph.Dim (pgraph.py:89-98)
  int ident;
  Size size;
  E expr;
  std::string origin;
  int origin_step, origin_pos;
  bool strided = false;
  bool reduce_pure = false;
};

struct Weight {  // pgraph.Weight (pgraph.py:101-104)
  std::vector<Size> sizes;
  std::vector<E> exprs;
};

struct Step {  // pgraph.Step (pgraph.py:107-124)
  std::string kind;
  std::vector<int> targets;
  bool has_param = false;
  Size param;
  std::vector<std::string> modes;
  std::vector<int> produced;
};

struct Graph {  // pgraph.PGraph (pgraph.py:161-181)
  std::shared_ptr<const Spec> spec;
  std::vector<Dim> dims;
  std::vector<Weight> weights;
  std::vector<Step> steps;
  bool in_reduction = true;
  bool after_contract = false;
  int next_id = 0;
  std::vector<E> reduce_iters;
  const Dim& dim_by_ident(int ident) const;
};

Graph graph_root(std::shared_ptr<const Spec> spec);              // pgraph.root (pgraph.py:184-202)
Graph graph_apply(const Graph& g, const Step& step);             // pgraph.apply (pgraph.py:223-251)
bool match_input(const Graph& g, std::vector<int>* perm);        // pgraph.match_input (pgraph.py:418-439)
Graph parse_steps(const std::string& text, std::shared_ptr<const Spec> spec);  // pgraph.py:675-709
Graph parse_operator(const std::string& doc);                    // pgraph.py:730-790
std::string print_steps(const Graph& g);                         // pgraph.py:659-672
std::string print_operator(const Graph& g);                      // pgraph.py:712-727
double graph_distance(const Graph& g);                             // shapedist.graph_distance (shapedist.py:415-420)

}  // namespace syno
