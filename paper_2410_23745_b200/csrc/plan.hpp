// Concrete execution plan: loop nests with every size evaluated, iterators
// renumbered as loop indices, batch axes made explicit, plus the backward
// stages derived from the unstaged nest.
//
// Every stage, forward or backward, has the one shape the reference's
// _run_stage evaluates (codegen.py:515-546):
//     out[axes] = scale * sum_{reduces} prod_terms term[coords(axes, reduces)]
// where a term reads zero when any coordinate is out of range
// (codegen.py:535-541).  Backward stages come from two derivations:
//   * gather form: the target term's coordinates are solved for loop
//     iterators ("transposed gather"); unsolved coordinates
//     become equality checks.  No atomics, deterministic.
//   * scatter form: the reference's own algorithm (codegen.py:727-742,
//     np.add.at) with device atomics, used when inversion would cost more.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "nest.hpp"

namespace syno {

enum class COp : uint8_t { Loop, Const, Add, Sub, Mul, FloorDiv, Mod };

struct CNode;
using CE = std::shared_ptr<const CNode>;
struct CNode {
  COp op;
  int loop = -1;       // Loop
  int64_t value = 0;   // Const
  CE lhs, rhs;
};

CE c_loop(int l);
CE c_const(int64_t v);
CE c_bin(COp op, CE a, CE b);
void c_loops(const CE& e, std::vector<int>* out);  // sorted unique loop ids
int64_t c_eval(const CE& e, const int64_t* loop_vals);
std::string c_render(const CE& e);

// Tensor roles bound at run time.
enum TensorKind : int {
  TK_X = 0,       // operator input (batch + input dims)
  TK_W = 1,       // weight j
  TK_STAGE = 2,   // intermediate t_k (workspace, accumulator precision)
  TK_Y = 3,       // operator output
  TK_DY = 4,      // upstream gradient
  TK_DX = 5,      // input gradient
  TK_DW = 6,      // weight gradient j
  TK_PHANTOM = 7, // validity-only term (value 1 when in range)
  TK_DSTAGE = 8,  // gradient of intermediate t_k (workspace, accumulator precision)
  TK_SCRATCH = 9, // engine-internal partial sums (accumulator precision)
  TK_SCRATCH_IN = 10, // engine-internal operand in the operator's dtype
  TK_PERM = 11,       // engine-internal permuted copy of an input (operator's dtype; DevStage::perm_in)
  TK_PRE = 12,        // engine-internal partial sums of a factored gather (accumulator precision; DevStage::gpre)
};

struct CTensor {
  int kind = TK_X;
  int index = 0;
  std::vector<int64_t> extents;
  int64_t numel() const {
    int64_t n = 1;
    for (auto e : extents) n *= e;
    return n;
  }
  bool operator==(const CTensor& o) const { return kind == o.kind && index == o.index; }
};

struct CTerm {
  CTensor t;
  std::vector<CE> coords;
};

struct CStage {
  std::vector<int64_t> axis_ext;  // loops [0, A)
  std::vector<int64_t> red_ext;   // loops [A, A+R)
  std::vector<CTerm> terms;
  CTensor out;                    // written row-major over the axes (gather form)
  bool scatter = false;           // scatter form: out is indexed by `target` instead
  CTerm target;
  double scale = 1.0;             // multiplicity of reduces no term reads
  bool dead = false;              // some term is never in range: out == 0
  int nloops() const { return (int)(axis_ext.size() + red_ext.size()); }
  int64_t ext(int l) const { return l < (int)axis_ext.size() ? axis_ext[l] : red_ext[l - axis_ext.size()]; }
  double grid_points() const;
  std::string describe() const;
};

struct Plan {
  bool nest_only = false;  // from a parsed multi-stage loop nest: forward (run_nest) on the stage engine only
  int64_t batch = 1;
  std::vector<int64_t> batch_ext;
  std::vector<int64_t> x_ext, y_ext;              // including batch
  std::vector<std::vector<int64_t>> w_ext;
  std::vector<std::vector<int64_t>> stage_ext;    // t_k extents (batch-prefixed when data-dependent)
  std::vector<CStage> forward;                    // staged or unstaged, in order
  CStage unstaged;                                // batch-explicit unstaged stage (backward source)
  std::vector<CStage> grad_x;                     // stages producing dX (one)
  std::vector<std::vector<CStage>> grad_w;        // per weight
  // Staged backward (SYNO_STAGED handles whose rfactored nest has several
  // stages and reads every tensor in exactly one term): reverse-mode through
  // the forward stages; outputs are TK_DX, TK_DW j or TK_DSTAGE k.  The
  // forward intermediates are recomputed first.  Empty: unstaged backward.
  std::vector<CStage> bwd_staged;
  int64_t flops_unstaged = 0, flops_staged = 0;   // codegen.flops, batch included
};

// Gradient of <dy, out> with respect to term j of stage S (gather form when
// the target's coordinates invert at acceptable cost, else scatter form).
CStage derive_gradient(const CStage& S, int j, const CTensor& grad);
// Same, with an explicit upstream tensor (dy, or the gradient of an intermediate).
CStage derive_gradient(const CStage& S, int j, const CTensor& grad, const CTensor& upstream);

// Quasi-affine simplification (csrc/simplify.cpp): the same values for every
// loop assignment within `loop_ext`, with multiples pulled out of floor
// divisions / modulos and range-resolved ones removed.
CE c_simplify(const CE& e, const std::vector<int64_t>& loop_ext);
// Interval bounds of e over the loop extents (false: unbounded / unknown).
bool c_range(const CE& e, const std::vector<int64_t>& loop_ext, int64_t* lo, int64_t* hi);
void simplify_stage(CStage* s);
// e as c0 + sum coef * atom over its top-level + - and constant products.
void c_sum_parts(const CE& e, int64_t* c0, std::vector<std::pair<int64_t, CE>>* parts);

Plan build_plan(const LoopNest& unstaged, const LoopNest& staged_or_same, const std::vector<Size>& batch_dims,
                const Assignment& env, bool derive_backward = true);

}  // namespace syno
