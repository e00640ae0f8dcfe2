// Tensor-core (tcgen05) path for contraction-shaped operators.
//
// An operator qualifies when its unstaged stage (codegen.build_loop_nest,
// codegen.py:297-362) has the shape of a (strided, windowed) convolution in
// the broad sense: every x coordinate is a batch/pixel iterator, the one
// channel reduction, or an unfold window  S*i + r - c  (pgraph.py:390-403);
// every weight coordinate is a bare iterator; exactly one output axis is read
// only by weights (C_out / E3).  conv3x3, conv3x3_s2, sep_shared (two
// weights, folded), pointwise, 1x1-s2 shortcuts and QKV projections all
// match.  Everything else runs on the universal engine.
#pragma once

#include <cuda_runtime.h>

#include <memory>

#include "engine.hpp"

namespace syno {

// Host-only structural check (no device work): does the operator take the
// tensor-core path for bf16?
bool tc_matches(const Plan& plan);

// nullptr when the operator does not match (see above).
TcPlanPtr tc_build(const Plan& plan, cudaStream_t stream);

// bf16 only.  Return false (launching nothing) when not applicable.
bool tc_forward(TcPlan& tp, DType dt, const Bindings& b, cudaStream_t stream);
bool tc_backward(TcPlan& tp, DType dt, const Bindings& b, cudaStream_t stream);
std::string tc_describe(const TcPlan* tp);

}  // namespace syno
