// Tensor-core (tcgen05) fast path for contraction-shaped stages.
#pragma once

#include <cuda_runtime.h>

#include "engine.hpp"

namespace syno {

// Runs `ds` on the tensor-core path when its shape allows it; returns false
// (and launches nothing) otherwise so the caller uses the universal kernel.
bool tc_try_stage(DType dt, const DevStage& ds, const Bindings& b, void* out, cudaStream_t stream);

}  // namespace syno
