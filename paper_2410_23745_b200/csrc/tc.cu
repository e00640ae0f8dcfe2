// Tensor-core fast path (placeholder until the tcgen05 kernels land).
#include "tc.hpp"

namespace syno {

bool tc_try_stage(DType, const DevStage&, const Bindings&, void*, cudaStream_t) { return false; }

}  // namespace syno
