// gate_pick_ktop1.cu -- instantiates the k-top-1 gate kernels.
#include "gate_impl.cuh"

namespace moe {
GateKernel pick_ktop1(int L, int K, bool fused) {
  return fused ? pick_l<KIND_KTOP1, true>(L, K) : pick_l<KIND_KTOP1, false>(L, K);
}
}  // namespace moe
