// gate_pick_topk.cu -- instantiates the top-k gate kernels (k_gate_select /
// k_gate_fused, KIND_TOPK, every lane count L and register width K).
#include "gate_impl.cuh"

namespace moe {
GateKernel pick_topk(int L, int K, bool fused) {
  return fused ? pick_l<KIND_TOPK, true>(L, K) : pick_l<KIND_TOPK, false>(L, K);
}
}  // namespace moe
