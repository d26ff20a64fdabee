// gate_layout_misc.cu -- instantiates the fused gate + layout kernel
// (gate_layout.cuh) for the k-top-1 and hash gates.
#include "gate_layout.cuh"

namespace moe {
FusedKernel pick_fused_ktop1(int L, int K, int U) { return pick_fused_l<KIND_KTOP1>(L, K, U); }
FusedKernel pick_fused_hash(int U) {
  return U == 4 ? k_gate_layout<KIND_HASH, 1, 1, 4> : k_gate_layout<KIND_HASH, 1, 1, 2>;
}
}  // namespace moe
