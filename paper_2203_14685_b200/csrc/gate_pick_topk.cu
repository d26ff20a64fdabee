// gate_pick_topk.cu -- instantiates the top-k gate kernels (k_gate_select,
// KIND_TOPK, every lane count L and register width K).
#include "gate_impl.cuh"

namespace moe {
GateKernel pick_topk(int L, int K) { return pick_l<KIND_TOPK>(L, K); }
}  // namespace moe
