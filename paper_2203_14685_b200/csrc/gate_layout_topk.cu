// gate_layout_topk.cu -- instantiates the fused gate + layout kernel
// (gate_layout.cuh) for the top-k gate: every lane count L, register width
// K <= 8 and row segment U.
#include "gate_layout.cuh"

namespace moe {
FusedKernel pick_fused_topk(int L, int K, int U) { return pick_fused_l<KIND_TOPK>(L, K, U); }
}  // namespace moe
