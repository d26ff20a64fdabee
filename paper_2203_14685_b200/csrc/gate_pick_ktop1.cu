// gate_pick_ktop1.cu -- instantiates the k-top-1 gate kernels.
#include "gate_impl.cuh"

namespace moe {
GateKernel pick_ktop1(int L, int K) { return pick_l<KIND_KTOP1>(L, K); }
}  // namespace moe
