// gate_pick_misc.cu -- instantiates the hash, SAM and Dense-to-Sparse gate
// kernels.
#include "gate_impl.cuh"

namespace moe {

GateKernel pick_hash() { return k_gate_select<KIND_HASH, 1, 1>; }

template <int L>
static GateKernel pick_sam_k(int K) {
  switch (K) {
    case 1: return k_gate_select<KIND_SAM, L, 1>;
    case 2: return k_gate_select<KIND_SAM, L, 2>;
    case 4: return k_gate_select<KIND_SAM, L, 4>;
    default: return k_gate_select<KIND_SAM, L, 8>;
  }
}

GateKernel pick_sam(int L, int K) {
  switch (L) {
    case 1: return pick_sam_k<1>(K);
    case 2: return pick_sam_k<2>(K);
    case 4: return pick_sam_k<4>(K);
    case 8: return pick_sam_k<8>(K);
    case 16: return pick_sam_k<16>(K);
    default: return pick_sam_k<32>(K);
  }
}

GateKernel pick_d2s(int L) {
  switch (L) {
    case 1: return k_gate_select<KIND_D2S, 1, 1>;
    case 2: return k_gate_select<KIND_D2S, 2, 1>;
    case 4: return k_gate_select<KIND_D2S, 4, 1>;
    case 8: return k_gate_select<KIND_D2S, 8, 1>;
    case 16: return k_gate_select<KIND_D2S, 16, 1>;
    default: return k_gate_select<KIND_D2S, 32, 1>;
  }
}

}  // namespace moe
