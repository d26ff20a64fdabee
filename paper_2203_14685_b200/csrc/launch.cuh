// launch.cuh -- host-side launchers of the kernels (internal, C++): what
// api.cu / p2p.cu / comm.cu call after validating the C-ABI arguments.
#pragma once
#include "comm.cuh"

namespace moe {

size_t gate_workspace_bytes(const moe_gate_desc_t& d);
int gate_kernel_count(const moe_gate_desc_t& d, int ngroups);
moe_status_t gate_launch(const moe_gate_desc_t& d, const moe_gate_inputs_t& in,
                         const moe_routing_t& out, void* ws, cudaStream_t stream);
moe_status_t gate_check(void* ws, cudaStream_t stream, int32_t* bad);
moe_status_t gate_bwd_launch(const moe_gate_desc_t& d, const moe_gate_inputs_t& in,
                             const moe_routing_t& r, const float* d_weight, float* d_logits,
                             float* d_group_logits, cudaStream_t stream);

// offsets != NULL: the dropless packed form ([offsets[E]][row], no padding)
moe_status_t layout_launch(const moe_gate_desc_t& d, const moe_routing_t& r, const void* x,
                           int dtype_size, int dcols, void* dispatch, cudaStream_t stream,
                           const int32_t* offsets = nullptr);
moe_status_t reverse_launch(const moe_gate_desc_t& d, const moe_routing_t& r, const void* back,
                            int dtype, int dtype_size, int dcols, void* y, cudaStream_t stream,
                            const int32_t* offsets = nullptr);
moe_status_t layout_launch_peers(const moe_gate_desc_t& d, const moe_routing_t& r, const void* x,
                                 int dtype_size, int dcols, const PeerPtrs& dst, int E_local,
                                 int rank, cudaStream_t stream, const int32_t* offsets = nullptr,
                                 const int32_t* peer_base = nullptr);
moe_status_t reverse_launch_peers(const moe_gate_desc_t& d, const moe_routing_t& r,
                                  const PeerPtrs& src, int E_local, int rank, int dtype,
                                  int dtype_size, int dcols, void* y, cudaStream_t stream,
                                  const int32_t* offsets = nullptr,
                                  const int32_t* peer_base = nullptr);
moe_status_t expert_offsets_launch(const int32_t* load, int E, int cap, int32_t* offsets,
                                   cudaStream_t stream);
moe_status_t combine_bwd_launch(const moe_gate_desc_t& d, const moe_routing_t& r, const void* dy,
                                const PeerPtrs& back, const PeerPtrs& d_back, int E_local,
                                int rank, int dtype, int dtype_size, int dcols, float* d_weight,
                                cudaStream_t stream, const int32_t* offsets = nullptr,
                                const int32_t* peer_base = nullptr);
moe_status_t expert_scale_launch(const void* in, void* out, int nsrc, int E_local, int e_base,
                                 int cap, int dcols, int dtype, int dtype_size,
                                 cudaStream_t stream);
moe_status_t chunk_permute_launch(const void* src, void* dst, int N, int G, long long chunk_bytes,
                                  cudaStream_t stream);

}  // namespace moe
