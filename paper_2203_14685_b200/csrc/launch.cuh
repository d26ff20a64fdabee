// launch.cuh -- host-side launchers of the kernels (internal, C++): what
// api.cu / p2p.cu / comm.cu call after validating the C-ABI arguments.
#pragma once
#include "comm.cuh"

namespace moe {

// Steps 1 + 2 in one persistent kernel (gate_layout.cuh): the gate and the
// row scatter into `dst` (local: dst.p[0] = dispatch, E_local = E; peer
// mode: the owners' receive buffers, with the optional duplicate-row and
// padding-count tables of the one-sided dispatch).  UNSUPPORTED (nothing
// launched) when the shape has no fused kernel: SLOT priority, SAM, D2S,
// k > 8, rows not a multiple of 32 bytes; callers then launch gate + layout.
bool gate_layout_supported(const moe_gate_desc_t& d, int row_bytes);
struct TraceBuf {  // moe_set_trace: a device buffer of %globaltimer stamps
  void* buf = nullptr;
  size_t bytes = 0;
};
extern TraceBuf g_trace;
moe_status_t gate_layout_launch(const moe_gate_desc_t& d, const moe_gate_inputs_t& in,
                                const moe_routing_t& out, void* ws, const void* x,
                                int dtype_size, int dcols, const PeerPtrs& dst, int E_local,
                                int rank, const PeerPtrs* pad_tab, const PeerPtrs* dup_tab,
                                cudaStream_t stream,
                                const PeerPtrs* wt_tab = nullptr);
size_t gate_workspace_bytes(const moe_gate_desc_t& d);
// host checks of moe_gate_ex's arguments (api.cu), without launching
moe_status_t gate_validate(const moe_gate_desc_t* desc, const moe_gate_inputs_t* in,
                           const moe_routing_t* out, void* ws, size_t ws_bytes);
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
                                 const int32_t* peer_base = nullptr,
                                 const PeerPtrs* pad_tab = nullptr,
                                 const PeerPtrs* dup_tab = nullptr,
                                 const PeerPtrs* wt_tab = nullptr);
// The owner's half of the dispatch dedupe (RowArgs::dedupe): after the exit
// barrier, copy every recv row whose table entry says "= row i" and clear
// the entry.  tab: this rank's table, n_rows entries.
moe_status_t dup_fill_launch(char* recv, int* tab, long long n_rows, int row_bytes,
                             cudaStream_t stream, int* pairs = nullptr);
moe_status_t reverse_launch_peers(const moe_gate_desc_t& d, const moe_routing_t& r,
                                  const PeerPtrs& src, int E_local, int rank, int dtype,
                                  int dtype_size, int dcols, void* y, cudaStream_t stream,
                                  const int32_t* offsets = nullptr,
                                  const int32_t* peer_base = nullptr, int dup_alias = 0,
                                  const PeerPtrs* pre = nullptr);
// The peer combine kernel (k_reverse_k) serves this shape: k <= 2, rows a
// multiple of 32 bytes, tuning reverse_kspec (the pre-combined pairs need it).
bool reverse_kspec_used(const moe_gate_desc_t& d, int row_bytes);
// At least ~5% of the padded rows are padding by construction (E*cap >
// 1.05*S*k, e.g. the hash gate's C = 1.25): local padding over NVLink, and
// the padding rows zeroed first in local mode (L2 order for the combine).
inline bool pad_heavy(const moe_gate_desc_t& d) {
  return (double)d.E * d.capacity > 1.05 * (double)d.S * d.k;
}

moe_status_t expert_offsets_launch(const int32_t* load, int E, int cap, int32_t* offsets,
                                   cudaStream_t stream);
moe_status_t combine_bwd_launch(const moe_gate_desc_t& d, const moe_routing_t& r, const void* dy,
                                const PeerPtrs& back, const PeerPtrs& d_back, int E_local,
                                int rank, int dtype, int dtype_size, int dcols, float* d_weight,
                                cudaStream_t stream, const int32_t* offsets = nullptr,
                                const int32_t* peer_base = nullptr);
moe_status_t push_bwd_launch(const moe_gate_desc_t& d, const moe_routing_t& r, const PeerPtrs& wtab,
                             const PeerPtrs& dwtab, char* dbuf_local, const char* eo_local,
                             float* d_weight, int P, int rank, int dtype, int row_bytes, int phase,
                             cudaStream_t stream);
moe_status_t expert_scale_launch(const void* in, void* out, int nsrc, int E_local, int e_base,
                                 int cap, int dcols, int dtype, int dtype_size,
                                 cudaStream_t stream);
moe_status_t chunk_permute_launch(const void* src, void* dst, int N, int G, long long chunk_bytes,
                                  cudaStream_t stream);

}  // namespace moe
