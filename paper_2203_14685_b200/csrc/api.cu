// api.cu -- the C ABI of libmoe_b200.so (include/moe.h): host-side argument
// validation (before anything is enqueued), error reporting, and dispatch to
// the kernels of gate.cu / layout.cu.  moe_alltoall lives in comm.cu.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "launch.cuh"

namespace moe {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

moe_status_t cuda_status(cudaError_t e, const char* what) {
  set_error("%s: CUDA error %d (%s)", what, (int)e, cudaGetErrorString(e));
  return MOE_ERR_CUDA;
}

int device_sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

// ------------------------------------------------------------ tuning table
// Filled once from the environment (MOE_<FIELD>), then only by
// moe_set_tuning: no launch reads the environment.
namespace {
struct TuneField {
  const char* env;
  int32_t moe_tuning_t::*f;
  int32_t dflt, lo, hi;
};
const TuneField kTune[] = {
    {"MOE_GATE_TILES", &moe_tuning_t::gate_tiles, 256, 1, 1 << 20},
    {"MOE_GATE_MAX_TILE", &moe_tuning_t::gate_max_tile, 0, 0, 256},
    {"MOE_GATE_TWO_MAXW", &moe_tuning_t::gate_two_maxw, 4096, 0, 1 << 30},
    {"MOE_LAYOUT_U", &moe_tuning_t::layout_u, 0, 0, 4},
    {"MOE_LAYOUT_PADS_FIRST", &moe_tuning_t::layout_pads_first, -1, -1, 1},
    {"MOE_REVERSE_KU", &moe_tuning_t::reverse_ku, 0, 0, 4},
    {"MOE_REVERSE_TPW", &moe_tuning_t::reverse_tpw, -1, -1, 1},
    {"MOE_REVERSE_KSPEC", &moe_tuning_t::reverse_kspec, 1, 0, 1},
    {"MOE_REVERSE_BACKWARDS", &moe_tuning_t::reverse_backwards, -1, -1, 1},
    {"MOE_REVERSE_Y_EF", &moe_tuning_t::reverse_y_ef, -1, -1, 1},
    {"MOE_ROW_CTAS_PER_SM", &moe_tuning_t::row_ctas_per_sm, 0, 0, 64},
    {"MOE_REVERSE_CTAS_PER_SM", &moe_tuning_t::reverse_ctas_per_sm, 0, 0, 64},
    {"MOE_COMBINE_CTAS_PER_SM", &moe_tuning_t::combine_ctas_per_sm, 8, 0, 64},
    {"MOE_COMBINE_BWD_KSPEC", &moe_tuning_t::combine_bwd_kspec, 1, 0, 1},
    {"MOE_GATE_BWD_LANES", &moe_tuning_t::gate_bwd_lanes, 0, 0, 32},
    {"MOE_P2P_DEDUPE", &moe_tuning_t::p2p_dedupe, 1, 0, 1},
    {"MOE_P2P_LOCAL_PAD", &moe_tuning_t::p2p_local_pad, -1, -1, 1},
    {"MOE_A2A_CTAS_PER_SM", &moe_tuning_t::a2a_ctas_per_sm, 4, 1, 64},
    {"MOE_BARRIER_TIMEOUT_MS", &moe_tuning_t::barrier_timeout_ms, 60000, 0, 1 << 30},
    {"MOE_BARRIER_PDL", &moe_tuning_t::barrier_pdl, 1, 0, 1},
    {"MOE_DISABLE_P2P", &moe_tuning_t::disable_p2p, 0, 0, 1},
    {"MOE_NCCL_ALLTOALL", &moe_tuning_t::nccl_alltoall, 0, 0, 1},
    {"MOE_NCCL_MAX_CTAS", &moe_tuning_t::nccl_max_ctas, 0, 0, 64},
    {"MOE_NCCL_MIN_CTAS", &moe_tuning_t::nccl_min_ctas, 0, 0, 64},
    {"MOE_NCCL_CTA_POLICY", &moe_tuning_t::nccl_cta_policy, -1, -1, 2},
    {"MOE_LAYOUT_TOKENS_PER_WARP", &moe_tuning_t::layout_tokens_per_warp, 2, 0, 1 << 20},
    {"MOE_P2P_PRECOMBINE", &moe_tuning_t::p2p_precombine, 1, 0, 1},
};
moe_tuning_t g_tune;
std::once_flag g_tune_once;

bool tune_valid(const moe_tuning_t& t) {
  for (const TuneField& f : kTune)
    if (t.*(f.f) < f.lo || t.*(f.f) > f.hi) {
      set_error("moe_set_tuning: %s = %d outside [%d, %d]", f.env, t.*(f.f), f.lo, f.hi);
      return false;
    }
  if (t.layout_u == 3 || t.reverse_ku == 1 || t.reverse_ku == 3) {
    set_error("moe_set_tuning: layout_u must be 0, 1, 2 or 4 and reverse_ku 0, 2 or 4");
    return false;
  }
  if (t.gate_bwd_lanes & (t.gate_bwd_lanes - 1)) {
    set_error("moe_set_tuning: gate_bwd_lanes must be 0 or a power of two");
    return false;
  }
  return true;
}
}  // namespace

const moe_tuning_t& tuning() {
  std::call_once(g_tune_once, [] {
    moe_tuning_t t{};
    for (const TuneField& f : kTune) {
      const char* v = getenv(f.env);
      t.*(f.f) = (v && *v) ? atoi(v) : f.dflt;
    }
    if (!tune_valid(t))  // a bad environment value: keep the defaults
      for (const TuneField& f : kTune) t.*(f.f) = f.dflt;
    g_tune = t;
  });
  return g_tune;
}

static bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

static int dtype_size(int32_t dt) { return dt == MOE_F32 ? 4 : dt == MOE_BF16 ? 2 : 0; }

// Checks shared by every call that takes a gate description.
static moe_status_t check_desc(const char* fn, const moe_gate_desc_t* d) {
  if (!d) {
    set_error("%s: desc is NULL", fn);
    return MOE_ERR_INVALID_ARG;
  }
  if (d->S < 1 || d->E < 1 || d->k < 1 || d->k > d->E || d->capacity < 1) {
    set_error("%s: need S>=1, E>=1, 1<=k<=E, capacity>=1 (S=%d E=%d k=%d capacity=%d)", fn, d->S,
              d->E, d->k, d->capacity);
    return MOE_ERR_INVALID_ARG;
  }
  if (d->kind < MOE_GATE_TOPK || d->kind > MOE_GATE_D2S) {
    set_error("%s: invalid gate kind %d", fn, d->kind);
    return MOE_ERR_INVALID_ARG;
  }
  if (d->weight_mode != MOE_W_RENORM && d->weight_mode != MOE_W_SOFTMAX) {
    set_error("%s: invalid weight_mode %d", fn, d->weight_mode);
    return MOE_ERR_INVALID_ARG;
  }
  if (d->priority != MOE_PRIO_TOKEN && d->priority != MOE_PRIO_SLOT) {
    set_error("%s: invalid priority %d", fn, d->priority);
    return MOE_ERR_INVALID_ARG;
  }
  if (d->kind == MOE_GATE_KTOP1 && d->E % d->k != 0) {
    set_error("%s: k-top-1 needs E %% k == 0 (E=%d, k=%d prototypes)", fn, d->E, d->k);
    return MOE_ERR_INVALID_ARG;
  }
  if (d->kind == MOE_GATE_D2S && d->k != d->E) {
    set_error("%s: Dense-to-Sparse needs k == E (every expert is a candidate slot; k=%d, E=%d)",
              fn, d->k, d->E);
    return MOE_ERR_INVALID_ARG;
  }
  if (d->kind == MOE_GATE_HASH && d->k != 1) {
    set_error("%s: hash gate needs k == 1 (k=%d)", fn, d->k);
    return MOE_ERR_INVALID_ARG;
  }
  if (d->E > 256) {
    set_error("%s: E=%d > 256 is not supported", fn, d->E);
    return MOE_ERR_UNSUPPORTED;
  }
  if ((long long)d->S * d->k >= (1ll << 30) || (long long)d->E * d->capacity >= (1ll << 31)) {
    set_error("%s: need S*k < 2^30 and E*capacity < 2^31 (S=%d k=%d E=%d capacity=%d)", fn, d->S,
              d->k, d->E, d->capacity);
    return MOE_ERR_UNSUPPORTED;
  }
  return MOE_OK;
}

static moe_status_t check_rows(const char* fn, const moe_gate_desc_t* d, const moe_routing_t* r,
                               const void* a, const char* an, const void* b, const char* bn,
                               int32_t dcols, int32_t dtype, bool need_weight, bool need_load) {
  moe_status_t s = check_desc(fn, d);
  if (s != MOE_OK) return s;
  if (!r || !r->expert_idx || !r->slot_idx || (need_weight && !r->weight) ||
      (need_load && !r->load)) {
    set_error("%s: routing or one of its required arrays is NULL", fn);
    return MOE_ERR_INVALID_ARG;
  }
  if (!a || !b) {
    set_error("%s: %s or %s is NULL", fn, an, bn);
    return MOE_ERR_INVALID_ARG;
  }
  const int ds = dtype_size(dtype);
  if (!ds) {
    set_error("%s: invalid dtype %d", fn, dtype);
    return MOE_ERR_INVALID_ARG;
  }
  if (dcols < 1) {
    set_error("%s: d=%d < 1", fn, dcols);
    return MOE_ERR_INVALID_ARG;
  }
  if (((long long)dcols * ds) % 16 != 0) {
    set_error("%s: row of d=%d x %d bytes is not a multiple of 16 bytes", fn, dcols, ds);
    return MOE_ERR_ALIGNMENT;
  }
  if (!aligned(a, 16) || !aligned(b, 16)) {
    set_error("%s: %s (%p) and %s (%p) must be 16-byte aligned", fn, an, a, bn, b);
    return MOE_ERR_ALIGNMENT;
  }
  return MOE_OK;
}

}  // namespace moe

using namespace moe;

extern "C" {

int32_t moe_capacity(int32_t S, int32_t E, int32_t k, double C) {
  if (S < 1 || E < 1 || k < 1 || !(C > 0.0)) return -1;
  const double c = std::ceil(C * (double)S * (double)k / (double)E);
  if (!(c >= 1.0) || c > 2147483647.0) return -1;
  return (int32_t)c;
}

int32_t moe_gate_kernel_count(const moe_gate_desc_t* desc, int32_t n_groups) {
  if (check_desc("moe_gate_kernel_count", desc) != MOE_OK) return -1;
  return gate_kernel_count(*desc, desc->kind == MOE_GATE_SAM ? std::max(1, n_groups) : 1);
}

size_t moe_gate_workspace_bytes(const moe_gate_desc_t* desc) {
  if (check_desc("moe_gate_workspace_bytes", desc) != MOE_OK) return 0;
  return gate_workspace_bytes(*desc);
}

moe_status_t moe_gate_ex(const moe_gate_desc_t* desc, const moe_gate_inputs_t* in,
                         const moe_routing_t* out, void* ws, size_t ws_bytes,
                         moe_stream_t stream) {
  moe_status_t s = gate_validate(desc, in, out, ws, ws_bytes);
  if (s != MOE_OK) return s;
  return gate_launch(*desc, *in, *out, ws, reinterpret_cast<cudaStream_t>(stream));
}

moe_status_t moe_gate_layout(const moe_gate_desc_t* desc, const moe_gate_inputs_t* in,
                             const moe_routing_t* out, void* ws, size_t ws_bytes, const void* x,
                             int32_t d, int32_t dtype, void* dispatch, moe_stream_t stream_) {
  moe_status_t s = gate_validate(desc, in, out, ws, ws_bytes);
  if (s != MOE_OK) return s;
  s = check_rows("moe_gate_layout", desc, out, x, "x", dispatch, "dispatch", d, dtype, false, true);
  if (s != MOE_OK) return s;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const int ds = dtype_size(dtype);
  if (!gate_layout_supported(*desc, d * ds)) {  // the two steps, one after the other
    s = gate_launch(*desc, *in, *out, ws, stream);
    if (s != MOE_OK) return s;
    return layout_launch(*desc, *out, x, ds, d, dispatch, stream);
  }
  PeerPtrs dst{};
  dst.p[0] = static_cast<char*>(dispatch);
  return gate_layout_launch(*desc, *in, *out, ws, x, ds, d, dst, desc->E, 0, nullptr, nullptr,
                            stream);
}

}  // extern "C"

moe_status_t moe::gate_validate(const moe_gate_desc_t* desc, const moe_gate_inputs_t* in,
                                const moe_routing_t* out, void* ws, size_t ws_bytes) {
  moe_status_t s = check_desc("moe_gate", desc);
  if (s != MOE_OK) return s;
  if (!in) {
    set_error("moe_gate: inputs are NULL");
    return MOE_ERR_INVALID_ARG;
  }
  if (!out || !out->expert_idx || !out->slot_idx || !out->weight || !out->load) {
    set_error("moe_gate: out or one of expert_idx/slot_idx/weight/load is NULL");
    return MOE_ERR_INVALID_ARG;
  }
  if (desc->kind == MOE_GATE_HASH) {
    if (!in->token_ids || !in->table || in->vocab < 1) {
      set_error("moe_gate: hash gate needs token_ids, table and vocab >= 1 (vocab=%d)", in->vocab);
      return MOE_ERR_INVALID_ARG;
    }
  } else if (!in->logits) {
    set_error("moe_gate: logits is NULL");
    return MOE_ERR_INVALID_ARG;
  } else if (!aligned(in->logits, 16)) {
    set_error("moe_gate: logits must be 16-byte aligned (TMA bulk copy source)");
    return MOE_ERR_ALIGNMENT;
  }
  if (desc->kind == MOE_GATE_SAM) {
    const int G = in->n_groups;
    if (!in->group_logits || G < 1 || desc->E % G != 0 || desc->k > desc->E / G) {
      set_error("moe_gate: SAM needs group_logits and n_groups dividing E with k <= E/n_groups "
                "(n_groups=%d E=%d k=%d)", G, desc->E, desc->k);
      return MOE_ERR_INVALID_ARG;
    }
    if (desc->k > 8) {
      set_error("moe_gate: SAM supports k <= 8 experts per group (k=%d)", desc->k);
      return MOE_ERR_UNSUPPORTED;
    }
  }
  if (desc->kind == MOE_GATE_D2S && (!(in->tau > 0.0) || !(in->eps >= 0.0))) {
    set_error("moe_gate: Dense-to-Sparse needs tau > 0 and eps >= 0 (tau=%g eps=%g)", in->tau,
              in->eps);
    return MOE_ERR_INVALID_ARG;
  }
  const size_t need = gate_workspace_bytes(*desc);
  if (!ws || ws_bytes < need) {
    set_error("moe_gate: workspace %zu bytes < %zu needed (or NULL)", ws_bytes, need);
    return MOE_ERR_WORKSPACE;
  }
  if (!aligned(ws, 16)) {
    set_error("moe_gate: workspace must be 16-byte aligned");
    return MOE_ERR_ALIGNMENT;
  }
  return MOE_OK;
}

extern "C" {

moe_status_t moe_gate(const moe_gate_desc_t* desc, const float* logits, const int32_t* token_ids,
                      const int32_t* table, int32_t vocab, const moe_routing_t* out, void* ws,
                      size_t ws_bytes, moe_stream_t stream) {
  if (desc && (desc->kind == MOE_GATE_SAM || desc->kind == MOE_GATE_D2S)) {
    set_error("moe_gate: SAM and Dense-to-Sparse gates take extra inputs: use moe_gate_ex");
    return MOE_ERR_INVALID_ARG;
  }
  moe_gate_inputs_t in{};
  in.logits = logits;
  in.token_ids = token_ids;
  in.table = table;
  in.vocab = vocab;
  return moe_gate_ex(desc, &in, out, ws, ws_bytes, stream);
}

moe_status_t moe_gate_check(void* ws, moe_stream_t stream, int32_t* bad_count) {
  if (!ws || !bad_count) {
    set_error("moe_gate_check: NULL ws or bad_count");
    return MOE_ERR_INVALID_ARG;
  }
  return gate_check(ws, reinterpret_cast<cudaStream_t>(stream), bad_count);
}

moe_status_t moe_layout(const moe_gate_desc_t* desc, const moe_routing_t* routing, const void* x,
                        int32_t d, int32_t dtype, void* dispatch, moe_stream_t stream) {
  moe_status_t s =
      check_rows("moe_layout", desc, routing, x, "x", dispatch, "dispatch", d, dtype, false, true);
  if (s != MOE_OK) return s;
  return layout_launch(*desc, *routing, x, dtype_size(dtype), d, dispatch,
                       reinterpret_cast<cudaStream_t>(stream));
}

moe_status_t moe_reverse_layout(const moe_gate_desc_t* desc, const moe_routing_t* routing,
                                const void* back, int32_t d, int32_t dtype, void* y,
                                moe_stream_t stream) {
  moe_status_t s = check_rows("moe_reverse_layout", desc, routing, back, "back", y, "y", d, dtype,
                              true, false);
  if (s != MOE_OK) return s;
  return reverse_launch(*desc, *routing, back, dtype, dtype_size(dtype), d, y,
                        reinterpret_cast<cudaStream_t>(stream));
}

moe_status_t moe_expert_offsets(const moe_gate_desc_t* desc, const moe_routing_t* routing,
                                int32_t* offsets, moe_stream_t stream) {
  moe_status_t s = check_desc("moe_expert_offsets", desc);
  if (s != MOE_OK) return s;
  if (!routing || !routing->load || !offsets) {
    set_error("moe_expert_offsets: routing.load and offsets are required");
    return MOE_ERR_INVALID_ARG;
  }
  return expert_offsets_launch(routing->load, desc->E, desc->capacity, offsets,
                               reinterpret_cast<cudaStream_t>(stream));
}

moe_status_t moe_layout_packed(const moe_gate_desc_t* desc, const moe_routing_t* routing,
                               const int32_t* offsets, const void* x, int32_t d, int32_t dtype,
                               void* packed, moe_stream_t stream) {
  moe_status_t s = check_rows("moe_layout_packed", desc, routing, x, "x", packed, "packed", d,
                              dtype, false, true);
  if (s != MOE_OK) return s;
  if (!offsets) {
    set_error("moe_layout_packed: offsets is NULL");
    return MOE_ERR_INVALID_ARG;
  }
  return layout_launch(*desc, *routing, x, dtype_size(dtype), d, packed,
                       reinterpret_cast<cudaStream_t>(stream), offsets);
}

moe_status_t moe_reverse_layout_packed(const moe_gate_desc_t* desc,
                                       const moe_routing_t* routing, const int32_t* offsets,
                                       const void* back, int32_t d, int32_t dtype, void* y,
                                       moe_stream_t stream) {
  moe_status_t s = check_rows("moe_reverse_layout_packed", desc, routing, back, "back", y, "y", d,
                              dtype, true, false);
  if (s != MOE_OK) return s;
  if (!offsets) {
    set_error("moe_reverse_layout_packed: offsets is NULL");
    return MOE_ERR_INVALID_ARG;
  }
  return reverse_launch(*desc, *routing, back, dtype, dtype_size(dtype), d, y,
                        reinterpret_cast<cudaStream_t>(stream), offsets);
}

moe_status_t moe_reverse_layout_backward(const moe_gate_desc_t* desc,
                                         const moe_routing_t* routing, const void* dy,
                                         const void* back, int32_t d, int32_t dtype,
                                         void* d_back, float* d_weight, moe_stream_t stream) {
  moe_status_t s = check_rows("moe_reverse_layout_backward", desc, routing, dy, "dy", back, "back",
                              d, dtype, true, true);
  if (s != MOE_OK) return s;
  if (!d_back || !d_weight || !aligned(d_back, 16)) {
    set_error("moe_reverse_layout_backward: d_back (16-byte aligned) and d_weight are required");
    return d_back && d_weight ? MOE_ERR_ALIGNMENT : MOE_ERR_INVALID_ARG;
  }
  PeerPtrs b{}, g{};
  b.p[0] = const_cast<char*>(static_cast<const char*>(back));
  g.p[0] = static_cast<char*>(d_back);
  return combine_bwd_launch(*desc, *routing, dy, b, g, desc->E, 0, dtype, dtype_size(dtype), d,
                            d_weight, reinterpret_cast<cudaStream_t>(stream));
}

moe_status_t moe_layout_backward(const moe_gate_desc_t* desc, const moe_routing_t* routing,
                                 const void* d_dispatch, int32_t d, int32_t dtype, void* dx,
                                 moe_stream_t stream) {
  moe_status_t s = check_rows("moe_layout_backward", desc, routing, d_dispatch, "d_dispatch", dx,
                              "dx", d, dtype, false, false);
  if (s != MOE_OK) return s;
  moe_routing_t unit = *routing;
  unit.weight = nullptr;  // the adjoint of the copy is the combine with w = 1
  return reverse_launch(*desc, unit, d_dispatch, dtype, dtype_size(dtype), d, dx,
                        reinterpret_cast<cudaStream_t>(stream));
}

moe_status_t moe_reverse_layout_packed_backward(const moe_gate_desc_t* desc,
                                                const moe_routing_t* routing,
                                                const int32_t* offsets, const void* dy,
                                                const void* back, int32_t d, int32_t dtype,
                                                void* d_back, float* d_weight,
                                                moe_stream_t stream) {
  moe_status_t s = check_rows("moe_reverse_layout_packed_backward", desc, routing, dy, "dy", back,
                              "back", d, dtype, true, false);
  if (s != MOE_OK) return s;
  if (!offsets || !d_back || !d_weight) {
    set_error("moe_reverse_layout_packed_backward: offsets, d_back and d_weight are required");
    return MOE_ERR_INVALID_ARG;
  }
  if (!aligned(d_back, 16)) {
    set_error("moe_reverse_layout_packed_backward: d_back must be 16-byte aligned");
    return MOE_ERR_ALIGNMENT;
  }
  PeerPtrs b{}, g{};
  b.p[0] = const_cast<char*>(static_cast<const char*>(back));
  g.p[0] = static_cast<char*>(d_back);
  return combine_bwd_launch(*desc, *routing, dy, b, g, desc->E, 0, dtype, dtype_size(dtype), d,
                            d_weight, reinterpret_cast<cudaStream_t>(stream), offsets);
}

moe_status_t moe_layout_packed_backward(const moe_gate_desc_t* desc,
                                        const moe_routing_t* routing, const int32_t* offsets,
                                        const void* d_packed, int32_t d, int32_t dtype, void* dx,
                                        moe_stream_t stream) {
  moe_status_t s = check_rows("moe_layout_packed_backward", desc, routing, d_packed, "d_packed",
                              dx, "dx", d, dtype, false, false);
  if (s != MOE_OK) return s;
  if (!offsets) {
    set_error("moe_layout_packed_backward: offsets is NULL");
    return MOE_ERR_INVALID_ARG;
  }
  moe_routing_t unit = *routing;
  unit.weight = nullptr;
  return reverse_launch(*desc, unit, d_packed, dtype, dtype_size(dtype), d, dx,
                        reinterpret_cast<cudaStream_t>(stream), offsets);
}

moe_status_t moe_gate_backward_ex(const moe_gate_desc_t* desc, const moe_gate_inputs_t* in,
                                  const moe_routing_t* routing, const float* d_weight,
                                  float* d_logits, float* d_group_logits, moe_stream_t stream) {
  moe_status_t s = check_desc("moe_gate_backward", desc);
  if (s != MOE_OK) return s;
  if (desc->kind == MOE_GATE_HASH) {
    set_error("moe_gate_backward: the hash gate has no logits (no gradient)");
    return MOE_ERR_INVALID_ARG;
  }
  if (!in || !in->logits || !routing || !routing->expert_idx || !routing->slot_idx ||
      !d_weight || !d_logits) {
    set_error("moe_gate_backward: logits, routing.expert_idx/slot_idx, d_weight, d_logits required");
    return MOE_ERR_INVALID_ARG;
  }
  if (desc->kind == MOE_GATE_SAM) {
    const int G = in->n_groups;
    if (!in->group_logits || !d_group_logits || G < 1 || desc->E % G != 0) {
      set_error("moe_gate_backward: SAM needs group_logits, d_group_logits and n_groups | E");
      return MOE_ERR_INVALID_ARG;
    }
  }
  if (desc->kind == MOE_GATE_D2S && !(in->tau > 0.0)) {
    set_error("moe_gate_backward: Dense-to-Sparse needs tau > 0");
    return MOE_ERR_INVALID_ARG;
  }
  return gate_bwd_launch(*desc, *in, *routing, d_weight, d_logits, d_group_logits,
                         reinterpret_cast<cudaStream_t>(stream));
}

moe_status_t moe_gate_backward(const moe_gate_desc_t* desc, const float* logits,
                               const moe_routing_t* routing, const float* d_weight,
                               float* d_logits, moe_stream_t stream) {
  if (desc && (desc->kind == MOE_GATE_SAM || desc->kind == MOE_GATE_D2S)) {
    set_error("moe_gate_backward: SAM and Dense-to-Sparse need moe_gate_backward_ex");
    return MOE_ERR_INVALID_ARG;
  }
  moe_gate_inputs_t in{};
  in.logits = logits;
  return moe_gate_backward_ex(desc, &in, routing, d_weight, d_logits, nullptr, stream);
}

moe_status_t moe_expert_scale(const void* in, void* out, int32_t nsrc, int32_t E_local,
                              int32_t e_base, int32_t cap, int32_t d, int32_t dtype,
                              moe_stream_t stream) {
  const int ds = dtype_size(dtype);
  if (!in || !out || nsrc < 1 || E_local < 1 || e_base < 0 || cap < 1 || d < 1 || !ds) {
    set_error("moe_expert_scale: bad arguments (nsrc=%d E_local=%d e_base=%d cap=%d d=%d dtype=%d)",
              nsrc, E_local, e_base, cap, d, dtype);
    return MOE_ERR_INVALID_ARG;
  }
  if (((long long)d * ds) % 16 != 0 || !aligned(in, 16) || !aligned(out, 16)) {
    set_error("moe_expert_scale: rows and pointers must be 16-byte aligned");
    return MOE_ERR_ALIGNMENT;
  }
  return expert_scale_launch(in, out, nsrc, E_local, e_base, cap, d, dtype, ds,
                             reinterpret_cast<cudaStream_t>(stream));
}

moe_status_t moe_set_trace(void* buf, size_t bytes) {
  g_trace.buf = bytes ? buf : nullptr;
  g_trace.bytes = buf ? bytes : 0;
  return MOE_OK;
}

moe_status_t moe_get_tuning(moe_tuning_t* out) {
  if (!out) {
    set_error("moe_get_tuning: out is NULL");
    return MOE_ERR_INVALID_ARG;
  }
  *out = tuning();
  return MOE_OK;
}

moe_status_t moe_set_tuning(const moe_tuning_t* t) {
  if (!t) {
    set_error("moe_set_tuning: NULL table");
    return MOE_ERR_INVALID_ARG;
  }
  tuning();  // the one-time environment read happens first, never after
  if (!tune_valid(*t)) return MOE_ERR_INVALID_ARG;
  g_tune = *t;
  return MOE_OK;
}

const char* moe_status_str(moe_status_t s) {
  switch (s) {
    case MOE_OK: return "MOE_OK";
    case MOE_ERR_INVALID_ARG: return "MOE_ERR_INVALID_ARG";
    case MOE_ERR_UNSUPPORTED: return "MOE_ERR_UNSUPPORTED";
    case MOE_ERR_ALIGNMENT: return "MOE_ERR_ALIGNMENT";
    case MOE_ERR_WORKSPACE: return "MOE_ERR_WORKSPACE";
    case MOE_ERR_CUDA: return "MOE_ERR_CUDA";
    case MOE_ERR_NCCL: return "MOE_ERR_NCCL";
    case MOE_ERR_TIMEOUT: return "MOE_ERR_TIMEOUT";
  }
  return "MOE_ERR_UNKNOWN";
}

const char* moe_last_error(void) { return g_err; }

const char* moe_version(void) {
  static char v[128];
  if (!v[0])
    snprintf(v, sizeof v, "libmoe_b200 sm_100a nccl-%d.%d.%d cuda-%d", NCCL_MAJOR, NCCL_MINOR,
             NCCL_PATCH, CUDART_VERSION);
  return v;
}

}  // extern "C"
