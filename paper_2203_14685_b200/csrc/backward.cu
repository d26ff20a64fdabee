// backward.cu -- the backward of the routing path:
// Algorithm 1 is a training process, so each forward
// step has an adjoint, with the routing held fixed.
//
//  k_combine_bwd  adjoint of step 6 + the combine:
//                 token-centric, one warp per token.  dy[t] is read once per
//                 admitted slot (L1-resident after the first), the expert
//                 output row once; each slot gets d_back[e][s] = w * dy[t]
//                 (a dispatch-style scatter: the product is exact in fp32
//                 for fp32 rows and in fp64 for bf16 rows, then rounded once,
//                 RNE) and d_weight[t,j] = <dy[t], back[e][s]> (fp32 FMA per
//                 lane in column order, warp tree reduction).  The padding
//                 rows of d_back are zero-filled in the same launch.  In peer
//                 mode the expert rows are read from, and the gradient rows
//                 stored into, the owner rank's memory over NVLink.
//  (adjoint of step 2 = the combine with unit weights: layout.cu's reverse
//   kernels with weight == NULL.)
//  k_gate_bwd     adjoint of Eq. 1's weights w.r.t. the
//                 logits: warp per token, fp64, one rounding to fp32.
#include "launch.cuh"
#include "rows.cuh"

namespace moe {

// RNE of the EXACT product w * v to bf16, in fp32/integer arithmetic: hi =
// RN_fp32(w*v), lo = the exact remainder (FMA).  RN to fp32 is monotone and
// every bf16 midpoint is an fp32 number, so RNE(hi) is the correct rounding
// unless hi sits exactly on a midpoint (low half 0x8000); then the sign of lo
// decides, and only an exact tie (lo == 0) goes to even.  Bit-identical to
// rounding the exact (fp64) product once.
__device__ __forceinline__ uint32_t mul_rne_bf16(float w, float v) {
  const float hi = __fmul_rn(w, v);
  const float lo = fmaf(w, v, -hi);
  const uint32_t b = __float_as_uint(hi);
  const uint32_t r = b & 0xFFFFu;
  uint32_t up;
  if (r == 0x8000u && lo != 0.f)
    up = ((lo > 0.f) == (hi > 0.f)) ? 1u : 0u;  // exact magnitude above the midpoint
  else
    up = (r > 0x8000u || (r == 0x8000u && (b & 0x10000u))) ? 1u : 0u;
  return (b >> 16) + up;
}

// Two lanes of a bf16x2 word: the common case is one hardware RNE convert of
// hi = RN_fp32(w*v) (cvt.rn.bf16x2.f32); only when either hi sits exactly on
// a bf16 midpoint (low half 0x8000, ~2^-16 of values) is the exact
// remainder consulted (mul_rne_bf16).  Same bits as mul_rne_bf16 on both.
__device__ __forceinline__ uint32_t mul2_rne_bf16(float w, uint32_t v2) {
  const float a = bf16lo(v2), b = bf16hi(v2);
  const float ha = __fmul_rn(w, a), hb = __fmul_rn(w, b);
  const uint32_t ba = __float_as_uint(ha), bb = __float_as_uint(hb);
  if (((ba & 0xFFFFu) == 0x8000u) | ((bb & 0xFFFFu) == 0x8000u))
    return mul_rne_bf16(w, a) | (mul_rne_bf16(w, b) << 16);
  return pack_bf16x2(ha, hb);
}

template <int DT>
__device__ __forceinline__ V8 scale_vec(float w, const V8& v) {
  V8 o;
  if constexpr (DT == MOE_F32) {
#pragma unroll
    for (int q = 0; q < 8; ++q) o.w[q] = __float_as_uint(__fmul_rn(w, __uint_as_float(v.w[q])));
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) o.w[q] = mul2_rne_bf16(w, v.w[q]);
  }
  return o;
}

template <int DT>
__device__ __forceinline__ float dot_vec(const V8& a, const V8& b, float acc) {
  if constexpr (DT == MOE_F32) {
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = fmaf(__uint_as_float(a.w[q]), __uint_as_float(b.w[q]), acc);
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      acc = fmaf(bf16lo(a.w[q]), bf16lo(b.w[q]), acc);
      acc = fmaf(bf16hi(a.w[q]), bf16hi(b.w[q]), acc);
    }
  }
  return acc;
}

// a.src = dy [S, row]; a.speer = expert outputs [E][cap][row] (per owner);
// a.dpeer = d_back, same mapping; a.weight = combine weights.
template <int DT, int U>
__global__ void __launch_bounds__(kRowThreads) k_combine_bwd(RowArgs a, float* d_weight) {
  constexpr int VB = 32, SEG = 32 * U * VB;
  __shared__ int s_beg[257];
  pdl_wait();
  pdl_trigger();
  pad_prefix(a, s_beg);
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  const int nw = gridDim.x * kRowWarps;
  if (a.pads_first) zero_pad_rows<32>(a, s_beg, gw, nw);  // see RowArgs::pads_first
  for (int t = gw; t < a.S; t += nw) {
    const char* dyrow = a.src + (size_t)t * a.row_bytes;
    for (int j = 0; j < a.k; ++j) {
      const size_t i = (size_t)t * a.k + j;
      const int s = __ldg(a.slot_idx + i);
      if (s < 0) {
        if (lane == 0) d_weight[i] = 0.f;
        continue;
      }
      const int e = __ldg(a.expert_idx + i);
      const float w = __ldg(a.weight + i);
      const char* brow = src_row(a, e, s);
      char* drow = dst_row_of(a, e, s);
      float dot = 0.f;
      for (int seg = 0; seg < a.row_bytes; seg += SEG) {
        V8 g[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int off = seg + (lane + 32 * u) * VB;
          if (off < a.row_bytes) {
            g[u] = ld_v8(dyrow + off);  // L1-cached: re-read for the next slot
            b[u] = ld_stream_v8(brow + off);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int off = seg + (lane + 32 * u) * VB;
          if (off < a.row_bytes) {
            st_v8(drow + off, scale_vec<DT>(w, g[u]));
            dot = dot_vec<DT>(g[u], b[u], dot);
          }
        }
      }
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, m);
      if (lane == 0) d_weight[i] = dot;
    }
  }
  if (!a.pads_first) zero_pad_rows<32>(a, s_beg, gw, nw);  // zero gradient, empty slots
  if (a.sys_fence) __threadfence_system();
}

// k <= 2 specialisation: dy and both expert rows of a segment are loaded
// before any arithmetic ((1 + KK) * U vectors in flight per lane), then each
// slot's scaled row is stored and its dot accumulated.  Same arithmetic
// order as k_combine_bwd (column order per lane, then the warp tree).
template <int DT, int KK, int U>
__global__ void __launch_bounds__(kRowThreads, 3) k_combine_bwd_k(RowArgs a, float* d_weight) {
  constexpr int VB = 32, SEG = 32 * U * VB;
  __shared__ int s_beg[257];
  pdl_wait();
  pdl_trigger();
  pad_prefix(a, s_beg);
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  const int nw = gridDim.x * kRowWarps;
  if (a.pads_first) zero_pad_rows<32>(a, s_beg, gw, nw);  // see RowArgs::pads_first
  for (int t = gw; t < a.S; t += nw) {
    const char* dyrow = a.src + (size_t)t * a.row_bytes;
    const char* brow[KK];
    char* drow[KK];
    float w[KK], dot[KK];
#pragma unroll
    for (int j = 0; j < KK; ++j) {
      const size_t i = (size_t)t * KK + j;
      const int s = __ldg(a.slot_idx + i);
      brow[j] = nullptr;
      drow[j] = nullptr;
      w[j] = 0.f;
      dot[j] = 0.f;
      if (s >= 0) {
        const int e = __ldg(a.expert_idx + i);
        w[j] = __ldg(a.weight + i);
        brow[j] = src_row(a, e, s);
        drow[j] = dst_row_of(a, e, s);
      }
    }
    for (int seg = 0; seg < a.row_bytes; seg += SEG) {
      V8 g[U], b[KK][U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int off = seg + (lane + 32 * u) * VB;
        if (off < a.row_bytes) g[u] = ld_stream_v8(dyrow + off);
      }
#pragma unroll
      for (int j = 0; j < KK; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int off = seg + (lane + 32 * u) * VB;
          if (brow[j] && off < a.row_bytes) b[j][u] = ld_stream_v8(brow[j] + off);
        }
#pragma unroll
      for (int j = 0; j < KK; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int off = seg + (lane + 32 * u) * VB;
          if (brow[j] && off < a.row_bytes) {
            st_v8(drow[j] + off, scale_vec<DT>(w[j], g[u]));
            dot[j] = dot_vec<DT>(g[u], b[j][u], dot[j]);
          }
        }
    }
#pragma unroll
    for (int j = 0; j < KK; ++j) {
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) dot[j] += __shfl_xor_sync(0xffffffffu, dot[j], m);
      if (lane == 0) d_weight[(size_t)t * KK + j] = brow[j] ? dot[j] : 0.f;
    }
  }
  if (!a.pads_first) zero_pad_rows<32>(a, s_beg, gw, nw);
  if (a.sys_fence) __threadfence_system();
}

// 16-byte rows (row % 32 != 0): same contract, 16-byte vectors.
template <int DT>
__global__ void __launch_bounds__(kRowThreads) k_combine_bwd16(RowArgs a, float* d_weight) {
  __shared__ int s_beg[257];
  pdl_wait();
  pdl_trigger();
  pad_prefix(a, s_beg);
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  const int nw = gridDim.x * kRowWarps;
  if (a.pads_first) zero_pad_rows<16>(a, s_beg, gw, nw);  // see RowArgs::pads_first
  for (int t = gw; t < a.S; t += nw) {
    const char* dyrow = a.src + (size_t)t * a.row_bytes;
    for (int j = 0; j < a.k; ++j) {
      const size_t i = (size_t)t * a.k + j;
      const int s = __ldg(a.slot_idx + i);
      if (s < 0) {
        if (lane == 0) d_weight[i] = 0.f;
        continue;
      }
      const int e = __ldg(a.expert_idx + i);
      const float w = __ldg(a.weight + i);
      const char* brow = src_row(a, e, s);
      char* drow = dst_row_of(a, e, s);
      float dot = 0.f;
      for (int off = lane * 16; off < a.row_bytes; off += 32 * 16) {
        const V4 g = *reinterpret_cast<const V4*>(dyrow + off);
        const V4 b = ld_stream_v4(brow + off);
        V8 g8{}, b8{};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          g8.w[q] = g.w[q];
          b8.w[q] = b.w[q];
        }
        const V8 o8 = scale_vec<DT>(w, g8);
        V4 o;
#pragma unroll
        for (int q = 0; q < 4; ++q) o.w[q] = o8.w[q];
        st_v4(drow + off, o);
        // the upper half of g8/b8 is zero: it adds exact zeros to the dot
        dot = dot_vec<DT>(g8, b8, dot);
      }
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, m);
      if (lane == 0) d_weight[i] = dot;
    }
  }
  if (!a.pads_first) zero_pad_rows<16>(a, s_beg, gw, nw);
  if (a.sys_fence) __threadfence_system();
}

moe_status_t combine_bwd_launch(const moe_gate_desc_t& d, const moe_routing_t& r, const void* dy,
                                const PeerPtrs& back, const PeerPtrs& d_back, int E_local,
                                int rank, int dtype, int dtype_size, int dcols, float* d_weight,
                                cudaStream_t stream, const int32_t* offsets,
                                const int32_t* peer_base) {
  RowArgs a{};
  a.offsets = offsets;      // packed form: no padding rows to zero
  a.peer_base = peer_base;
  a.src = static_cast<const char*>(dy);
  a.expert_idx = r.expert_idx;
  a.slot_idx = r.slot_idx;
  a.weight = r.weight;
  a.load = r.load;
  a.S = d.S;
  a.E = d.E;
  a.k = d.k;
  a.cap = d.capacity;
  a.row_bytes = dtype_size * dcols;
  a.d = dcols;
  a.speer = back;
  a.dpeer = d_back;
  a.E_local = E_local;
  a.rank = rank;
  a.sys_fence = E_local != d.E;
  // padding rows first when they are many (C4b: combine 46.2 -> 42.0 us,
  // its adjoint likewise; C3's 2% gained nothing)
  const moe_tuning_t& tu = tuning();
  a.pads_first = tu.layout_pads_first >= 0 ? tu.layout_pads_first
                                           : (E_local == d.E && pad_heavy(d) ? 1 : 0);
  const bool f = dtype == MOE_F32;
  const void* kern;
  // measured: one 1 KiB segment per round beats two (more warps in flight):
  // C2 65.5 -> 58.9 us, C3 63.5 -> 61.5, C4a 121 -> 111, C4b 73.8 -> 69.6
#define MOE_CBK(KK, UU) (f ? (const void*)k_combine_bwd_k<MOE_F32, KK, UU> : (const void*)k_combine_bwd_k<MOE_BF16, KK, UU>)
  if (a.row_bytes % 32 == 0 && a.k <= 2 && tu.combine_bwd_kspec)
    kern = a.k == 1 ? MOE_CBK(1, 1) : MOE_CBK(2, 1);
  else if (a.row_bytes % 32 == 0)
    kern = a.row_bytes >= 2048 ? (f ? (const void*)k_combine_bwd<MOE_F32, 2> : (const void*)k_combine_bwd<MOE_BF16, 2>)
                               : (f ? (const void*)k_combine_bwd<MOE_F32, 1> : (const void*)k_combine_bwd<MOE_BF16, 1>);
#undef MOE_CBK
  else
    kern = f ? (const void*)k_combine_bwd16<MOE_F32> : (const void*)k_combine_bwd16<MOE_BF16>;
  void* args[] = {&a, &d_weight};
  // persistent grid: the layout's small-CTA grid (scatter_grid) measured
  // slower here (C2 backward 97.5 -> 101.0 us, C4a 175.8 -> 183.6)
  cudaError_t e = launch_pdl(kern, dim3(row_grid(kern)), dim3(kRowThreads), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_reverse_layout_backward: launch");
  return MOE_OK;
}

// ------------------------------------------------------------ push-form combine adjoint
// The NVLink combine adjoint without reading expert outputs across the link:
// the token owner pushes dy rows (unscaled, by the dispatch kernel in peer
// mode) and the slot weights to the experts' owners; each owner scales the
// rows in place (d_expert_out = w * dy, the same exact rounding) and takes
// the dot with its LOCAL expert output row, writing the 4-byte result into
// the token owner's dw table; the token owner then picks d_weight from it.
// NVLink bytes: one row per admitted slot instead of two.
__global__ void k_scatter_w(const int32_t* expert_idx, const int32_t* slot_idx,
                            const float* weight, PeerPtrs wtab, int n, int El, int cap,
                            int rank) {
  pdl_wait();
  pdl_trigger();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int s = __ldg(slot_idx + i);
    if (s < 0) continue;
    const int e = __ldg(expert_idx + i), q = e / El;
    reinterpret_cast<float*>(wtab.p[q])[(size_t)(rank * El + e - q * El) * cap + s] = __ldg(weight + i);
  }
  __threadfence_system();
}

// Owner side: rows [P][El][cap] of dbuf hold dy (padding rows 0).
template <int DT, int U>
__global__ void __launch_bounds__(kRowThreads) k_scale_dot(char* dbuf, const char* eo,
                                                           const float* wtab, PeerPtrs dwtab,
                                                           int El, int cap, int rank,
                                                           int row_bytes, long long nrows) {
  constexpr int VB = 32, SEG = 32 * U * VB;
  const int lane = threadIdx.x & 31;
  pdl_wait();
  pdl_trigger();
  const long long nw = (long long)gridDim.x * kRowWarps;
  for (long long row = (long long)blockIdx.x * kRowWarps + (threadIdx.x >> 5); row < nrows;
       row += nw) {
    const float w = __ldg(wtab + row);
    char* g_row = dbuf + row * row_bytes;
    const char* b_row = eo + row * row_bytes;
    float dot = 0.f;
    for (int seg = 0; seg < row_bytes; seg += SEG) {
      V8 g[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int off = seg + (lane + 32 * u) * VB;
        if (off < row_bytes) {
          g[u] = ld_stream_v8(g_row + off);
          b[u] = ld_stream_v8(b_row + off);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int off = seg + (lane + 32 * u) * VB;
        if (off < row_bytes) {
          st_v8(g_row + off, scale_vec<DT>(w, g[u]));
          dot = dot_vec<DT>(g[u], b[u], dot);
        }
      }
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, m);
    if (lane == 0) {
      const long long per_src = (long long)El * cap;
      const int src = (int)(row / per_src);
      const long long rem = row - src * per_src;  // le * cap + s
      reinterpret_cast<float*>(dwtab.p[src])[(size_t)rank * per_src + rem] = dot;
    }
  }
  __threadfence_system();
}

__global__ void k_gather_dw(const int32_t* expert_idx, const int32_t* slot_idx, const float* dwtab,
                            float* d_weight, int n, int cap) {
  pdl_wait();
  pdl_trigger();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int s = __ldg(slot_idx + i);
    d_weight[i] = s >= 0 ? dwtab[(size_t)__ldg(expert_idx + i) * cap + s] : 0.f;
  }
}

moe_status_t push_bwd_launch(const moe_gate_desc_t& d, const moe_routing_t& r, const PeerPtrs& wtab,
                             const PeerPtrs& dwtab, char* dbuf_local, const char* eo_local,
                             float* d_weight, int P, int rank, int dtype, int row_bytes, int phase,
                             cudaStream_t stream) {
  const int El = d.E / P, n = d.S * d.k;
  cudaError_t e = cudaSuccess;
  if (phase == 0) {  // token side: weights to the owners
    const int grid = std::min((n + 255) / 256, device_sm_count() * 4);
    void* args[] = {(void*)&r.expert_idx, (void*)&r.slot_idx, (void*)&r.weight, (void*)&wtab,
                    (void*)&n, (void*)&El, (void*)&d.capacity, &rank};
    e = launch_pdl((const void*)k_scatter_w, dim3(std::max(1, grid)), dim3(256), 0, stream, args);
  } else if (phase == 1) {  // owner side
    const bool f = dtype == MOE_F32;
    // one 1 KiB segment per round, as k_combine_bwd_k (more warps in flight)
    const void* kern = f ? (const void*)k_scale_dot<MOE_F32, 1> : (const void*)k_scale_dot<MOE_BF16, 1>;
    long long nrows = (long long)d.E * d.capacity;
    const float* wl = reinterpret_cast<const float*>(wtab.p[rank]);
    int cap = d.capacity;
    void* args[] = {&dbuf_local, (void*)&eo_local, (void*)&wl, (void*)&dwtab, (void*)&El, &cap,
                    &rank, &row_bytes, &nrows};
    e = launch_pdl(kern, dim3(row_grid(kern)), dim3(kRowThreads), 0, stream, args);
  } else {  // token side: d_weight from the local dw table
    const int grid = std::min((n + 255) / 256, device_sm_count() * 4);
    const float* dwl = reinterpret_cast<const float*>(dwtab.p[rank]);
    int cap = d.capacity;
    void* args[] = {(void*)&r.expert_idx, (void*)&r.slot_idx, (void*)&dwl, (void*)&d_weight,
                    (void*)&n, &cap};
    e = launch_pdl((const void*)k_gather_dw, dim3(std::max(1, grid)), dim3(256), 0, stream, args);
  }
  if (e != cudaSuccess) return cuda_status(e, "moe_combine_backward_push_p2p: launch");
  return MOE_OK;
}

// ------------------------------------------------------------ gate adjoint
// L lanes per token (32/L tokens per warp in flight), each lane owning the
// experts e = l, l+L, ... (coalesced stores of the d_logits row).  With G_e =
// m_j g_j at e = e_j (0 elsewhere) and p the Eq. 1 probabilities over the
// softmax's domain:
//   d_logits[e] = p_e * (G_e - sum_{j in the domain} G_{e_j} p_{e_j}),
// i.e. sum_j m_j g_j p_j (delta(e, e_j) - p_e) (orc_gate_bwd's Jacobian sum
// regrouped); 0 outside the domain.  Domains: RENORM top-k = the k selected
// (max = l[e_0]); SOFTMAX top-k = the row (max = l[e_0]); SOFTMAX k-top-1 =
// prototype slice j (max = l[e_j]).  k-top-1 RENORM: zero.  fp64, one
// rounding.
struct GateBwdArgs {
  const float* logits;
  const int32_t* expert_idx;
  const int32_t* slot_idx;
  const float* d_weight;
  float* d_logits;
  int S, E, k, kind, mode;
  // SAM (R17): group logits [S, ngroups] and their gradient; D2S (R18):
  // uniforms [S, E] (NULL = eval) and the temperature
  const float* glogits;
  int ngroups;
  float* d_glogits;
  const float* uniforms;
  double tau;
};

constexpr int kGateBwdThreads = 256;

template <int L>
__device__ __forceinline__ double lanes_sum(double x) {
#pragma unroll
  for (int m = 1; m < L; m <<= 1) x += __shfl_xor_sync(0xffffffffu, x, m);
  return x;
}

// G_e: the (masked) weight gradient of expert e if selected, else 0
__device__ __forceinline__ double g_of(const GateBwdArgs& a, size_t t, int e) {
  const int32_t* sel = a.expert_idx + t * a.k;
  for (int j = 0; j < a.k; ++j)
    if (__ldg(sel + j) == e)
      return __ldg(a.slot_idx + t * a.k + j) >= 0 ? (double)__ldg(a.d_weight + t * a.k + j) : 0.0;
  return 0.0;
}

template <int L>
__global__ void __launch_bounds__(kGateBwdThreads) k_gate_bwd(GateBwdArgs a) {
  const int l = threadIdx.x % L;
  const int groups = gridDim.x * (kGateBwdThreads / L);
  pdl_wait();
  pdl_trigger();
  for (int base = blockIdx.x * (kGateBwdThreads / L); base < a.S; base += groups) {
    const int tt = base + threadIdx.x / L;
    const bool valid = tt < a.S;
    const size_t t = valid ? (size_t)tt : 0;
    const float* row = a.logits + t * a.E;
    float* out = a.d_logits + t * a.E;
    const int32_t* sel = a.expert_idx + t * a.k;
    const double mx0 = (double)__ldg(row + __ldg(sel));
    if (a.kind == MOE_GATE_SAM && a.mode == MOE_W_SOFTMAX) {
      // w_j = P(g) q_{e_j}, q = softmax over group g's logits (max = l[e_0]),
      // c = sum_j G_j w_j: d_l[e] = G_e w_e - q_e c on the group;
      // d_gl[h] = c (delta(h, g) - P(h))
      const int n = a.E / a.ngroups;
      const int g = valid ? __ldg(sel) / n : 0;
      const float* gl = a.glogits + t * a.ngroups;
      const double glg = (double)__ldg(gl + g);
      double pz = 0.0, pgz = 0.0;
      if (valid) {
        for (int e = g * n + l; e < (g + 1) * n; e += L) pz += exp((double)__ldg(row + e) - mx0);
        for (int h = l; h < a.ngroups; h += L) pgz += exp((double)__ldg(gl + h) - glg);
      }
      const double z = lanes_sum<L>(pz), pg = 1.0 / lanes_sum<L>(pgz);
      double c = 0.0;
      for (int j = 0; j < a.k; ++j)
        c += g_of(a, t, __ldg(sel + j)) * pg * (exp((double)__ldg(row + __ldg(sel + j)) - mx0) / z);
      if (valid) {
        for (int e = l; e < a.E; e += L) {
          double v = 0.0;
          if (e / n == g) {
            const double q = exp((double)__ldg(row + e) - mx0) / z;
            v = g_of(a, t, e) * pg * q - q * c;
          }
          out[e] = (float)v;
        }
        for (int h = l; h < a.ngroups; h += L) {
          const double ph = exp((double)__ldg(gl + h) - glg) * pg;
          a.d_glogits[t * a.ngroups + h] = (float)(c * ((h == g ? 1.0 : 0.0) - ph));
        }
      }
    } else if (a.kind == MOE_GATE_D2S) {
      // z = (l + G)/tau; domain: survivors (RENORM) or the row (SOFTMAX);
      // max over either = z of slot 0; d_l[e] = (1/tau)(G_e q_e - q_e c)
      const float* u = a.uniforms ? a.uniforms + t * a.E : nullptr;
      auto zf = [&](int e) {
        const double gn = u ? -log(-log((double)__ldg(u + e))) : 0.0;
        return ((double)__ldg(row + e) + gn) / a.tau;
      };
      const double zm = zf(valid ? __ldg(sel) : 0);
      auto in_dom = [&](int e) {
        if (a.mode == MOE_W_SOFTMAX) return true;
        for (int j = 0; j < a.k; ++j) {
          const int ej = __ldg(sel + j);
          if (ej < 0) return false;  // survivors are a prefix of the slots
          if (ej == e) return true;
        }
        return false;
      };
      double pz = 0.0;
      if (valid)
        for (int e = l; e < a.E; e += L)
          if (in_dom(e)) pz += exp(zf(e) - zm);
      const double z = lanes_sum<L>(pz);
      double c = 0.0;
      if (valid)
        for (int e = l; e < a.E; e += L) {
          const double ge = g_of(a, t, e);
          if (ge != 0.0) c += ge * (exp(zf(e) - zm) / z);
        }
      c = lanes_sum<L>(c);
      if (valid)
        for (int e = l; e < a.E; e += L) {
          double v = 0.0;
          if (in_dom(e)) {
            const double q = exp(zf(e) - zm) / z;
            v = (g_of(a, t, e) * q - q * c) / a.tau;
          }
          out[e] = (float)v;
        }
    } else if (a.kind == MOE_GATE_KTOP1 && a.mode == MOE_W_RENORM) {
      if (valid)
        for (int e = l; e < a.E; e += L) out[e] = 0.f;
    } else if (a.mode == MOE_W_RENORM && (a.kind == MOE_GATE_TOPK || a.kind == MOE_GATE_SAM)) {
      // (SAM RENORM: Eq. 1 on the k selected expert logits; no group gradient)
      if (a.kind == MOE_GATE_SAM && valid)
        for (int h = l; h < a.ngroups; h += L) a.d_glogits[t * a.ngroups + h] = 0.f;
      // domain = the k selected: every lane evaluates the k terms itself
      double z = 0.0, c = 0.0;
      for (int j = 0; j < a.k; ++j) z += exp((double)__ldg(row + __ldg(sel + j)) - mx0);
      for (int j = 0; j < a.k; ++j) {
        const size_t i = t * a.k + j;
        const double gj = __ldg(a.slot_idx + i) >= 0 ? (double)__ldg(a.d_weight + i) : 0.0;
        c += gj * (exp((double)__ldg(row + __ldg(sel + j)) - mx0) / z);
      }
      if (valid)
        for (int e = l; e < a.E; e += L) {
          double v = 0.0;
          for (int j = 0; j < a.k; ++j)
            if (__ldg(sel + j) == e) {
              const size_t i = t * a.k + j;
              const double gj = __ldg(a.slot_idx + i) >= 0 ? (double)__ldg(a.d_weight + i) : 0.0;
              v = (exp((double)__ldg(row + e) - mx0) / z) * (gj - c);
            }
          out[e] = (float)v;
        }
    } else if (a.kind == MOE_GATE_TOPK) {
      // domain = the row: the L lanes share the partition sum
      double part = 0.0;
      if (valid)
        for (int e = l; e < a.E; e += L) part += exp((double)__ldg(row + e) - mx0);
      const double z = lanes_sum<L>(part);
      double c = 0.0;
      for (int j = 0; j < a.k; ++j) {
        const size_t i = t * a.k + j;
        const double gj = __ldg(a.slot_idx + i) >= 0 ? (double)__ldg(a.d_weight + i) : 0.0;
        c += gj * (exp((double)__ldg(row + __ldg(sel + j)) - mx0) / z);
      }
      if (valid)
        for (int e = l; e < a.E; e += L) {
          const double p = exp((double)__ldg(row + e) - mx0) / z;
          out[e] = (float)(p * (g_of(a, t, e) - c));
        }
    } else {  // k-top-1 SOFTMAX: slice j = [j*n, (j+1)*n), max = l[e_j]
      const int n = a.E / a.k;
      if (valid)
        for (int e = l; e < a.E; e += L) {
          const int j = e / n;
          const size_t i = t * a.k + j;
          const double mj = (double)__ldg(row + __ldg(sel + j));
          double z = 0.0;
          for (int e2 = j * n; e2 < (j + 1) * n; ++e2) z += exp((double)__ldg(row + e2) - mj);
          const double gj = __ldg(a.slot_idx + i) >= 0 ? (double)__ldg(a.d_weight + i) : 0.0;
          const double p = exp((double)__ldg(row + e) - mj) / z;
          const double G = (__ldg(sel + j) == e) ? gj : 0.0;
          out[e] = (float)(p * (G - gj * (1.0 / z)));  // p_{e_j} = 1/z at the slice max
        }
    }
  }
}

moe_status_t gate_bwd_launch(const moe_gate_desc_t& d, const moe_gate_inputs_t& in,
                             const moe_routing_t& r, const float* d_weight, float* d_logits,
                             float* d_group_logits, cudaStream_t stream) {
  GateBwdArgs a{in.logits, r.expert_idx, r.slot_idx, d_weight, d_logits, d.S, d.E, d.k, d.kind,
                d.weight_mode, in.group_logits, d.kind == MOE_GATE_SAM ? in.n_groups : 1,
                d_group_logits, in.uniforms, in.tau};
  // lanes per token (tuning gate_bwd_lanes overrides)
  int L = tuning().gate_bwd_lanes;
  if (L <= 0) {
    L = 1;  // ~8 experts per lane (one per lane measured slower at E = 8)
    while (L < 32 && d.E / (L * 2) >= 8) L *= 2;
  }
  const void* kern = L == 1 ? (const void*)k_gate_bwd<1> : L == 2 ? (const void*)k_gate_bwd<2>
                     : L == 4 ? (const void*)k_gate_bwd<4> : L == 8 ? (const void*)k_gate_bwd<8>
                     : L == 16 ? (const void*)k_gate_bwd<16> : (const void*)k_gate_bwd<32>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGateBwdThreads, 0);
  const int tokens_per_cta = kGateBwdThreads / L;
  const int need = (d.S + tokens_per_cta - 1) / tokens_per_cta;
  const int grid = std::min(need, std::max(1, per_sm) * device_sm_count());
  void* args[] = {&a};
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(kGateBwdThreads), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_gate_backward: launch");
  return MOE_OK;
}

}  // namespace moe
