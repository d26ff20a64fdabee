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
#include "rows.cuh"

namespace moe {

template <int DT>
__device__ __forceinline__ V8 scale_vec(float w, const V8& v) {
  V8 o;
  if constexpr (DT == MOE_F32) {
#pragma unroll
    for (int q = 0; q < 8; ++q) o.w[q] = __float_as_uint(__fmul_rn(w, __uint_as_float(v.w[q])));
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      // w (24 bits) x bf16 (8 bits) is exact in fp64; one RNE to bf16
      const __nv_bfloat16 lo = __double2bfloat16((double)w * (double)bf16lo(v.w[q]));
      const __nv_bfloat16 hi = __double2bfloat16((double)w * (double)bf16hi(v.w[q]));
      o.w[q] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
    }
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
  // zero gradient for the padding (empty) slots
  const int npad = s_beg[a.E];
  const V8 z = V8{{0, 0, 0, 0, 0, 0, 0, 0}};
  for (int p = gw; p < npad; p += nw) {
    int lo = 0, hi = a.E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_beg[mid] <= p) lo = mid; else hi = mid - 1;
    }
    char* drow = dst_row_of(a, lo, min(__ldg(a.load + lo), a.cap) + (p - s_beg[lo]));
    for (int off = lane * VB; off < a.row_bytes; off += 32 * VB) st_v8(drow + off, z);
  }
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
  const int npad = s_beg[a.E];
  for (int p = gw; p < npad; p += nw) {
    int lo = 0, hi = a.E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_beg[mid] <= p) lo = mid; else hi = mid - 1;
    }
    char* drow = dst_row_of(a, lo, min(__ldg(a.load + lo), a.cap) + (p - s_beg[lo]));
    for (int off = lane * 16; off < a.row_bytes; off += 32 * 16) st_v4(drow + off, V4{{0, 0, 0, 0}});
  }
  if (a.sys_fence) __threadfence_system();
}

moe_status_t combine_bwd_launch(const moe_gate_desc_t& d, const moe_routing_t& r, const void* dy,
                                const PeerPtrs& back, const PeerPtrs& d_back, int E_local,
                                int rank, int dtype, int dtype_size, int dcols, float* d_weight,
                                cudaStream_t stream) {
  RowArgs a{};
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
  const bool f = dtype == MOE_F32;
  const void* kern;
  if (a.row_bytes % 32 == 0)
    kern = a.row_bytes >= 2048 ? (f ? (const void*)k_combine_bwd<MOE_F32, 2> : (const void*)k_combine_bwd<MOE_BF16, 2>)
                               : (f ? (const void*)k_combine_bwd<MOE_F32, 1> : (const void*)k_combine_bwd<MOE_BF16, 1>);
  else
    kern = f ? (const void*)k_combine_bwd16<MOE_F32> : (const void*)k_combine_bwd16<MOE_BF16>;
  void* args[] = {&a, &d_weight};
  cudaError_t e = launch_pdl(kern, dim3(row_grid(kern)), dim3(kRowThreads), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_reverse_layout_backward: launch");
  return MOE_OK;
}

// ------------------------------------------------------------ gate adjoint
// One warp per token.  With G_e = m_j g_j at e = e_j (0 elsewhere) and p the
// Eq. 1 probabilities over the softmax's domain:
//   d_logits[e] = p_e * (G_e - sum_{j in the domain} G_{e_j} p_{e_j}),
// i.e. sum_j m_j g_j p_j (delta(e, e_j) - p_e) (orc_gate_bwd's Jacobian sum
// regrouped); 0 outside the domain.  Domains: RENORM top-k = the k selected
// (max = l[e_0]); SOFTMAX top-k = the row (max = l[e_0]); SOFTMAX k-top-1 =
// prototype slice j (max = l[e_j]).  k-top-1 RENORM: zero.
struct GateBwdArgs {
  const float* logits;
  const int32_t* expert_idx;
  const int32_t* slot_idx;
  const float* d_weight;
  float* d_logits;
  int S, E, k, kind, mode;
};

constexpr int kGateBwdWarps = 4;

__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) x += __shfl_xor_sync(0xffffffffu, x, m);
  return x;
}

__global__ void __launch_bounds__(kGateBwdWarps * 32) k_gate_bwd(GateBwdArgs a) {
  __shared__ double s_G[kGateBwdWarps][256];  // G_e of this warp's token
  __shared__ double s_c[kGateBwdWarps][512];  // k-top-1: per slice (z_j, G_{e_j} p_{e_j})
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();
  pdl_trigger();
  double* G = s_G[warp];
  double* C = s_c[warp];
  for (int t = blockIdx.x * kGateBwdWarps + warp; t < a.S; t += gridDim.x * kGateBwdWarps) {
    const float* row = a.logits + (size_t)t * a.E;
    float* out = a.d_logits + (size_t)t * a.E;
    const int32_t* sel = a.expert_idx + (size_t)t * a.k;
    if (a.kind == MOE_GATE_KTOP1 && a.mode == MOE_W_RENORM) {
      for (int e = lane; e < a.E; e += 32) out[e] = 0.f;
      continue;
    }
    for (int e = lane; e < a.E; e += 32) G[e] = 0.0;
    __syncwarp();
    for (int j = lane; j < a.k; j += 32) {
      const size_t i = (size_t)t * a.k + j;
      G[sel[j]] = __ldg(a.slot_idx + i) >= 0 ? (double)__ldg(a.d_weight + i) : 0.0;
    }
    __syncwarp();
    if (a.kind == MOE_GATE_TOPK && a.mode == MOE_W_RENORM) {
      const double mx = (double)__ldg(row + sel[0]);
      double z = 0.0;
      for (int j = lane; j < a.k; j += 32) z += exp((double)__ldg(row + sel[j]) - mx);
      z = warp_sum_d(z);
      double c = 0.0;
      for (int j = lane; j < a.k; j += 32) c += G[sel[j]] * (exp((double)__ldg(row + sel[j]) - mx) / z);
      c = warp_sum_d(c);
      for (int e = lane; e < a.E; e += 32) out[e] = 0.f;
      __syncwarp();
      for (int j = lane; j < a.k; j += 32) {
        const int e = sel[j];
        const double p = exp((double)__ldg(row + e) - mx) / z;
        out[e] = (float)(p * (G[e] - c));
      }
    } else if (a.kind == MOE_GATE_TOPK) {
      const double mx = (double)__ldg(row + sel[0]);
      double z = 0.0;
      for (int e = lane; e < a.E; e += 32) z += exp((double)__ldg(row + e) - mx);
      z = warp_sum_d(z);
      double c = 0.0;
      for (int j = lane; j < a.k; j += 32) c += G[sel[j]] * (exp((double)__ldg(row + sel[j]) - mx) / z);
      c = warp_sum_d(c);
      for (int e = lane; e < a.E; e += 32) {
        const double p = exp((double)__ldg(row + e) - mx) / z;
        out[e] = (float)(p * (G[e] - c));
      }
    } else {  // k-top-1 SOFTMAX: slice j = experts [j*n, (j+1)*n), max = l[e_j]
      const int n = a.E / a.k;
      for (int j = lane; j < a.k; j += 32) {
        const double mx = (double)__ldg(row + sel[j]);
        double z = 0.0;
        for (int e = j * n; e < (j + 1) * n; ++e) z += exp((double)__ldg(row + e) - mx);
        C[2 * j] = z;
        C[2 * j + 1] = G[sel[j]] * (1.0 / z);  // G_{e_j} p_{e_j}: p at the slice max = 1/z
      }
      __syncwarp();
      for (int e = lane; e < a.E; e += 32) {
        const int j = e / n;
        const double p = exp((double)__ldg(row + e) - (double)__ldg(row + sel[j])) / C[2 * j];
        out[e] = (float)(p * (G[e] - C[2 * j + 1]));
      }
    }
    __syncwarp();
  }
}

moe_status_t gate_bwd_launch(const moe_gate_desc_t& d, const float* logits, const moe_routing_t& r,
                             const float* d_weight, float* d_logits, cudaStream_t stream) {
  GateBwdArgs a{logits, r.expert_idx, r.slot_idx, d_weight, d_logits, d.S, d.E, d.k, d.kind,
                d.weight_mode};
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_gate_bwd,
                                                kGateBwdWarps * 32, 0);
  const int need = (d.S + kGateBwdWarps - 1) / kGateBwdWarps;
  const int grid = std::min(need, std::max(1, per_sm) * device_sm_count());
  void* args[] = {&a};
  cudaError_t e = launch_pdl((const void*)k_gate_bwd, dim3(grid), dim3(kGateBwdWarps * 32), 0,
                             stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_gate_backward: launch");
  return MOE_OK;
}

}  // namespace moe
