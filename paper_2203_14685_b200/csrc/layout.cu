// layout.cu -- moe_layout (Alg. 1 step 2),
// moe_reverse_layout (step 6 + the weighted combine of step 4,
// PAPER.md:56-59, 64-65), the bench expert stand-in (R16) and the chunk
// permutation used by the hierarchical AllToAll.
//
// All four are HBM-bound row movers.  Design:
//  - persistent grid (SMs x resident CTAs), one warp per row task;
//  - 32-byte vector loads/stores (LDG/STG.E.256) when the row is a multiple
//    of 32 bytes, else 16-byte; streaming loads bypass L1 and are marked
//    evict-first in L2;
//  - layout is token-centric: each x row is read ONCE and written to its <= k
//    admitted slots; the zero-fill of the padding rows is appended to the same
//    launch as extra row tasks (no separate memset);
//  - reverse is token-centric: <= k row loads, fp32 FMA in ascending j from
//    0, one RNE store; fully dropped tokens store zeros.
#include <algorithm>

#include "launch.cuh"
#include "rows.cuh"

namespace moe {

// ------------------------------------------------------------ Layout_Transform
template <int VB, int U>
__global__ void __launch_bounds__(kRowThreads) k_layout(RowArgs a) {
  using V = Vec<VB>;
  __shared__ int s_beg[257];
  row_trace(a, 0);
  pdl_wait();     // routing comes from moe_gate
  pdl_trigger();
  row_trace(a, 1);
  pad_prefix(a, s_beg);
  const int lane = threadIdx.x & 31;
  const long long npad = s_beg[a.E];
  const long long n_tasks = (long long)a.S + npad;
  const long long wstride = (long long)gridDim.x * kRowWarps;
  constexpr int SEG = 32 * U * VB;  // bytes one warp moves per segment
  for (long long task0 = (long long)blockIdx.x * kRowWarps + (threadIdx.x >> 5); task0 < n_tasks;
       task0 += wstride) {
    // task order: tokens then padding rows, or padding rows first
    const long long task = !a.pads_first ? task0 : task0 < npad ? a.S + task0 : task0 - npad;
    if (task < a.S) {
      const int t = (int)task;
      const char* srow = a.src + (size_t)t * a.row_bytes;
      for (int seg = 0; seg < a.row_bytes; seg += SEG) {
        typename V::T r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int off = seg + (lane + 32 * u) * VB;
          if (off < a.row_bytes) r[u] = V::ld_stream(srow + off);
        }
        for (int j = 0; j < a.k; ++j) {
          const int s = __ldg(a.slot_idx + (size_t)t * a.k + j);
          if (s < 0) continue;
          const int e = __ldg(a.expert_idx + (size_t)t * a.k + j);
          if (j > 0 && dedupe_row(a, t, j, e, s, seg == 0 ? lane : 1)) continue;
          char* drow = dst_row_of(a, e, s);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int off = seg + (lane + 32 * u) * VB;
            if (off < a.row_bytes) V::st(drow + off, r[u]);
          }
        }
      }
    } else {
      // padding row: binary search its expert in the prefix
      const int p = (int)(task - a.S);
      int lo = 0, hi = a.E - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_beg[mid] <= p) lo = mid; else hi = mid - 1;
      }
      char* drow = dst_row_of(a, lo, min(__ldg(a.load + lo), a.cap) + (p - s_beg[lo]));
      const typename V::T z = V::zero();
      for (int off = lane * VB; off < a.row_bytes; off += 32 * VB) V::st(drow + off, z);
    }
  }
  if (a.sys_fence) __threadfence_system();
  row_trace_end(a);
}

// ------------------------------------------------------------ Reverse + combine
template <int DT, int U>
__global__ void __launch_bounds__(kRowThreads) k_reverse(RowArgs a) {
  constexpr int VB = 32;
  constexpr int NA = DT == MOE_F32 ? 8 : 16;  // accumulators per vector
  constexpr int SEG = 32 * U * VB;
  const int lane = threadIdx.x & 31;
  const int wstride = gridDim.x * kRowWarps;
  row_trace(a, 0);
  pdl_wait();     // expert outputs come from the AllToAll / the layout
  pdl_trigger();
  row_trace(a, 1);
  for (int tl = blockIdx.x * kRowWarps + (threadIdx.x >> 5); tl < a.S; tl += wstride) {
    const int t = a.rev ? a.S - 1 - tl : tl;  // rev: last tokens first (L2 reuse)
    char* yrow = a.dst + (size_t)t * a.row_bytes;
    for (int seg = 0; seg < a.row_bytes; seg += SEG) {
      float acc[U][NA];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < NA; ++q) acc[u][q] = 0.f;
      for (int j = 0; j < a.k; j += 2) {
        // two slots per round so both rows' loads are in flight together
        int s0 = __ldg(a.slot_idx + (size_t)t * a.k + j);
        int s1 = j + 1 < a.k ? __ldg(a.slot_idx + (size_t)t * a.k + j + 1) : -1;
        V8 r0[U], r1[U];
        float w0 = 0.f, w1 = 0.f;
        if (s0 >= 0) {
          const int e = __ldg(a.expert_idx + (size_t)t * a.k + j);
          w0 = row_weight(a, (size_t)t * a.k + j);
          const char* b = src_row_item(a, t, j, e, s0);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int off = seg + (lane + 32 * u) * VB;
            if (off < a.row_bytes) r0[u] = ld_stream_v8(b + off);
          }
        }
        if (s1 >= 0) {
          const int e = __ldg(a.expert_idx + (size_t)t * a.k + j + 1);
          w1 = row_weight(a, (size_t)t * a.k + j + 1);
          const char* b = src_row_item(a, t, j + 1, e, s1);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int off = seg + (lane + 32 * u) * VB;
            if (off < a.row_bytes) r1[u] = ld_stream_v8(b + off);
          }
        }
        if (s0 >= 0) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (seg + (lane + 32 * u) * VB < a.row_bytes) fma_vec<DT>(acc[u], w0, r0[u]);
        }
        if (s1 >= 0) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (seg + (lane + 32 * u) * VB < a.row_bytes) fma_vec<DT>(acc[u], w1, r1[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int off = seg + (lane + 32 * u) * VB;
        if (off < a.row_bytes) {
          if (a.y_ef) st_v8_ef(yrow + off, pack_vec<DT>(acc[u]));
          else st_v8(yrow + off, pack_vec<DT>(acc[u]));
        }
      }
    }
  }
  row_trace_end(a);
}

// k <= 2 specialisation: every load of a U-vector segment of the KK rows of
// TPW consecutive tokens is issued before the first FMA (TPW*KK*U*32 bytes in
// flight per lane; the host picks TPW*KK*U = 4), and each output vector is
// finished and stored straight away, so the accumulators cost 16 registers
// instead of U*16.  Switch (k = 1) on 4 KiB rows: U = 4; on 2 KiB rows:
// U = 2, TPW = 2.  Same arithmetic order as k_reverse: fp32 FMA from 0 in
// ascending j, one RNE store.
// AL (k = 2, alias-mode NVLink combine only): a token's two slots may name
// the same row, which is then loaded once.
template <int DT, int KK, int U, int TPW, bool AL = false>
__global__ void __launch_bounds__(kRowThreads) k_reverse_k(RowArgs a) {
  constexpr int VB = 32;
  constexpr int NA = DT == MOE_F32 ? 8 : 16;
  constexpr int SEG = 32 * U * VB;
  const int lane = threadIdx.x & 31;
  const int wstride = gridDim.x * kRowWarps * TPW;
  row_trace(a, 0);
  pdl_wait();
  pdl_trigger();
  row_trace(a, 1);
  for (int tb = (blockIdx.x * kRowWarps + (threadIdx.x >> 5)) * TPW; tb < a.S; tb += wstride) {
    const char* b[TPW][KK];
    float w[TPW][KK];
    // pre-combined pairs (RowArgs::pre, k = 2 only): both admitted slots on
    // one remote owner -> that owner already computed the token's y row
    // (same fp32 FMA order, one rounding) into its pre row of the second
    // slot: one read, stored as is
    bool pc[TPW];
#pragma unroll
    for (int p = 0; p < TPW; ++p) {
      pc[p] = false;
      int e_first = 0, s_first = -1;
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        const int tl = tb + p;
        const int t = a.rev ? a.S - 1 - tl : tl;
        const int s = tl < a.S ? __ldg(a.slot_idx + (size_t)t * KK + j) : -1;
        b[p][j] = nullptr;
        w[p][j] = 0.f;
        if (s >= 0) {
          const int e = __ldg(a.expert_idx + (size_t)t * KK + j);
          b[p][j] = AL ? src_row_item(a, t, j, e, s) : src_row(a, e, s);
          w[p][j] = row_weight(a, (size_t)t * KK + j);
          if constexpr (KK == 2 && !AL) {
            if (j == 0) {
              e_first = e;
              s_first = s;
            } else if (a.pre.p[0] && s_first >= 0) {
              const int q = e / a.E_local;
              if (q == e_first / a.E_local && q != a.rank) {
                pc[p] = true;
                b[p][0] = a.pre.p[q] + row_index(a, q, e, s) * a.row_bytes;
                b[p][1] = nullptr;
              }
            }
          }
        }
      }
    }
    // alias-mode combine (src_row_item): both slots of a token may name the
    // same row (sent once by the deduped dispatch); it is loaded once
    bool dup1[TPW];
#pragma unroll
    for (int p = 0; p < TPW; ++p) dup1[p] = AL && KK == 2 && b[p][KK - 1] == b[p][0];
    for (int seg = 0; seg < a.row_bytes; seg += SEG) {
      V8 r[TPW][KK][U];
#pragma unroll
      for (int p = 0; p < TPW; ++p)
#pragma unroll
        for (int j = 0; j < KK; ++j)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int off = seg + (lane + 32 * u) * VB;
            if (b[p][j] && off < a.row_bytes && !(j == 1 && dup1[p]))
              r[p][j][u] = ld_stream_v8(b[p][j] + off);
          }
      if constexpr (AL) {
#pragma unroll
        for (int p = 0; p < TPW; ++p)
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < 8; ++q)
              r[p][KK - 1][u].w[q] = dup1[p] ? r[p][0][u].w[q] : r[p][KK - 1][u].w[q];
      }
#pragma unroll
      for (int p = 0; p < TPW; ++p) {
        if (tb + p >= a.S) break;
        char* yrow = a.dst + (size_t)(a.rev ? a.S - 1 - (tb + p) : tb + p) * a.row_bytes;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int off = seg + (lane + 32 * u) * VB;
          if (off < a.row_bytes) {
            float acc[NA];
#pragma unroll
            for (int q = 0; q < NA; ++q) acc[q] = 0.f;
#pragma unroll
            for (int j = 0; j < KK; ++j)
              if (b[p][j]) fma_vec<DT>(acc, w[p][j], r[p][j][u]);
            if constexpr (KK == 2 && !AL) {
              const V8 o = pc[p] ? r[p][0][u] : pack_vec<DT>(acc);
              if (a.y_ef) st_v8_ef(yrow + off, o);
              else st_v8(yrow + off, o);
            } else {
              if (a.y_ef) st_v8_ef(yrow + off, pack_vec<DT>(acc));
              else st_v8(yrow + off, pack_vec<DT>(acc));
            }
          }
        }
      }
    }
  }
  row_trace_end(a);
}

// 16-byte fallback of the combine for rows that are not a multiple of 32 B.
template <int DT>
__global__ void __launch_bounds__(kRowThreads) k_reverse16(RowArgs a) {
  const int lane = threadIdx.x & 31;
  const int wstride = gridDim.x * kRowWarps;
  constexpr int NA = DT == MOE_F32 ? 4 : 8;
  row_trace(a, 0);
  pdl_wait();
  pdl_trigger();
  row_trace(a, 1);
  for (int tl = blockIdx.x * kRowWarps + (threadIdx.x >> 5); tl < a.S; tl += wstride) {
    const int t = a.rev ? a.S - 1 - tl : tl;
    char* yrow = a.dst + (size_t)t * a.row_bytes;
    for (int off = lane * 16; off < a.row_bytes; off += 32 * 16) {
      float acc[NA];
#pragma unroll
      for (int q = 0; q < NA; ++q) acc[q] = 0.f;
      for (int j = 0; j < a.k; ++j) {
        const int s = __ldg(a.slot_idx + (size_t)t * a.k + j);
        if (s < 0) continue;
        const int e = __ldg(a.expert_idx + (size_t)t * a.k + j);
        const float w = row_weight(a, (size_t)t * a.k + j);
        const V4 v = ld_stream_v4(src_row_item(a, t, j, e, s) + off);
        if constexpr (DT == MOE_F32) {
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] = fmaf(w, __uint_as_float(v.w[q]), acc[q]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[2 * q] = fmaf(w, bf16lo(v.w[q]), acc[2 * q]);
            acc[2 * q + 1] = fmaf(w, bf16hi(v.w[q]), acc[2 * q + 1]);
          }
        }
      }
      V4 o;
      if constexpr (DT == MOE_F32) {
#pragma unroll
        for (int q = 0; q < 4; ++q) o.w[q] = __float_as_uint(acc[q]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) o.w[q] = pack_bf16x2(acc[2 * q], acc[2 * q + 1]);
      }
      st_v4(yrow + off, o);
    }
  }
  row_trace_end(a);
}

// ------------------------------------------------------------ expert stand-in
// One warp per row of [nsrc][E_local][cap] rows; s_e = 1 + (e mod 8)/8 is
// exact, and one fp32 multiply of a bf16 (or fp32) value rounds once.
template <int DT>
__global__ void __launch_bounds__(kRowThreads) k_expert_scale(const char* in, char* out,
                                                              long long n_rows, int row_bytes,
                                                              int cap, int E_local, int e_base) {
  const int lane = threadIdx.x & 31;
  const long long wstride = (long long)gridDim.x * kRowWarps;
  for (long long row = (long long)blockIdx.x * kRowWarps + (threadIdx.x >> 5); row < n_rows;
       row += wstride) {
    const int le = (int)((row / cap) % E_local);
    const float s = 1.0f + (float)((e_base + le) % 8) * 0.125f;  // exact
    const char* src = in + row * row_bytes;
    char* dst = out + row * row_bytes;
    for (int off = lane * 16; off < row_bytes; off += 32 * 16) {
      V4 x = ld_stream_v4(src + off);
      V4 o;
      if constexpr (DT == MOE_F32) {
#pragma unroll
        for (int q = 0; q < 4; ++q) o.w[q] = __float_as_uint(__fmul_rn(__uint_as_float(x.w[q]), s));
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          o.w[q] = pack_bf16x2(__fmul_rn(bf16lo(x.w[q]), s), __fmul_rn(bf16hi(x.w[q]), s));
      }
      st_v4(dst + off, o);
    }
  }
}

// ------------------------------------------------------------ chunk permute
// dst chunk (n, g, m) <- src chunk (g, m, n) for n, m < G and g < N:
// phase (4) of the hierarchical AllToAll, "reorder by destination device".
__global__ void __launch_bounds__(kRowThreads) k_chunk_permute(const char* src, char* dst, int N,
                                                               int G, long long chunk_bytes) {
  const long long vecs = chunk_bytes / 16;
  const long long total = (long long)N * G * G * vecs;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const long long c = i / vecs, v = i % vecs;  // c = destination chunk (n, g, m)
    const int m = (int)(c % G);
    const int g = (int)((c / G) % N);
    const int n = (int)(c / ((long long)G * N));
    const long long sc = ((long long)g * G + m) * G + n;
    st_v4(dst + c * chunk_bytes + v * 16, ld_stream_v4(src + sc * chunk_bytes + v * 16));
  }
}

// dst chunk [y][x] <- src chunk [x][y] for x < X, y < Y: the two local
// reorders of the two-level hierarchical AllToAll (HIER_2D).
__global__ void __launch_bounds__(kRowThreads) k_chunk_transpose(const char* src, char* dst, int X,
                                                                 int Y, long long chunk_bytes) {
  const long long vecs = chunk_bytes / 16;
  const long long total = (long long)X * Y * vecs;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const long long c = i / vecs, v = i % vecs;  // c = destination chunk (y, x)
    const long long y = c / X, x = c % X;
    st_v4(dst + c * chunk_bytes + v * 16, ld_stream_v4(src + (x * Y + y) * chunk_bytes + v * 16));
  }
}

// ------------------------------------------------------------ expert offsets
// Dropless packed form (NEXT-4; SPEC.md:241-245 Permutation.expert_offsets):
// offsets[e] = sum_{e' < e} min(load[e'], cap), one CTA, warp scan (E <= 256).
__global__ void __launch_bounds__(32) k_expert_offsets(const int32_t* load, int E, int cap,
                                                       int32_t* offsets) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x;
  int carry = 0;
  if (lane == 0) offsets[0] = 0;
  for (int base = 0; base < E; base += 32) {
    const int e = base + lane;
    const int v = e < E ? min(__ldg(load + e), cap) : 0;
    int incl = v;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, incl, m);
      if (lane >= m) incl += o;
    }
    if (e < E) offsets[e + 1] = carry + incl;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
}

moe_status_t expert_offsets_launch(const int32_t* load, int E, int cap, int32_t* offsets,
                                   cudaStream_t stream) {
  void* args[] = {(void*)&load, &E, &cap, &offsets};
  cudaError_t e = launch_pdl((const void*)k_expert_offsets, dim3(1), dim3(32), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_expert_offsets: launch");
  return MOE_OK;
}

// ------------------------------------------------------------ host side

// moe_set_trace: the row kernels' per-CTA stamps go to the trace buffer's
// second half (layout, dispatch) and last quarter (reverse, combine)
static void row_trace_set(RowArgs& a, bool reverse) {
  if (!g_trace.buf) return;
  const long long n = (long long)(g_trace.bytes / sizeof(unsigned long long));
  a.trace = static_cast<unsigned long long*>(g_trace.buf) + (reverse ? 3 * n / 4 : n / 2);
  a.trace_n = n / 4;
}

moe_status_t layout_launch_peers(const moe_gate_desc_t& d, const moe_routing_t& r, const void* x,
                                 int dtype_size, int dcols, const PeerPtrs& dst, int E_local,
                                 int rank, cudaStream_t stream, const int32_t* offsets,
                                 const int32_t* peer_base, const PeerPtrs* pad_tab,
                                 const PeerPtrs* dup_tab, const PeerPtrs* wt_tab) {
  RowArgs a{};
  row_trace_set(a, false);
  if (dup_tab && !offsets) {
    a.dedupe = 1;
    a.dup = *dup_tab;
    if (wt_tab) a.wt = *wt_tab;
  }
  if (pad_tab) {
    a.skip_pads = 1;
    a.ptab = *pad_tab;
  }
  a.offsets = offsets;
  a.peer_base = peer_base;
  a.src = static_cast<const char*>(x);
  a.expert_idx = r.expert_idx;
  a.slot_idx = r.slot_idx;
  a.weight = r.weight;  // read only by the dedupe's slot-weight stores
  a.load = r.load;
  a.S = d.S;
  a.E = d.E;
  a.k = d.k;
  a.cap = d.capacity;
  a.row_bytes = dtype_size * dcols;
  a.d = dcols;
  a.dpeer = dst;
  a.E_local = E_local;
  a.rank = rank;
  a.sys_fence = E_local != d.E;
  // padding rows first when they are many (C4b: combine 46.2 -> 42.0 us,
  // its adjoint likewise; C3's 2% gained nothing)
  const moe_tuning_t& tu = tuning();
  a.pads_first = tu.layout_pads_first >= 0 ? tu.layout_pads_first
                                           : (E_local == d.E && pad_heavy(d) ? 1 : 0);
  // Measured alternatives, removed: a TMA bulk-copy pipeline (slower into
  // local HBM and over NVLink: C2 at P=2 121.2 vs 117.5 us), two tokens per
  // warp (no gain), an L2 prefetch of x before the PDL wait (C2 +3 us).
  const void* kern;
  if (a.row_bytes % 32 == 0) {
    // measured: 2 KiB segments for rows <= 2 KiB (C2 36.3 -> 35.4 us)
    const int lu = tu.layout_u > 0 ? tu.layout_u : (a.row_bytes <= 2048 ? 2 : 4);
    kern = lu == 1 ? (const void*)k_layout<32, 1> : lu == 2 ? (const void*)k_layout<32, 2>
                                                            : (const void*)k_layout<32, 4>;
  } else {
    kern = (const void*)k_layout<16, 4>;
  }
  // Local layout: a grid of ~2 tokens per warp, not the persistent one.  The
  // persistent grid's CTAs end up to 15 us apart at C2 (moe_set_trace: some
  // SMs get less of the write bandwidth), an idle tail the block scheduler
  // removes when it hands out small CTAs as SMs free up (measured: C2 layout
  // 37.0 -> 34.9 us, C3 44.6 -> 43.0, C4a 70.4 -> 66.1, C4b 52.1 -> 50.0;
  // the reverse, whose reversed walk reuses L2, measured slower that way and
  // stays persistent).  The one-sided dispatch (stores to peers, a system
  // fence per CTA) keeps the persistent grid: measured slower on 2 GPUs with
  // the small-CTA grid (C2 step 249.3 -> 257.0 us; 1 token per warp 271.4).
  const int grid = scatter_grid(kern, d.S, a.sys_fence);
  void* args[] = {&a};
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(kRowThreads), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_layout: k_layout launch");
  return MOE_OK;
}

moe_status_t layout_launch(const moe_gate_desc_t& d, const moe_routing_t& r, const void* x,
                           int dtype_size, int dcols, void* dispatch, cudaStream_t stream,
                           const int32_t* offsets) {
  PeerPtrs dst{};
  dst.p[0] = static_cast<char*>(dispatch);
  return layout_launch_peers(d, r, x, dtype_size, dcols, dst, d.E, 0, stream, offsets, nullptr);
}

moe_status_t reverse_launch_peers(const moe_gate_desc_t& d, const moe_routing_t& r,
                                  const PeerPtrs& src, int E_local, int rank, int dtype,
                                  int dtype_size, int dcols, void* y, cudaStream_t stream,
                                  const int32_t* offsets, const int32_t* peer_base,
                                  int dup_alias, const PeerPtrs* pre) {
  RowArgs a{};
  if (pre) a.pre = *pre;
  row_trace_set(a, true);
  a.dedupe = dup_alias;  // reverse: read deduped slots from their first row (src_row_item)
  a.offsets = offsets;
  a.peer_base = peer_base;
  a.dst = static_cast<char*>(y);
  // Local mode walks the tokens last to first: the expert (or the layout)
  // wrote the rows of the LAST tokens last -- slots follow token order in
  // every expert -- so those are the rows still in L2; y is stored
  // evict-first so it does not push them out.  Measured at N=1: C2 reverse
  // 36.0 -> 31.6 us, C4a 72.2 -> 64.7 us.  Over NVLink the rows live in the
  // peers' L2s and the order does not help (C2 at N=2: 252 -> 255 us).
  const moe_tuning_t& tu = tuning();
  const int local_dflt = E_local == d.E ? 1 : 0;
  a.rev = tu.reverse_backwards >= 0 ? tu.reverse_backwards : local_dflt;
  a.y_ef = tu.reverse_y_ef >= 0 ? tu.reverse_y_ef : local_dflt;
  a.expert_idx = r.expert_idx;
  a.slot_idx = r.slot_idx;
  a.weight = r.weight;
  a.S = d.S;
  a.E = d.E;
  a.k = d.k;
  a.cap = d.capacity;
  a.row_bytes = dtype_size * dcols;
  a.d = dcols;
  a.speer = src;
  a.E_local = E_local;
  a.rank = rank;
  // Measured alternatives, removed: a TMA-staged combine (won for Switch on
  // >= 4 KiB rows only in the forward walk; the reversed register walk is
  // faster, C3 40.0 vs 52.3 us), 16-byte vectors, two segments per round; a
  // small-CTA grid (as the layout's) with blocks of 2-8 consecutive tokens
  // per warp (C2 step 70.2 -> 71.2 us, C3 89.7 -> 90.6, C4b 94.9 -> 95.0,
  // C4a 139.0 -> 138.6; profiles/r02_n1_grid/ab_rev_blocked.txt).
  const void* kern;
  // k <= 2 path: vectors per lane per round (x k rows); measured: 2 for
  // k = 2 (one 1 KiB segment of both rows: C2 36.3 -> 35.6 us), 4 for k = 1
  // (peer mode: 4 -- both 2 KiB rows in flight hide the NVLink latency better,
  // C2 at P=2: 129.2 -> 127.3 us)
  const int KU = tu.reverse_ku > 0 ? tu.reverse_ku : (d.k == 2 && E_local == d.E) ? 2 : 4;
  const bool kspec = reverse_kspec_used(d, a.row_bytes);
  if (kspec) {
    // TPW * k * U = KU vectors in flight per lane, U covering at most one
    // row (1 KiB of row per U step)
    const bool f = dtype == MOE_F32;
    const int segs = std::max(1, a.row_bytes / 1024);  // 1 KiB per U step
    const int per = std::max(1, KU / a.k);                // U * TPW
    const int Uc = std::min(per, segs) >= 4 ? 4 : std::min(per, segs) >= 2 ? 2 : 1;
    // two tokens per warp round for Switch on <= 2 KiB rows (C4b: 51.3 vs
    // 53.5 us); no gain for k = 2
    const int tpw = tu.reverse_tpw >= 0 ? tu.reverse_tpw : (a.k == 1 && a.row_bytes <= 2048);
    const int T = tpw ? std::max(1, per / Uc) : 1;
#define MOE_RK(KK, UU, TT) (f ? (const void*)k_reverse_k<MOE_F32, KK, UU, TT> : (const void*)k_reverse_k<MOE_BF16, KK, UU, TT>)
    if (a.k == 1)
      kern = Uc == 4 ? (T >= 2 ? MOE_RK(1, 4, 2) : MOE_RK(1, 4, 1))
             : Uc == 2 ? (T >= 4 ? MOE_RK(1, 2, 4) : T >= 2 ? MOE_RK(1, 2, 2) : MOE_RK(1, 2, 1))
                       : (T >= 4 ? MOE_RK(1, 1, 4) : T >= 2 ? MOE_RK(1, 1, 2) : MOE_RK(1, 1, 1));
    else if (a.dedupe)  // alias-mode NVLink combine
      kern = Uc >= 2 ? (f ? (const void*)k_reverse_k<MOE_F32, 2, 2, 1, true>
                          : (const void*)k_reverse_k<MOE_BF16, 2, 2, 1, true>)
                     : (f ? (const void*)k_reverse_k<MOE_F32, 2, 1, 1, true>
                          : (const void*)k_reverse_k<MOE_BF16, 2, 1, 1, true>);
    else
      kern = Uc >= 2 ? (T >= 2 ? MOE_RK(2, 2, 2) : MOE_RK(2, 2, 1)) : (T >= 2 ? MOE_RK(2, 1, 2) : MOE_RK(2, 1, 1));
#undef MOE_RK
  } else if (a.row_bytes % 32 == 0) {
    kern = dtype == MOE_F32 ? (const void*)k_reverse<MOE_F32, 1> : (const void*)k_reverse<MOE_BF16, 1>;
  } else {
    kern = dtype == MOE_F32 ? (const void*)k_reverse16<MOE_F32> : (const void*)k_reverse16<MOE_BF16>;
  }
  void* args[] = {&a};
  // CTAs per SM: the tuning's per-mode value (peer = the NVLink combine:
  // 8 measured 5% faster than the occupancy limit, C2 at N=2 reads 118.8 vs
  // 124.9 us, C4a 223.2 vs 230.4), else the row movers' setting, else the
  // occupancy limit
  const int cps = E_local != d.E ? tu.combine_ctas_per_sm : tu.reverse_ctas_per_sm;
  const int grid = cps > 0 ? cps * device_sm_count() : row_grid(kern);
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(kRowThreads), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_reverse_layout: launch");
  return MOE_OK;
}

bool reverse_kspec_used(const moe_gate_desc_t& d, int row_bytes) {
  return tuning().reverse_kspec && row_bytes % 32 == 0 && d.k <= 2;
}

moe_status_t reverse_launch(const moe_gate_desc_t& d, const moe_routing_t& r, const void* back,
                            int dtype, int dtype_size, int dcols, void* y, cudaStream_t stream,
                            const int32_t* offsets) {
  PeerPtrs src{};
  src.p[0] = const_cast<char*>(static_cast<const char*>(back));
  return reverse_launch_peers(d, r, src, d.E, 0, dtype, dtype_size, dcols, y, stream, offsets,
                              nullptr);
}

moe_status_t expert_scale_launch(const void* in, void* out, int nsrc, int E_local, int e_base,
                                 int cap, int dcols, int dtype, int dtype_size,
                                 cudaStream_t stream) {
  const int row_bytes = dcols * dtype_size;
  const long long n_rows = (long long)nsrc * E_local * cap;
  const void* kern =
      dtype == MOE_F32 ? (const void*)k_expert_scale<MOE_F32> : (const void*)k_expert_scale<MOE_BF16>;
  const char* pin = static_cast<const char*>(in);
  char* pout = static_cast<char*>(out);
  void* args[] = {&pin, &pout, (void*)&n_rows, (void*)&row_bytes, &cap, &E_local, &e_base};
  int grid = (int)std::min<long long>((n_rows + kRowWarps - 1) / kRowWarps,
                                      (long long)row_grid(kern));
  if (grid < 1) return MOE_OK;
  cudaError_t e = cudaLaunchKernel(kern, dim3(grid), dim3(kRowThreads), args, 0, stream);
  if (e != cudaSuccess) return cuda_status(e, "moe_expert_scale: launch");
  return MOE_OK;
}

moe_status_t chunk_permute_launch(const void* src, void* dst, int N, int G, long long chunk_bytes,
                                  cudaStream_t stream) {
  const long long total = (long long)N * G * G * (chunk_bytes / 16);
  int grid = (int)std::min<long long>((total + kRowThreads - 1) / kRowThreads,
                                      (long long)row_grid((const void*)k_chunk_permute));
  if (grid < 1) return MOE_OK;
  k_chunk_permute<<<grid, kRowThreads, 0, stream>>>(static_cast<const char*>(src),
                                                    static_cast<char*>(dst), N, G, chunk_bytes);
  MOE_CHECK_LAUNCH("moe_alltoall: k_chunk_permute launch");
  return MOE_OK;
}

moe_status_t chunk_transpose_launch(const void* src, void* dst, int X, int Y, long long chunk_bytes,
                                    cudaStream_t stream) {
  const long long total = (long long)X * Y * (chunk_bytes / 16);
  int grid = (int)std::min<long long>((total + kRowThreads - 1) / kRowThreads,
                                      (long long)row_grid((const void*)k_chunk_transpose));
  if (grid < 1) return MOE_OK;
  k_chunk_transpose<<<grid, kRowThreads, 0, stream>>>(static_cast<const char*>(src),
                                                      static_cast<char*>(dst), X, Y, chunk_bytes);
  MOE_CHECK_LAUNCH("moe_alltoall: k_chunk_transpose launch");
  return MOE_OK;
}

}  // namespace moe
