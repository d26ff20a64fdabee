// rows.cuh -- shared pieces of the row-moving kernels (layout.cu,
// backward.cu): the argument block with its peer-pointer row mapping, the
// padding-row prefix, 32-byte vector FMA/pack helpers and the grid size.
#pragma once
#include <algorithm>

#include "comm.cuh"

namespace moe {

constexpr int kRowThreads = 256;
constexpr int kRowWarps = kRowThreads / 32;

struct RowArgs {
  const char* src;
  char* dst;
  const int32_t* expert_idx;
  const int32_t* slot_idx;
  const float* weight;
  const int32_t* load;
  int S, E, k, cap;
  int row_bytes;
  int d;
  // layout destination: expert e lives on rank q = e / E_local and its rows
  // go to dpeer.p[q] + ((rank*E_local + e mod E_local)*cap + s)*row.  Local
  // moe_layout: dpeer.p[0] = dispatch, E_local = E, rank = 0.
  PeerPtrs dpeer;
  int E_local, rank;
  int sys_fence;  // stores went to peers: fence.sys before the CTA exits
  // reverse source: row (e, s) is read from speer.p[q] + ((rank*E_local +
  // e mod E_local)*cap + s)*row (same mapping; local: speer.p[0] = back)
  PeerPtrs speer;
  // dropless packed form (NEXT-4): when `offsets` ([E+1] expert offsets of
  // the sender) is set, row (e, s) is row base_q + offsets[e] -
  // offsets[q*E_local] + s of rank q's buffer, base_q = peer_base[q] (the
  // rows earlier source ranks put there; 0 locally); no padding rows.
  const int32_t* offsets;
  const int32_t* peer_base;
  // reverse only: walk the tokens from last to first (rev) -- the rows the
  // layout wrote last are the ones still in L2 -- and store y evict-first
  // (y_ef) so the stores do not push them out
  int rev, y_ef;
  // padded one-sided dispatch with LOCAL padding: the senders skip the zero
  // rows and CTA 0 stores min(load, cap) of each owner's experts into the
  // owner's padding-count table (ptab.p[q] + [rank][le]); the owner zero-fills
  // its own padding rows after the exit barrier (k_pad_fill)
  int skip_pads;
  PeerPtrs ptab;
  // layout only: zero the padding rows before the token rows, so the rows
  // written last (still in L2 for the combine's reversed walk) are rows the
  // combine reads
  int pads_first;
  // peer mode: a row going to the same remote owner as an earlier admitted
  // row of the same token (top-2 with both experts on one peer) is not sent
  // again; its recv row index gets "= row i" (i + 1) in the owner's table
  // dup.p[q] (int32 per recv row) and the owner copies it locally after the
  // exit barrier (k_dup_fill).  Reverse (peer combine): alias mode, see
  // src_row_item.
  int dedupe;
  PeerPtrs dup;
  // with dedupe: the owners' slot-weight tables (float per recv row): a pair
  // sent once gets both slots' combine weights, for the combine's
  // pre-combine (p == nullptr: not written)
  PeerPtrs wt;
  // peer combine (k_reverse_k, k = 2): a token whose two admitted slots sit
  // on one remote owner reads that owner's pre-combined row (pre.p[q], the
  // row of its second slot) instead of both expert rows; pre.p[0] == nullptr
  // = off
  PeerPtrs pre;
  // profiling (moe_set_trace): per CTA [entry, after the grid-dependency
  // wait, end] %globaltimer stamps at trace[4 * blockIdx.x + i], NULL = off
  unsigned long long* trace;
  long long trace_n;
};

__device__ __forceinline__ void row_trace(const RowArgs& a, int i) {
  const long long w = 4LL * blockIdx.x + i;
  if (a.trace && threadIdx.x == 0 && w < a.trace_n) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[w] = t;
  }
}
// the CTA's end stamp: after every warp of it is done
__device__ __forceinline__ void row_trace_end(const RowArgs& a) {
  if (a.trace) {
    __syncthreads();
    row_trace(a, 2);
  }
}

__device__ __forceinline__ size_t row_index(const RowArgs& a, int q, int e, int s) {
  if (a.offsets) {
    const int base = a.peer_base ? __ldg(a.peer_base + q) : 0;
    return (size_t)(base + __ldg(a.offsets + e) - __ldg(a.offsets + q * a.E_local) + s);
  }
  return (size_t)(a.rank * a.E_local + (e - q * a.E_local)) * a.cap + s;
}

__device__ __forceinline__ const char* src_row(const RowArgs& a, int e, int s) {
  const int q = e / a.E_local;
  return a.speer.p[q] + row_index(a, q, e, s) * a.row_bytes;
}

__device__ __forceinline__ char* dst_row_of(const RowArgs& a, int e, int s) {
  const int q = e / a.E_local;
  return a.dpeer.p[q] + row_index(a, q, e, s) * a.row_bytes;
}

// Dedupe (RowArgs::dedupe): if row j of token t (expert e, slot s, remote
// owner q) duplicates an earlier admitted row j' < j of t on the same owner,
// record it in q's table and return true (the caller skips the row).  Any
// lane may call it; only lane 0 stores.
__device__ __forceinline__ bool dedupe_row(const RowArgs& a, int t, int j, int e, int s, int lane) {
  const int q = e / a.E_local;
  if (!a.dedupe || q == a.rank) return false;
  for (int jj = 0; jj < j; ++jj) {
    const size_t i = (size_t)t * a.k + jj;
    const int s2 = __ldg(a.slot_idx + i);
    if (s2 < 0) continue;
    const int e2 = __ldg(a.expert_idx + i);
    if (e2 / a.E_local != q) continue;
    if (lane == 0) {
      const size_t rb = row_index(a, q, e, s), ra = row_index(a, q, e2, s2);
      reinterpret_cast<int*>(a.dup.p[q])[rb] = (int)ra + 1;
      if (a.wt.p[q] && a.weight) {
        reinterpret_cast<float*>(a.wt.p[q])[ra] = __ldg(a.weight + i);
        reinterpret_cast<float*>(a.wt.p[q])[rb] = __ldg(a.weight + (size_t)t * a.k + j);
      }
    }
    return true;
  }
  return false;
}

// Reverse source row of item (t, j) at (e, s).  With RowArgs::dedupe set on
// a peer-mode combine that runs before the owners' duplicate-row copies
// (moe_combine_p2p with NO_ENTRY_BARRIER after a deduped dispatch), a row
// the dispatch sent once for two slots of t is read from the first slot's
// row: recv still holds exactly what the dispatch sent, so the bytes are the
// same and the owner's copy into the second row is not waited for.
__device__ __forceinline__ const char* src_row_item(const RowArgs& a, int t, int j, int e, int s) {
  if (a.dedupe) {
    const int q = e / a.E_local;
    if (q != a.rank) {
      for (int jj = 0; jj < j; ++jj) {
        const size_t i = (size_t)t * a.k + jj;
        const int s2 = __ldg(a.slot_idx + i);
        if (s2 < 0) continue;
        const int e2 = __ldg(a.expert_idx + i);
        if (e2 / a.E_local == q) return src_row(a, e2, s2);
      }
    }
  }
  return src_row(a, e, s);
}

template <int VB>
struct Vec;
template <>
struct Vec<32> {
  using T = V8;
  static __device__ __forceinline__ T ld_stream(const void* p) { return ld_stream_v8(p); }
  static __device__ __forceinline__ T ld(const void* p) { return ld_v8(p); }
  static __device__ __forceinline__ void st(void* p, const T& v) { st_v8(p, v); }
  static __device__ __forceinline__ T zero() { return V8{{0, 0, 0, 0, 0, 0, 0, 0}}; }
};
template <>
struct Vec<16> {
  using T = V4;
  static __device__ __forceinline__ T ld_stream(const void* p) { return ld_stream_v4(p); }
  static __device__ __forceinline__ T ld(const void* p) {
    V4 r;
    asm volatile("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
                 : "l"(p));
    return r;
  }
  static __device__ __forceinline__ void st(void* p, const T& v) { st_v4(p, v); }
  static __device__ __forceinline__ T zero() { return V4{{0, 0, 0, 0}}; }
};

// Exclusive prefix of the padding-row counts cap - min(load[e], cap) into
// s_beg[0..E] (E <= 256), computed by every CTA (tiny).
__device__ __forceinline__ void pad_prefix(const RowArgs& a, int* s_beg) {
  __shared__ int s_cnt[257];
  const int tid = threadIdx.x;
  for (int e = tid; e < a.E; e += blockDim.x) {
    const int adm = a.offsets ? 0 : min(__ldg(a.load + e), a.cap);
    s_cnt[e] = (a.offsets || a.skip_pads) ? 0 : a.cap - adm;  // packed / local padding: none here
    if (a.skip_pads && blockIdx.x == 0) {
      const int q = e / a.E_local;
      reinterpret_cast<int*>(a.ptab.p[q])[a.rank * kPadTabStride + (e - q * a.E_local)] = adm;
    }
  }
  __syncthreads();
  if (tid < 32) {
    int carry = 0;
    for (int base = 0; base < a.E; base += 32) {
      const int e = base + tid;
      int v = e < a.E ? s_cnt[e] : 0;
      int incl = v;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        int o = __shfl_up_sync(0xffffffffu, incl, m);
        if (tid >= m) incl += o;
      }
      if (e < a.E) s_beg[e] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tid == 0) s_beg[a.E] = carry;
  }
  __syncthreads();
}

struct F32Acc {
  static constexpr int kPerVec = 8;  // fp32 per 32 bytes
};

template <int DT>  // MOE_F32 or MOE_BF16; 32-byte vectors
__device__ __forceinline__ void fma_vec(float* acc, float w, const V8& v) {
  if constexpr (DT == MOE_F32) {
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = fmaf(w, __uint_as_float(v.w[q]), acc[q]);
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      acc[2 * q] = fmaf(w, bf16lo(v.w[q]), acc[2 * q]);
      acc[2 * q + 1] = fmaf(w, bf16hi(v.w[q]), acc[2 * q + 1]);
    }
  }
}
template <int DT>
__device__ __forceinline__ V8 pack_vec(const float* acc) {
  V8 o;
  if constexpr (DT == MOE_F32) {
#pragma unroll
    for (int q = 0; q < 8; ++q) o.w[q] = __float_as_uint(acc[q]);
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) o.w[q] = pack_bf16x2(acc[2 * q], acc[2 * q + 1]);
  }
  return o;
}

// Combine weight of item i; a NULL weight array means unit weights (the
// adjoint of Layout_Transform is the combine with w = 1).
__device__ __forceinline__ float row_weight(const RowArgs& a, size_t i) {
  return a.weight ? __ldg(a.weight + i) : 1.f;
}

// Persistent grid: SMs x resident CTAs of `kern` at kRowThreads threads.
// Zero-fill the padding rows [min(load_e, cap), cap) of every expert (the
// prefix s_beg from pad_prefix), a warp per row, warps gw of nw.
template <int VB>
__device__ __forceinline__ void zero_pad_rows(const RowArgs& a, const int* s_beg, int gw, int nw) {
  using V = Vec<VB>;
  const int lane = threadIdx.x & 31;
  const int npad = s_beg[a.E];
  const typename V::T z = V::zero();
  for (int p = gw; p < npad; p += nw) {
    int lo = 0, hi = a.E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_beg[mid] <= p) lo = mid; else hi = mid - 1;
    }
    char* drow = dst_row_of(a, lo, min(__ldg(a.load + lo), a.cap) + (p - s_beg[lo]));
    for (int off = lane * VB; off < a.row_bytes; off += 32 * VB) V::st(drow + off, z);
  }
}

inline int row_grid(const void* kern) {
  int per_sm = tuning().row_ctas_per_sm;
  if (per_sm <= 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowThreads, 0);
  return std::max(1, per_sm) * device_sm_count();
}

// Grid of the local layout: ~layout_tokens_per_warp tokens per warp, at
// least the persistent grid, so the block scheduler balances the tail over
// the SMs (DESIGN.md §6 k_layout); stores to peers keep the persistent grid.
inline int scatter_grid(const void* kern, long long S, bool peer) {
  int grid = row_grid(kern);
  const int tpw = tuning().layout_tokens_per_warp;
  if (tpw > 0 && !peer) {
    const long long per_cta = (long long)kRowWarps * tpw;
    grid = (int)std::max<long long>(grid, (S + per_cta - 1) / per_cta);
  }
  return grid;
}

}  // namespace moe
