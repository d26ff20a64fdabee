// gate_layout.cuh -- steps 1 + 2 of Algorithm 1 in ONE
// persistent kernel: the gate (Eq. 1 selection and weights, PAPER.md:100-106;
// capacity) and Layout_Transform, so the
// latency-bound gate hides behind the bandwidth-bound row scatter.
//
// Why it can be one pass.  Under TOKEN priority (R5, the default) the slot of
// item (t, j) is the number of earlier tokens' items for the same expert plus
// nothing else (a token names an expert at most once), i.e. an exclusive
// prefix sum over tokens.  The kernel walks tiles of T tokens in order of a
// device-side tile counter (so a tile only ever waits on tiles that running
// CTAs already hold -- no co-residency assumption) and, per tile:
//   1. bulk-prefetches the tile's x rows into L2 (they do not depend on the
//      routing), then selects + weighs its tokens (gate_tile, the gate's own
//      code) and ranks its items per expert inside the tile;
//   2. publishes its per-expert aggregate, then resolves the exclusive
//      prefix by a decoupled look-back over earlier tiles (a warp reads 32
//      predecessors' status words at once: aggregate "A" or inclusive
//      prefix "P", epoch-tagged so the workspace never needs clearing) and
//      publishes its inclusive prefix;
//   3. finishes its slots (>= cap: dropped, weight 0; slot_src), and
//   4. scatters its x rows (now in L2) to their <= k slots -- in peer mode
//      straight into the owner rank's receive buffer over NVLink, sending a
//      token's row once per remote owner (dedupe), as k_layout does.
// The CTA that finishes the last tile writes load[] and raises a ready
// word; every CTA then zero-fills its share of the padding rows [min(load,
// cap), cap) and of slot_src's empty entries.  The last CTA to finish resets
// the tile counter and advances the epoch (CUDA-graph replay safe).
// Outputs are bit-identical to moe_gate followed by moe_layout (tested).
#pragma once
#include "gate_impl.cuh"
#include "rows.cuh"

namespace moe {

struct FusedCtrl {        // at FusedLayout::ctrl_off of the gate workspace
  unsigned tile_next;     // tile counter (reset by the last CTA)
  unsigned done;          // CTAs finished (reset by the last CTA)
  unsigned epoch;         // launch number, tags the status words
  unsigned ready;         // = epoch + 1 once load[] of this launch is final
  unsigned bad;           // unused (invalid hash ids go to GateCtrl::bad)
  unsigned pad[11];
};

struct FusedArgs {
  GateArgs g;              // the gate (tile_tokens, n_tiles of the fused plan; ncols = E)
  RowArgs r;               // the rows: src = x, destinations, peer mode, dedupe
  FusedCtrl* fc;
  unsigned long long* st;  // [n_tiles][E] status: epoch:30 | flag:2 | count:32
};

constexpr unsigned kFlagA = 1, kFlagP = 2;

__device__ __forceinline__ unsigned long long st_pack(unsigned epoch, unsigned flag, unsigned v) {
  return ((unsigned long long)(epoch & 0x3FFFFFFFu) << 34) | ((unsigned long long)flag << 32) | v;
}
__device__ __forceinline__ unsigned st_flag(unsigned long long w, unsigned epoch) {
  return (unsigned)(w >> 34) == (epoch & 0x3FFFFFFFu) ? (unsigned)(w >> 32) & 3u : 0u;
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Exclusive prefix over tiles < tile of column c (one warp): look back 32
// tiles per round; wait until every tile up to the nearest inclusive prefix
// has published at least its aggregate.
__device__ __forceinline__ unsigned lookback(const unsigned long long* st, int tile, int c, int E,
                                             unsigned epoch, int lane) {
  unsigned excl = 0;
  for (int base = tile - 1;; base -= 32) {
    const int idx = base - lane;
    unsigned f, v;
    for (;;) {
      if (idx >= 0) {
        const unsigned long long w = ld_relaxed_gpu(st + (size_t)idx * E + c);
        f = st_flag(w, epoch);
        v = (unsigned)w;
      } else {
        f = kFlagP;  // before tile 0: prefix 0
        v = 0;
      }
      const unsigned pmask = __ballot_sync(0xffffffffu, f == kFlagP);
      const unsigned zmask = __ballot_sync(0xffffffffu, f == 0);
      const int firstP = pmask ? __ffs(pmask) - 1 : 32;
      const unsigned need = firstP < 31 ? ((2u << firstP) - 1u) : 0xffffffffu;
      if (!(zmask & need)) {
        unsigned s = lane <= firstP ? v : 0u;
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
        excl += s;
        if (firstP < 32) return excl;
        break;
      }
      __nanosleep(32);
    }
  }
}

template <int KIND, int L, int K, int U>
__global__ void __launch_bounds__(kGateThreads) k_gate_layout(FusedArgs f) {
  constexpr int VB = 32, SEG = 32 * U * VB;
  extern __shared__ __align__(16) int smem[];
  __shared__ unsigned s_bad;
  __shared__ __align__(8) unsigned long long s_mbar;
  __shared__ int s_tile;
  __shared__ unsigned s_epoch;
  __shared__ int s_agg[256], s_pre[256];
  const GateArgs& a = f.g;
  const RowArgs& ra = f.r;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int items = a.tile_tokens * a.k;
  int* s_exp = smem + a.lg_words;   // gate_tile's arrays (z_words = 0 here)
  int* s_rank = s_exp + items;
  const int* s_hist = s_rank + items;
  const int per = (items + kGateWarps - 1) / kGateWarps;

  pdl_wait();     // the logits' producer / the previous step are complete
  pdl_trigger();
  if (tid == 0) {
    if (KIND != KIND_HASH) gate_mbar_init(s_mbar);
    s_epoch = *reinterpret_cast<volatile unsigned*>(&f.fc->epoch);
  }
  __syncthreads();
  const unsigned epoch = s_epoch;
  unsigned parity = 0;
  for (;;) {
    if (tid == 0) s_tile = (int)atomicAdd(&f.fc->tile_next, 1u);
    __syncthreads();
    const int tile = s_tile;
    if (tile >= a.n_tiles) break;
    const int t0 = tile * a.tile_tokens;
    const int nt = min(a.tile_tokens, a.S - t0);
    if (tid == 0) {  // the tile's x rows (contiguous) stream into L2 meanwhile
      const unsigned long long beg = (unsigned long long)t0 * ra.row_bytes;
      const unsigned long long n = (unsigned long long)nt * ra.row_bytes;
      for (unsigned long long o = 0; o < n; o += 65536)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ra.src + beg + o),
                     "r"((unsigned)min(65536ull, n - o))
                     : "memory");
    }
    // ---- 1. select + weights + in-tile ranks (s_exp, s_rank, s_hist, s_agg)
    gate_tile<KIND, L, K>(a, smem, s_bad, s_mbar, tile, parity, s_agg);
    parity ^= 1u;
    if (KIND == KIND_HASH && tid == 0 && s_bad) atomicAdd(&a.ctrl->bad, s_bad);
    // ---- 2. publish the aggregate, look back, publish the inclusive prefix
    unsigned long long* st = f.st + (size_t)tile * a.E;
    if (tile == 0) {
      for (int c = tid; c < a.E; c += kGateThreads) {
        s_pre[c] = 0;
        st_relaxed_gpu(st + c, st_pack(epoch, kFlagP, (unsigned)s_agg[c]));
      }
    } else {
      for (int c = tid; c < a.E; c += kGateThreads)
        st_relaxed_gpu(st + c, st_pack(epoch, kFlagA, (unsigned)s_agg[c]));
      for (int c = warp; c < a.E; c += kGateWarps) {
        const unsigned ex = lookback(f.st, tile, c, a.E, epoch, lane);
        if (lane == 0) {
          s_pre[c] = (int)ex;
          st_relaxed_gpu(st + c, st_pack(epoch, kFlagP, ex + (unsigned)s_agg[c]));
        }
      }
    }
    __syncthreads();
    if (tile == a.n_tiles - 1) {  // the totals: requests per expert (TOKEN: the column)
      for (int c = tid; c < a.E; c += kGateThreads) a.load[c] = s_pre[c] + s_agg[c];
      __threadfence();
      __syncthreads();
      if (tid == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&f.fc->ready),
                                 "r"(epoch + 1u) : "memory");
    }
    // ---- 3. final slots (in s_rank), dropped items, slot_src
    for (int i = tid; i < nt * a.k; i += kGateThreads) {
      const int e = s_exp[i];
      const size_t gi = (size_t)t0 * a.k + i;
      int s = -1;
      if (e >= 0) {
        s = s_pre[e] + s_hist[(i / per) * a.ncols + e] + s_rank[i];
        if (s < a.cap) {
          if (a.slot_src) a.slot_src[(size_t)e * a.cap + s] = (int)gi;
        } else {
          s = -1;
          a.weight[gi] = 0.f;
        }
      }
      a.slot_idx[gi] = s;
      s_rank[i] = s;
    }
    __syncthreads();
    // ---- 4. scatter the tile's rows, a warp per token
    for (int tt = warp; tt < nt; tt += kGateWarps) {
      const int t = t0 + tt;
      const char* srow = ra.src + (size_t)t * ra.row_bytes;
      for (int seg = 0; seg < ra.row_bytes; seg += SEG) {
        V8 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int off = seg + (lane + 32 * u) * VB;
          if (off < ra.row_bytes) r[u] = ld_v8(srow + off);
        }
        for (int j = 0; j < a.k; ++j) {
          const int s = s_rank[tt * a.k + j];
          if (s < 0) continue;
          const int e = s_exp[tt * a.k + j];
          const int q = e / ra.E_local;
          if (ra.dedupe && q != ra.rank && j > 0) {
            // a row already bound for this remote owner: record "= row of j'"
            int jj = 0;
            for (; jj < j; ++jj) {
              const int s2 = s_rank[tt * a.k + jj];
              if (s2 >= 0 && s_exp[tt * a.k + jj] / ra.E_local == q) break;
            }
            if (jj < j) {
              if (seg == 0 && lane == 0)
                reinterpret_cast<int*>(ra.dup.p[q])[row_index(ra, q, e, s)] =
                    (int)row_index(ra, q, s_exp[tt * a.k + jj], s_rank[tt * a.k + jj]) + 1;
              continue;
            }
          }
          char* drow = dst_row_of(ra, e, s);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int off = seg + (lane + 32 * u) * VB;
            if (off < ra.row_bytes) st_v8(drow + off, r[u]);
          }
        }
      }
    }
    __syncthreads();  // s_tile, s_exp and s_rank are reused by the next tile
  }

  // ---- padding rows [min(load, cap), cap) and empty slot_src entries,
  // once the CTA of the last tile published load[]
  if (tid == 0)
    while (ld_acquire_gpu_u32(&f.fc->ready) != epoch + 1u) __nanosleep(64);
  __syncthreads();
  __shared__ int s_beg[257];
  if (tid < 32) {
    int carry = 0;
    for (int base = 0; base < a.E; base += 32) {
      const int e = base + lane;
      const int adm = e < a.E ? min(__ldcg(a.load + e), a.cap) : a.cap;
      if (ra.skip_pads && blockIdx.x == 0 && e < a.E) {  // owners zero their own padding
        const int q = e / ra.E_local;
        reinterpret_cast<int*>(ra.ptab.p[q])[ra.rank * kPadTabStride + (e - q * ra.E_local)] = adm;
      }
      const int v = ra.skip_pads ? 0 : a.cap - adm;
      int incl = v;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, m);
        if (lane >= m) incl += o;
      }
      if (e < a.E) s_beg[e] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_beg[a.E] = carry;
  }
  __syncthreads();
  const int gw = blockIdx.x * kGateWarps + warp, nw = gridDim.x * kGateWarps;
  const V8 z = V8{{0, 0, 0, 0, 0, 0, 0, 0}};
  for (int p = gw; p < s_beg[a.E]; p += nw) {
    int lo = 0, hi = a.E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_beg[mid] <= p) lo = mid; else hi = mid - 1;
    }
    char* drow = dst_row_of(ra, lo, min(__ldcg(a.load + lo), a.cap) + (p - s_beg[lo]));
    for (int off = lane * VB; off < ra.row_bytes; off += 32 * VB) st_v8(drow + off, z);
  }
  if (a.slot_src)
    for (int e = gw; e < a.E; e += nw)
      for (int s = min(__ldcg(a.load + e), a.cap) + lane; s < a.cap; s += 32)
        a.slot_src[(size_t)e * a.cap + s] = -1;
  if (ra.sys_fence) __threadfence_system();
  // ---- the last CTA out resets the counters for the next launch
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&f.fc->done, 1u) == gridDim.x - 1) {
      f.fc->tile_next = 0;
      f.fc->done = 0;
      __threadfence();
      f.fc->epoch = epoch + 1u;
    }
  }
}

using FusedKernel = void (*)(FusedArgs);

template <int KIND, int L>
inline FusedKernel pick_fused_k(int K, int U) {
  switch (K) {
    case 1: return U == 4 ? k_gate_layout<KIND, L, 1, 4> : k_gate_layout<KIND, L, 1, 2>;
    case 2: return U == 4 ? k_gate_layout<KIND, L, 2, 4> : k_gate_layout<KIND, L, 2, 2>;
    case 4: return U == 4 ? k_gate_layout<KIND, L, 4, 4> : k_gate_layout<KIND, L, 4, 2>;
    default: return U == 4 ? k_gate_layout<KIND, L, 8, 4> : k_gate_layout<KIND, L, 8, 2>;
  }
}
template <int KIND>
inline FusedKernel pick_fused_l(int L, int K, int U) {
  switch (L) {
    case 1: return pick_fused_k<KIND, 1>(K, U);
    case 2: return pick_fused_k<KIND, 2>(K, U);
    case 4: return pick_fused_k<KIND, 4>(K, U);
    case 8: return pick_fused_k<KIND, 8>(K, U);
    case 16: return pick_fused_k<KIND, 16>(K, U);
    default: return pick_fused_k<KIND, 32>(K, U);
  }
}

// gate_layout_topk.cu / gate_layout_misc.cu
FusedKernel pick_fused_topk(int L, int K, int U);
FusedKernel pick_fused_ktop1(int L, int K, int U);
FusedKernel pick_fused_hash(int U);

}  // namespace moe
