// gate_layout.cuh -- steps 1 + 2 of Algorithm 1 in ONE
// persistent kernel: the gate (Eq. 1 selection and weights, PAPER.md:100-106;
// capacity) and Layout_Transform, so the
// latency-bound gate hides behind the bandwidth-bound row scatter.
//
// Why it can be one pass.  Under TOKEN priority (R5, the default) the slot of
// item (t, j) is the number of earlier tokens' items for the same expert (a
// token names an expert at most once): an exclusive prefix sum over tokens.
// Every CTA of the persistent grid runs two phases, each driven by its own
// device-side counter, so a CTA only ever waits on work that running CTAs
// already hold (no co-residency assumption):
//   G. gate tiles (the separate gate's tiles, in order): select + weigh the
//      tile's tokens and rank its items per expert (gate_tile, the gate's own
//      code); publish the per-expert aggregate, resolve the exclusive prefix
//      by a decoupled look-back over earlier tiles (a warp reads 32
//      predecessors' status words for 4 experts at once: aggregate "A" or
//      inclusive prefix "P", epoch-tagged so the workspace never needs
//      clearing), publish the inclusive prefix, write the final slots (>=
//      cap: dropped, weight 0; slot_src) and raise the tile's ready word.
//      (Measured slower and dropped: group totals instead of the look-back,
//      C2 prefix 7.7 vs 2.8 us);
//   S. scatter chunks of 32 tokens, in token order: bulk-prefetch the
//      chunk's x rows into L2, wait for the chunk's tile to be ready, then a
//      warp per token reads its x row once and stores it to its <= k slots --
//      in peer mode straight into the owner rank's receive buffer over
//      NVLink, a token's row once per remote owner (dedupe), as k_layout.
//      (Measured slower and dropped: a static token interleave over all
//      warps, C3 71 vs 63 us; warp-level claims of 4-token batches without
//      the prefetch, C3 73 us.)
// Most CTAs hold no gate tile and start scattering as soon as tile 0 is
// ready, so the gate's latency overlaps the row traffic.  The CTA of the last
// tile writes load[] and raises the totals word; every CTA then zero-fills
// its share of the padding rows [min(load, cap), cap) and of slot_src's empty
// entries.  The last CTA out resets the counters and advances the epoch
// (CUDA-graph replay safe).  Outputs are bit-identical to moe_gate followed
// by moe_layout (tested).

#pragma once
#include "gate_impl.cuh"
#include "rows.cuh"

namespace moe {

struct FusedCtrl {        // at FusedPlan::ctrl_off of the gate workspace
  unsigned tile_next;     // phase G counter (reset by the last CTA)
  unsigned chunk_next;    // phase S counter (reset by the last CTA)
  unsigned done;          // CTAs finished (reset by the last CTA)
  unsigned epoch;         // launch number, tags the status and ready words
  unsigned ready;         // = epoch + 1 once load[] of this launch is final
  unsigned pad[11];
};

constexpr int kScatterChunk = 32;  // tokens per phase-S work unit (divides every tile)

struct FusedArgs {
  GateArgs g;              // the gate (its tiles; ncols = E)
  RowArgs r;               // the rows: src = x, destinations, peer mode, dedupe
  FusedCtrl* fc;
  unsigned long long* st;  // [n_tiles][E] status: epoch:30 | flag:2 | count:32
  unsigned* tile_ready;    // [n_tiles] = epoch + 1 once the tile's slots are final
  // profiling (moe_set_trace): %globaltimer stamps, NULL = off.  Per tile
  // [claim, aggregate published, prefix published, ready]; per chunk
  // [claim, tile ready seen]; per CTA [start, end]
  unsigned long long* trace;
  long long trace_n;
};

// trace layout: [0..3] = n_tiles, n_chunks, gridDim.x, 0; stamps from 4 on
__device__ __forceinline__ void trace_at(const FusedArgs& f, long long i) {
  i += 4;
  if (f.trace && i < f.trace_n) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    f.trace[i] = t;
  }
}

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

// The same for CG consecutive columns c0 .. c0+CG-1 at once: each lane
// reads the CG status words of one predecessor with a single vector load
// (the tile's words are contiguous; E % CG == 0 keeps it aligned).
template <int CG>
__device__ __forceinline__ void lookback_cg(const unsigned long long* st, int tile, int c0, int E,
                                            unsigned epoch, int lane, unsigned* excl) {
  static_assert(CG == 4, "vector width");
#pragma unroll
  for (int j = 0; j < CG; ++j) excl[j] = 0;
  unsigned open = (1u << CG) - 1;  // columns still looking back
  for (int base = tile - 1; open; base -= 32) {
    const int idx = base - lane;
    for (;;) {
      unsigned long long w[CG];
      if (idx >= 0) {
        asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3])
                     : "l"(st + (size_t)idx * E + c0)
                     : "memory");
      }
      bool wait = false;
      unsigned s[CG];
      int firstP[CG];
#pragma unroll
      for (int j = 0; j < CG; ++j) {
        const unsigned f = idx >= 0 ? st_flag(w[j], epoch) : kFlagP;
        const unsigned v = idx >= 0 ? (unsigned)w[j] : 0u;
        const unsigned pmask = __ballot_sync(0xffffffffu, f == kFlagP);
        const unsigned zmask = __ballot_sync(0xffffffffu, f == 0);
        firstP[j] = pmask ? __ffs(pmask) - 1 : 32;
        const unsigned need = firstP[j] < 31 ? ((2u << firstP[j]) - 1u) : 0xffffffffu;
        if ((open >> j & 1u) && (zmask & need)) wait = true;
        s[j] = lane <= firstP[j] ? v : 0u;
      }
      if (wait) {
        __nanosleep(32);
        continue;
      }
#pragma unroll
      for (int j = 0; j < CG; ++j) {
        unsigned t = s[j];
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
        if (open >> j & 1u) {
          excl[j] += t;
          if (firstP[j] < 32) open &= ~(1u << j);
        }
      }
      break;
    }
  }
}

template <int KIND, int L, int K, int U>
__global__ void __launch_bounds__(kGateThreads, 4) k_gate_layout(FusedArgs f) {
  constexpr int VB = 32, SEG = 32 * U * VB;
  extern __shared__ __align__(16) int smem[];
  __shared__ unsigned s_bad;
  __shared__ __align__(8) unsigned long long s_mbar;
  __shared__ int s_work;
  __shared__ unsigned s_epoch;
  __shared__ int s_pre[257], s_agg[256];  // s_pre doubles as the padding prefix [E + 1]
  const GateArgs& a = f.g;
  const RowArgs& ra = f.r;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int items = a.tile_tokens * a.k;
  int* s_exp = smem + a.lg_words;   // gate_tile's arrays (z_words = 0 here)
  const int* s_rank = s_exp + items;
  const int* s_hist = s_rank + items;
  const int per = (items + kGateWarps - 1) / kGateWarps;

  pdl_wait();     // the logits' producer / the previous step are complete
  pdl_trigger();
  const int n_chunks = (a.S + kScatterChunk - 1) / kScatterChunk;
  const long long tr_chunk = 4LL * a.n_tiles, tr_cta = tr_chunk + 2LL * n_chunks;
  if (tid == 0) {
    if (f.trace && blockIdx.x == 0 && f.trace_n >= 4) {
      f.trace[0] = (unsigned long long)a.n_tiles;
      f.trace[1] = (unsigned long long)n_chunks;
      f.trace[2] = gridDim.x;
    }
    trace_at(f, tr_cta + 2LL * blockIdx.x);
    if (KIND != KIND_HASH) gate_mbar_init(s_mbar);
    s_epoch = *reinterpret_cast<volatile unsigned*>(&f.fc->epoch);
  }
  __syncthreads();
  const unsigned epoch = s_epoch;
  unsigned parity = 0;

  // ---------------- phase G: gate tiles in order.  A CTA leaves only once
  // the counter ran out, i.e. every tile is held by a running CTA, so phase
  // S never waits on a tile nobody holds (a plain read first spares the
  // atomic once it ran out).
  for (;;) {
    if (tid == 0)
      s_work = *reinterpret_cast<volatile unsigned*>(&f.fc->tile_next) >= (unsigned)a.n_tiles
                   ? a.n_tiles
                   : (int)atomicAdd(&f.fc->tile_next, 1u);
    __syncthreads();
    const int tile = s_work;
    if (tile >= a.n_tiles) break;
    if (tid == 0) trace_at(f, 4LL * tile);
    const int t0 = tile * a.tile_tokens;
    const int nt = min(a.tile_tokens, a.S - t0);
    gate_tile<KIND, L, K>(a, smem, s_bad, s_mbar, tile, parity, s_agg);
    parity ^= 1u;
    if (KIND == KIND_HASH && tid == 0 && s_bad) atomicAdd(&a.ctrl->bad, s_bad);
    // publish the aggregate, look back, publish the inclusive prefix
    unsigned long long* st = f.st + (size_t)tile * a.E;
    if (tile == 0) {
      for (int c = tid; c < a.E; c += kGateThreads) {
        s_pre[c] = 0;
        st_relaxed_gpu(st + c, st_pack(epoch, kFlagP, (unsigned)s_agg[c]));
      }
    } else {
      for (int c = tid; c < a.E; c += kGateThreads)
        st_relaxed_gpu(st + c, st_pack(epoch, kFlagA, (unsigned)s_agg[c]));
      if (tid == 0) trace_at(f, 4LL * tile + 1);
      if (a.E % 4 == 0) {  // four columns per vector load
        for (int c0 = warp * 4; c0 < a.E; c0 += kGateWarps * 4) {
          unsigned ex[4];
          lookback_cg<4>(f.st, tile, c0, a.E, epoch, lane, ex);
          if (lane < 4) {
            const unsigned e = lane == 0 ? ex[0] : lane == 1 ? ex[1] : lane == 2 ? ex[2] : ex[3];
            s_pre[c0 + lane] = (int)e;
            st_relaxed_gpu(st + c0 + lane, st_pack(epoch, kFlagP, e + (unsigned)s_agg[c0 + lane]));
          }
        }
      } else {
        for (int c = warp; c < a.E; c += kGateWarps) {
          const unsigned ex = lookback(f.st, tile, c, a.E, epoch, lane);
          if (lane == 0) {
            s_pre[c] = (int)ex;
            st_relaxed_gpu(st + c, st_pack(epoch, kFlagP, ex + (unsigned)s_agg[c]));
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0) trace_at(f, 4LL * tile + 2);
    // final slots, dropped items, slot_src
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
    }
    const bool last = tile == a.n_tiles - 1;
    if (last)  // the totals: requests per expert (TOKEN: the column)
      for (int c = tid; c < a.E; c += kGateThreads) a.load[c] = s_pre[c] + s_agg[c];
    __syncthreads();
    if (tid == 0) {  // one fence after the barrier covers the CTA's stores
      __threadfence();
      trace_at(f, 4LL * tile + 3);
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f.tile_ready + tile),
                   "r"(epoch + 1u) : "memory");
      if (last)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&f.fc->ready), "r"(epoch + 1u)
                     : "memory");
    }
  }

  // ---------------- phase S: scatter chunks of tokens in order
  for (;;) {
    __syncthreads();  // s_work is rewritten
    if (tid == 0) {
      const int c = (int)atomicAdd(&f.fc->chunk_next, 1u);
      s_work = c;
      if (c < n_chunks) {
        trace_at(f, tr_chunk + 2LL * c);
        // the chunk's x rows (contiguous) do not depend on the routing: they
        // stream into L2 while the tile may still be resolving
        const unsigned long long beg = (unsigned long long)c * kScatterChunk * ra.row_bytes;
        const unsigned long long n =
            (unsigned long long)(min(a.S, (c + 1) * kScatterChunk) - c * kScatterChunk) * ra.row_bytes;
        for (unsigned long long o = 0; o < n; o += 65536)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ra.src + beg + o),
                       "r"((unsigned)min(65536ull, n - o))
                       : "memory");
        const unsigned* rdy = f.tile_ready + (c * kScatterChunk) / a.tile_tokens;
        while (ld_acquire_gpu_u32(rdy) != epoch + 1u) __nanosleep(32);
        trace_at(f, tr_chunk + 2LL * c + 1);
      }
    }
    __syncthreads();
    const int c = s_work;
    if (c >= n_chunks) break;
    const int t_end = min(a.S, (c + 1) * kScatterChunk);
    for (int t = c * kScatterChunk + warp; t < t_end; t += kGateWarps) {
      // lane j < k: slot j of token t (written by another CTA: L2 loads)
      int my_e = -1, my_s = -1;
      if (lane < a.k) {
        my_s = __ldcg(a.slot_idx + (size_t)t * a.k + lane);
        my_e = __ldcg(a.expert_idx + (size_t)t * a.k + lane);
      }
      const char* srow = ra.src + (size_t)t * ra.row_bytes;
      for (int seg = 0; seg < ra.row_bytes; seg += SEG) {
        V8 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int off = seg + (lane + 32 * u) * VB;
          if (off < ra.row_bytes) r[u] = ld_stream_v8(srow + off);
        }
        for (int j = 0; j < a.k; ++j) {
          const int s = __shfl_sync(0xffffffffu, my_s, j);
          if (s < 0) continue;
          const int e = __shfl_sync(0xffffffffu, my_e, j);
          const int q = e / ra.E_local;
          if (ra.dedupe && q != ra.rank && j > 0) {
            // a row already bound for this remote owner: record "= row of j'"
            int jj = 0, e2 = -1, s2 = -1;
            for (; jj < j; ++jj) {
              s2 = __shfl_sync(0xffffffffu, my_s, jj);
              e2 = __shfl_sync(0xffffffffu, my_e, jj);
              if (s2 >= 0 && e2 / ra.E_local == q) break;
            }
            if (jj < j) {
              if (seg == 0 && lane == 0) {
                const size_t rb = row_index(ra, q, e, s), rr = row_index(ra, q, e2, s2);
                reinterpret_cast<int*>(ra.dup.p[q])[rb] = (int)rr + 1;
                if (ra.wt.p[q] && ra.weight) {  // this kernel wrote the weights: plain loads
                  const size_t it = (size_t)t * a.k;
                  reinterpret_cast<float*>(ra.wt.p[q])[rr] = __ldcg(ra.weight + it + jj);
                  reinterpret_cast<float*>(ra.wt.p[q])[rb] = __ldcg(ra.weight + it + j);
                }
              }
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
  }

  // ---------------- padding rows [min(load, cap), cap) and empty slot_src
  // entries, once the CTA of the last tile published load[]
  if (tid == 0)
    while (ld_acquire_gpu_u32(&f.fc->ready) != epoch + 1u) __nanosleep(64);
  __syncthreads();
  int* s_beg = s_pre;  // [E + 1] <= 257
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
  // ---------------- the last CTA out resets the counters for the next launch
  __syncthreads();
  if (tid == 0) {
    trace_at(f, tr_cta + 2LL * blockIdx.x + 1);
    __threadfence();
    if (atomicAdd(&f.fc->done, 1u) == gridDim.x - 1) {
      f.fc->tile_next = 0;
      f.fc->chunk_next = 0;
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
