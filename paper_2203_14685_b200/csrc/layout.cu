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
  if (a.prefetch) prefetch_share_l2(a.src, (size_t)a.S * a.row_bytes);
  pdl_wait();     // routing comes from moe_gate
  pdl_trigger();
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
}

// Layout for 32-byte-vector rows with TPW consecutive tokens per warp
// iteration: all TPW*U row loads are in flight before the first store (a
// 2 KiB row with U = 2, TPW = 2 keeps 4 KiB per warp in flight, like a
// 4 KiB row with U = 4).  The zero padding rows follow as their own
// grid-stride loop over warps.
template <int U, int TPW>
__global__ void __launch_bounds__(kRowThreads) k_layout_t(RowArgs a) {
  constexpr int VB = 32;
  constexpr int SEG = 32 * U * VB;
  __shared__ int s_beg[257];
  pdl_wait();
  pdl_trigger();
  pad_prefix(a, s_beg);
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  const int nw = gridDim.x * kRowWarps;
  for (int tb = gw * TPW; tb < a.S; tb += nw * TPW) {
    for (int seg = 0; seg < a.row_bytes; seg += SEG) {
      V8 r[TPW][U];
#pragma unroll
      for (int p = 0; p < TPW; ++p)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int off = seg + (lane + 32 * u) * VB;
          if (tb + p < a.S && off < a.row_bytes)
            r[p][u] = ld_stream_v8(a.src + (size_t)(tb + p) * a.row_bytes + off);
        }
#pragma unroll
      for (int p = 0; p < TPW; ++p) {
        const int t = tb + p;
        if (t >= a.S) break;
        for (int j = 0; j < a.k; ++j) {
          const int s = __ldg(a.slot_idx + (size_t)t * a.k + j);
          if (s < 0) continue;
          char* drow = dst_row_of(a, __ldg(a.expert_idx + (size_t)t * a.k + j), s);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int off = seg + (lane + 32 * u) * VB;
            if (off < a.row_bytes) st_v8(drow + off, r[p][u]);
          }
        }
      }
    }
  }
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

// ------------------------------------------------------------ gate-finalize + layout
// Layout_Transform fused with the last pass of the gate (the capacity
// slots): the select kernel left the provisional slots (rank inside the
// tile's column) and the per-tile column aggregates; every CTA reduces the
// aggregates into the exclusive prefix over tiles in shared memory (or reads
// the prefixes k_gate_scan made, for big tables), and each token's warp
// finishes its k slots (lane j: slot j) -- drop at >= cap, weight 0, slot_src
// -- then scatters the row to the final slots.  One kernel boundary fewer
// than gate (select -> slots) -> layout, with the same outputs bit for bit.
template <int U>
__global__ void __launch_bounds__(kRowThreads) k_layout_fin(RowArgs a, GateFinalize f) {
  constexpr int VB = 32, SEG = 32 * U * VB;
  extern __shared__ int fsm[];
  int* T = fsm;                // [ncols] column totals
  int* Pt = fsm + f.ncols;     // [ncols][n_tiles] exclusive prefixes (scanned == 0)
  __shared__ int s_beg[257];
  __shared__ int s_cnt[257];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();  // the select (and scan) kernels are complete
  pdl_trigger();
  for (int c = warp; c < f.ncols; c += kRowWarps) {
    if (f.scanned) {
      if (lane == 0) T[c] = __ldcg(f.totals + c);
      continue;
    }
    const unsigned* col = f.agg + (size_t)c * f.n_tiles;
    unsigned carry = 0;
    for (int base = 0; base < f.n_tiles; base += 256) {
      unsigned v[8], run = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + lane * 8 + u;
        v[u] = i < f.n_tiles ? __ldcg(col + i) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const unsigned x = v[u];
        v[u] = run;
        run += x;
      }
      unsigned incl = run;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const unsigned o = __shfl_up_sync(0xffffffffu, incl, m);
        if (lane >= m) incl += o;
      }
      const unsigned ex = carry + incl - run;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + lane * 8 + u;
        if (i < f.n_tiles) Pt[(size_t)c * f.n_tiles + i] = (int)(ex + v[u]);
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) T[c] = (int)carry;
  }
  __syncthreads();
  const bool slot_prio = f.prio == MOE_PRIO_SLOT;
  // per-expert requests (load), padding counts, and this CTA's share of the
  // load[] stores and of the empty slot_src entries
  for (int e = threadIdx.x; e < a.E; e += blockDim.x) {
    int ld = 0;
    if (slot_prio)
      for (int j = 0; j < a.k; ++j) ld += T[j * a.E + e];
    else
      ld = T[e];
    s_cnt[e] = a.cap - min(ld, a.cap);
  }
  __syncthreads();
  for (int e = blockIdx.x * kRowWarps + warp; e < a.E; e += gridDim.x * kRowWarps) {
    const int ld = a.cap - s_cnt[e] < a.cap ? a.cap - s_cnt[e] : a.cap;  // min(load, cap)
    if (lane == 0) {
      int full = 0;
      if (slot_prio)
        for (int j = 0; j < a.k; ++j) full += T[j * a.E + e];
      else
        full = T[e];
      f.load[e] = full;
    }
    if (f.slot_src)
      for (int s = ld + lane; s < a.cap; s += 32) f.slot_src[(size_t)e * a.cap + s] = -1;
  }
  if (threadIdx.x < 32) {
    int carry = 0;
    for (int base = 0; base < a.E; base += 32) {
      const int e = base + lane;
      const int v = e < a.E ? s_cnt[e] : 0;
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

  const int gw = blockIdx.x * kRowWarps + warp, nw = gridDim.x * kRowWarps;
  for (int t = gw; t < a.S; t += nw) {
    // finish the token's slots: lane j owns item t*k + j
    int my_e = -1, my_s = -1;
    if (lane < a.k) {
      const size_t gi = (size_t)t * a.k + lane;
      const int e = a.expert_idx[gi];
      if (e >= 0) {
        const int tile = t / f.tile_tokens;
        const int col = slot_prio ? lane * a.E + e : e;
        int s = f.slot_idx[gi] +
                (f.scanned ? (int)__ldcg(f.agg + (size_t)col * f.n_tiles + tile)
                           : Pt[(size_t)col * f.n_tiles + tile]);
        if (slot_prio)
          for (int jj = 0; jj < lane; ++jj) s += T[jj * a.E + e];
        if (s < a.cap) {
          if (f.slot_src) f.slot_src[(size_t)e * a.cap + s] = (int)gi;
        } else {
          s = -1;
          f.weight[gi] = 0.f;
        }
        f.slot_idx[gi] = s;
        my_e = e;
        my_s = s;
      }
    }
    const char* srow = a.src + (size_t)t * a.row_bytes;
    for (int seg = 0; seg < a.row_bytes; seg += SEG) {
      V8 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int off = seg + (lane + 32 * u) * VB;
        if (off < a.row_bytes) r[u] = ld_stream_v8(srow + off);
      }
      for (int j = 0; j < a.k; ++j) {
        const int s = __shfl_sync(0xffffffffu, my_s, j);
        if (s < 0) continue;
        char* drow = dst_row_of(a, __shfl_sync(0xffffffffu, my_e, j), s);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int off = seg + (lane + 32 * u) * VB;
          if (off < a.row_bytes) st_v8(drow + off, r[u]);
        }
      }
    }
  }
  // zero padding rows
  const int npad = s_beg[a.E];
  const V8 z = V8{{0, 0, 0, 0, 0, 0, 0, 0}};
  for (int p = gw; p < npad; p += nw) {
    int lo = 0, hi = a.E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_beg[mid] <= p) lo = mid; else hi = mid - 1;
    }
    char* drow = dst_row_of(a, lo, a.cap - s_cnt[lo] + (p - s_beg[lo]));
    for (int off = lane * VB; off < a.row_bytes; off += 32 * VB) st_v8(drow + off, z);
  }
  if (a.sys_fence) __threadfence_system();
}

moe_status_t layout_fin_launch(const moe_gate_desc_t& d, const moe_routing_t& r, const void* x,
                               int dtype_size, int dcols, const PeerPtrs& dst, int E_local,
                               int rank, const GateFinalize& fin, cudaStream_t stream) {
  RowArgs a{};
  a.src = static_cast<const char*>(x);
  a.expert_idx = r.expert_idx;
  a.slot_idx = r.slot_idx;
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
  const size_t smem = sizeof(int) * ((size_t)fin.ncols + (fin.scanned ? 0 : (size_t)fin.ncols * fin.n_tiles));
  const void* kern = a.row_bytes > 2048 ? (const void*)k_layout_fin<4> : (const void*)k_layout_fin<2>;
  if (smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "moe_gate_layout: smem attribute");
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowThreads, smem);
  const int grid = std::max(1, per_sm) * device_sm_count();
  void* args[] = {&a, (void*)&fin};
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(kRowThreads), smem, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_gate_layout: k_layout_fin launch");
  return MOE_OK;
}

// ------------------------------------------------------------ Layout_Transform, TMA
// The same contract as k_layout, with the rows moved by the copy engine
// instead of registers: every warp is an independent pipeline whose lane 0
// bulk-loads x rows into a ring of NS shared-memory stages
// (cp.async.bulk global->shared, mbarrier completion; SASS UBLKCP) and
// bulk-stores each staged row to its <= k destinations (cp.async.bulk
// shared->global, bulk groups).  A stage is reloaded once the stores issued
// kTmaLag tasks ago have finished READING it, so NS - kTmaLag loads and
// kTmaLag store groups are in flight per warp without a single register of
// payload: bytes in flight per SM are set by shared memory, not by occupancy.
// Each warp owns one contiguous range of the task list (x rows, then the
// zero padding rows, which are bulk-stored from a zeroed shared row).  The
// routing of 32 tasks is fetched at once (lane l: task base + l) and
// broadcast with shuffles, so lane 0 never waits on an index load.
constexpr int kTmaWarps = 4;
constexpr int kTmaThreads = kTmaWarps * 32;
constexpr int kTmaLag = 2;
constexpr int kTmaMaxK = 4;  // destinations fetched per lane; larger k reads the rest inline

struct TmaArgs {
  RowArgs a;
  int ns;  // stages per warp
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, unsigned src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ char* dst_row(const RowArgs& a, int e, int s) { return dst_row_of(a, e, s); }

__global__ void __launch_bounds__(kTmaThreads) k_layout_tma(TmaArgs ta) {
  const RowArgs& a = ta.a;
  const int NS = ta.ns;
  extern __shared__ __align__(128) char smem[];
  __shared__ int s_beg[257];
  __shared__ __align__(8) unsigned long long s_bar[kTmaWarps * 16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned rb = (unsigned)a.row_bytes;
  char* zero_row = smem;  // [row], then [warps][NS][row] stages
  char* stages = smem + rb;
  for (unsigned o = threadIdx.x * 16; o < rb; o += kTmaThreads * 16)
    *reinterpret_cast<uint4*>(zero_row + o) = make_uint4(0, 0, 0, 0);
  if (lane == 0)
    for (int s = 0; s < NS; ++s) mbar_init(smem_u32(&s_bar[warp * 16 + s]), 1);
  // generic-proxy zeros and barrier inits must be visible to the async proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  pdl_wait();  // routing comes from moe_gate
  pdl_trigger();
  pad_prefix(a, s_beg);  // ends with __syncthreads (also publishes the above)

  const long long n_tasks = (long long)a.S + s_beg[a.E];
  const long long gw = (long long)blockIdx.x * kTmaWarps + warp, GW = (long long)gridDim.x * kTmaWarps;
  const long long beg = n_tasks * gw / GW, end = n_tasks * (gw + 1) / GW;
  const long long tok_end = min(end, (long long)a.S);
  const int ntok = tok_end > beg ? (int)(tok_end - beg) : 0;  // x rows of this warp
  const unsigned st0 = smem_u32(stages + (size_t)warp * NS * rb);
  const unsigned bar0 = smem_u32(&s_bar[warp * 16]);

  // prologue: the first NS x rows
  if (lane == 0)
    for (int o = 0; o < min(NS, ntok); ++o)
      bulk_load(st0 + o * rb, a.src + (size_t)(beg + o) * rb, rb, bar0 + 8 * o);

  int ord = 0;  // x-row ordinal of the store cursor
  for (long long base = beg; base < end; base += 32) {
    // routing of tasks base .. base+31, one task per lane
    const long long my = base + lane;
    char* dst[kTmaMaxK];
#pragma unroll
    for (int j = 0; j < kTmaMaxK; ++j) dst[j] = nullptr;
    if (my < end) {
      if (my < a.S) {
        const int t = (int)my;
#pragma unroll
        for (int j = 0; j < kTmaMaxK; ++j) {
          if (j < a.k) {
            const int s = __ldg(a.slot_idx + (size_t)t * a.k + j);
            if (s >= 0) {
              const int e = __ldg(a.expert_idx + (size_t)t * a.k + j);
              if (j == 0 || !dedupe_row(a, t, j, e, s, 0)) dst[j] = dst_row(a, e, s);
            }
          }
        }
      } else {
        const int p = (int)(my - a.S);
        int lo = 0, hi = a.E - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_beg[mid] <= p) lo = mid; else hi = mid - 1;
        }
        dst[0] = dst_row(a, lo, min(__ldg(a.load + lo), a.cap) + (p - s_beg[lo]));
      }
    }
    const int cnt = (int)min(32LL, end - base);
    for (int u = 0; u < cnt; ++u) {
      char* d[kTmaMaxK];
#pragma unroll
      for (int j = 0; j < kTmaMaxK; ++j)
        d[j] = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst[j]), u));
      if (lane == 0) {
        const long long task = base + u;
        if (task < a.S) {
          const int st = ord % NS;
          mbar_wait(bar0 + 8 * st, (unsigned)(ord / NS) & 1u);
          const unsigned src = st0 + st * rb;
#pragma unroll
          for (int j = 0; j < kTmaMaxK; ++j)
            if (d[j]) bulk_store(d[j], src, rb);
          for (int j = kTmaMaxK; j < a.k; ++j) {  // k > kTmaMaxK (rare)
            const int t = (int)task;
            const int s = __ldg(a.slot_idx + (size_t)t * a.k + j);
            if (s >= 0) bulk_store(dst_row(a, __ldg(a.expert_idx + (size_t)t * a.k + j), s), src, rb);
          }
          bulk_commit();
          // the stage of ordinal ord - kTmaLag is free once its stores have read it
          const int o2 = ord - kTmaLag;
          if (o2 >= 0 && o2 + NS < ntok) {
            bulk_wait_read<kTmaLag>();
            const int st2 = o2 % NS;
            bulk_load(st0 + st2 * rb, a.src + (size_t)(beg + o2 + NS) * rb, rb, bar0 + 8 * st2);
          }
          ++ord;
        } else {
          bulk_store(d[0], smem_u32(zero_row), rb);
          bulk_commit();
        }
      }
    }
  }
  if (lane == 0) bulk_wait_all();
  if (a.sys_fence) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence_system();
  }
}

// ------------------------------------------------------------ Reverse + combine
template <int DT, int U>
__global__ void __launch_bounds__(kRowThreads) k_reverse(RowArgs a) {
  constexpr int VB = 32;
  constexpr int NA = DT == MOE_F32 ? 8 : 16;  // accumulators per vector
  constexpr int SEG = 32 * U * VB;
  const int lane = threadIdx.x & 31;
  const int wstride = gridDim.x * kRowWarps;
  pdl_wait();     // expert outputs come from the AllToAll / the layout
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
  for (int tb = (blockIdx.x * kRowWarps + (threadIdx.x >> 5)) * TPW; tb < a.S; tb += wstride) {
    const char* b[TPW][KK];
    float w[TPW][KK];
#pragma unroll
    for (int p = 0; p < TPW; ++p)
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
            if (a.y_ef) st_v8_ef(yrow + off, pack_vec<DT>(acc));
            else st_v8(yrow + off, pack_vec<DT>(acc));
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------ Reverse, TMA
// The combine with the k admitted rows of a token brought into shared memory
// by the copy engine: each warp is an independent pipeline over a contiguous
// token range.  Lane 0 bulk-loads the token's rows (cp.async.bulk, one
// mbarrier per stage with the summed expect_tx) up to NS tokens ahead; the
// whole warp then accumulates from shared memory in fp32 (ascending j from
// 0, the same order as k_reverse) and stores y with 32-byte vectors.  The
// routing of 32 tokens is fetched at once (lane l: token base + l) and
// handed to lane 0 by shuffles.  Meant for the NVLink combine, where the
// rows come from peers' memory: bytes in flight are set by shared memory.
constexpr int kRevTmaMaxK = 4;

template <int DT>
__global__ void __launch_bounds__(kTmaThreads) k_reverse_tma(TmaArgs ta) {
  const RowArgs& a = ta.a;
  const int NS = ta.ns;
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long s_bar[kTmaWarps * 16];
  __shared__ float s_w[kTmaWarps][16][kRevTmaMaxK];  // per stage: weights (0 = no row)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned rb = (unsigned)a.row_bytes, sb = rb * a.k;  // stage bytes
  if (lane == 0)
    for (int s = 0; s < NS; ++s) mbar_init(smem_u32(&s_bar[warp * 16 + s]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  pdl_wait();
  pdl_trigger();
  const long long gw = (long long)blockIdx.x * kTmaWarps + warp, GW = (long long)gridDim.x * kTmaWarps;
  const int beg = (int)((long long)a.S * gw / GW), end = (int)((long long)a.S * (gw + 1) / GW);
  const int ntok = end - beg;
  char* stages = smem + (size_t)warp * NS * sb;
  const unsigned st0 = smem_u32(stages), bar0 = smem_u32(&s_bar[warp * 16]);
  constexpr int NA = DT == MOE_F32 ? 8 : 16;

  // routing of the current issue batch: lane l holds token (ibase + l)
  const char* src[kRevTmaMaxK];
  float wt[kRevTmaMaxK];
  int ibase = -32;
  int issued = 0;
  for (int o = 0; o < ntok; ++o) {
    // keep up to NS tokens issued ahead of the consumer
    while (issued < ntok && issued < o + NS) {
      if (issued >= ibase + 32) {  // next routing batch (warp-uniform)
        ibase = issued;
        const int tl = beg + ibase + lane;
        const int t = a.rev ? a.S - 1 - tl : tl;  // rev: last tokens first (L2 reuse)
#pragma unroll
        for (int j = 0; j < kRevTmaMaxK; ++j) {
          src[j] = nullptr;
          wt[j] = 0.f;
          if (j < a.k && tl < end) {
            const int sl = __ldg(a.slot_idx + (size_t)t * a.k + j);
            if (sl >= 0) {
              src[j] = src_row_item(a, t, j, __ldg(a.expert_idx + (size_t)t * a.k + j), sl);
              wt[j] = row_weight(a, (size_t)t * a.k + j);
            }
          }
        }
      }
      const int from = issued - ibase;
      const int st = issued % NS;
      unsigned nrows = 0;
      const char* ps[kRevTmaMaxK];
#pragma unroll
      for (int j = 0; j < kRevTmaMaxK; ++j) {
        ps[j] = reinterpret_cast<const char*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(src[j]), from));
        const float w = __shfl_sync(0xffffffffu, wt[j], from);
        if (lane == 0) s_w[warp][st][j] = ps[j] ? w : 0.f;
        nrows += ps[j] ? 1u : 0u;
      }
      if (lane == 0) {
        const unsigned bar = bar0 + 8 * st;
        if (nrows == 0) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
        } else {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                       "r"(nrows * rb)
                       : "memory");
#pragma unroll
          for (int j = 0; j < kRevTmaMaxK; ++j)
            if (ps[j])
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                  ::"r"(st0 + st * sb + j * rb), "l"(ps[j]), "r"(rb), "r"(bar)
                  : "memory");
        }
      }
      ++issued;
    }
    __syncwarp();
    const int st = o % NS;
    mbar_wait(bar0 + 8 * st, (unsigned)(o / NS) & 1u);
    const char* stage = stages + (size_t)st * sb;
    char* yrow = a.dst + (size_t)(a.rev ? a.S - 1 - (beg + o) : beg + o) * rb;
    for (unsigned off = lane * 32u; off < rb; off += 32u * 32u) {
      float acc[NA];
#pragma unroll
      for (int q = 0; q < NA; ++q) acc[q] = 0.f;
      for (int j = 0; j < a.k; ++j) {
        const float w = s_w[warp][st][j];
        // a dropped slot has no row; a zero weight adds an exact +0 (acc
        // starts at +0), so skipping it leaves the same bits
        if (w == 0.f) continue;
        const V4* v4 = reinterpret_cast<const V4*>(stage + j * rb + off);
        V8 v;
        const V4 lo = v4[0], hi = v4[1];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v.w[q] = lo.w[q];
          v.w[q + 4] = hi.w[q];
        }
        fma_vec<DT>(acc, w, v);
      }
      if (a.y_ef) st_v8_ef(yrow + off, pack_vec<DT>(acc));
      else st_v8(yrow + off, pack_vec<DT>(acc));
    }
    __syncwarp();  // every lane done with the stage before lane 0 refills it
  }
}

// 16-byte fallback of the combine for rows that are not a multiple of 32 B.
template <int DT>
__global__ void __launch_bounds__(kRowThreads) k_reverse16(RowArgs a) {
  const int lane = threadIdx.x & 31;
  const int wstride = gridDim.x * kRowWarps;
  constexpr int NA = DT == MOE_F32 ? 4 : 8;
  pdl_wait();
  pdl_trigger();
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

moe_status_t layout_launch_peers(const moe_gate_desc_t& d, const moe_routing_t& r, const void* x,
                                 int dtype_size, int dcols, const PeerPtrs& dst, int E_local,
                                 int rank, cudaStream_t stream, const int32_t* offsets,
                                 const int32_t* peer_base, const PeerPtrs* pad_tab,
                                 const PeerPtrs* dup_tab) {
  RowArgs a{};
  if (dup_tab && !offsets) {
    a.dedupe = 1;
    a.dup = *dup_tab;
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
  a.prefetch = env_int("MOE_LAYOUT_PREFETCH", 0);  // measured slower (C2 +3 us, C3 +11 us): off
  // padding rows first when they are many (C4b: combine 46.2 -> 42.0 us,
  // its adjoint likewise; C3's 2% gained nothing)
  a.pads_first = env_int("MOE_LAYOUT_PADS_FIRST", E_local == d.E && pad_heavy(d) ? 1 : 0);
  // TMA pipeline: rows of 16-byte multiples with >= 2 stages per warp in a
  // ~100 KB per-CTA budget (two CTAs per SM)
  // TMA bulk stores: slower than the register path into local HBM, and
  // (re-measured at P=2 with the current barrier and dedupe) over NVLink
  // too (C2 121.2 vs 117.5 us, C3 120.8 vs 118.1, C4b 129.9 vs 124.4): off
  const int tma_env = a.sys_fence ? env_int("MOE_P2P_LAYOUT_TMA", 0) : env_int("MOE_LAYOUT_TMA", 0);
  const int budget = env_int("MOE_LAYOUT_TMA_SMEM", 100 * 1024);
  const int ns = std::min(16, (budget - a.row_bytes) / (kTmaWarps * std::max(1, a.row_bytes)));
  if (tma_env && a.row_bytes % 16 == 0 && ns >= 2) {
    TmaArgs ta{a, ns};
    const size_t smem = (size_t)a.row_bytes * (1 + kTmaWarps * ns);
    cudaError_t e = cudaFuncSetAttribute((const void*)k_layout_tma,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "moe_layout: smem attribute");
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_layout_tma, kTmaThreads, smem);
    const int occ = env_int("MOE_LAYOUT_CTAS_PER_SM", 0);
    const int grid = (occ > 0 ? occ : std::max(1, per_sm)) * device_sm_count();
    void* args[] = {&ta};
    e = launch_pdl((const void*)k_layout_tma, dim3(grid), dim3(kTmaThreads), smem, stream, args);
    if (e != cudaSuccess) return cuda_status(e, "moe_layout: k_layout_tma launch");
    return MOE_OK;
  }
  const void* kern;
  const int LT = env_int("MOE_LAYOUT_TPW", 0);  // measured: no gain over k_layout<32,4>;  // TPW * U = 4 vectors in flight per lane
  if (a.row_bytes % 32 == 0 && LT) {
    const int segs = std::max(1, a.row_bytes / 1024);
    kern = segs >= 4 ? (const void*)k_layout_t<4, 1>
           : segs >= 2 ? (const void*)k_layout_t<2, 2> : (const void*)k_layout_t<1, 4>;
  } else if (a.row_bytes % 32 == 0)
  {
    // measured: 2 KiB segments for rows <= 2 KiB (C2 36.3 -> 35.4 us)
    const int lu = env_int("MOE_LAYOUT_U", a.row_bytes <= 2048 ? 2 : 4);
    kern = lu == 1 ? (const void*)k_layout<32, 1> : lu == 2 ? (const void*)k_layout<32, 2>
                                                            : (const void*)k_layout<32, 4>;
  }
  else
    kern = (const void*)k_layout<16, 4>;
  void* args[] = {&a};
  const int occ = env_int("MOE_LAYOUT_CTAS_PER_SM", 0);
  const int grid = occ > 0 ? occ * device_sm_count() : row_grid(kern);
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
                                  int dup_alias) {
  RowArgs a{};
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
  const int local_dflt = E_local == d.E ? 1 : 0;
  a.rev = env_int("MOE_REVERSE_BACKWARDS", local_dflt);
  a.y_ef = env_int("MOE_REVERSE_Y_EF", local_dflt);
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
  // TMA-staged combine (peer mode by default: rows come over NVLink)
  {
    const bool peer = E_local != d.E;
    // measured: TMA staging won for Switch (k = 1) on >= 4 KiB rows in the
    // forward walk (C3: 48.5 vs 49.8 us) but not with the reversed walk,
    // where the register path finds the dispatch in L2 (C3: 40.0 vs 52.3 us);
    // it loses on 2 KiB rows (C4b: 69 vs 53 us) and over NVLink.  Off.
    const int tma_dflt = (!peer && a.k == 1 && a.row_bytes >= 4096 && !a.rev) ? 1 : 0;
    const int tma = peer ? env_int("MOE_P2P_REVERSE_TMA", 0) : env_int("MOE_REVERSE_TMA", tma_dflt);
    const int budget = env_int("MOE_REVERSE_TMA_SMEM", 100 * 1024);
    const int ns = std::min(16, budget / (kTmaWarps * std::max(1, a.row_bytes * a.k)));
    if (tma && a.row_bytes % 32 == 0 && a.k <= kRevTmaMaxK && ns >= 2) {
      TmaArgs ta{a, ns};
      const size_t smem = (size_t)a.row_bytes * a.k * kTmaWarps * ns;
      const void* kt = dtype == MOE_F32 ? (const void*)k_reverse_tma<MOE_F32>
                                        : (const void*)k_reverse_tma<MOE_BF16>;
      cudaError_t e = cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return cuda_status(e, "moe_reverse_layout: smem attribute");
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kt, kTmaThreads, smem);
      const int grid = std::max(1, per_sm) * device_sm_count();
      void* args[] = {&ta};
      e = launch_pdl(kt, dim3(grid), dim3(kTmaThreads), smem, stream, args);
      if (e != cudaSuccess) return cuda_status(e, "moe_reverse_layout: k_reverse_tma launch");
      return MOE_OK;
    }
  }
  const void* kern;
  const int U = env_int("MOE_REVERSE_U", 1);
  // k <= 2 path: vectors per lane per round (x k rows); measured: 2 for
  // k = 2 (one 1 KiB segment of both rows: C2 36.3 -> 35.6 us), 4 for k = 1
  // (peer mode: 4 -- both 2 KiB rows in flight hide the NVLink latency better,
  // C2 at P=2: 129.2 -> 127.3 us)
  const int KU = env_int("MOE_REVERSE_KU", (d.k == 2 && E_local == d.E) ? 2 : 4);
  const bool v16 = env_int("MOE_REVERSE_V16", 0) != 0;  // force 16-byte vectors (experiment)
  const bool kspec = !v16 && env_int("MOE_REVERSE_KSPEC", 1) && a.row_bytes % 32 == 0 && a.k <= 2;
  if (kspec) {
    // TPW * k * U = KU (default 4) vectors in flight per lane, U covering at
    // most one row (1 KiB of row per U step)
    const bool f = dtype == MOE_F32;
    const int segs = std::max(1, a.row_bytes / 1024);  // 1 KiB per U step
    const int per = std::max(1, KU / a.k);                // U * TPW
    const int Uc = std::min(per, segs) >= 4 ? 4 : std::min(per, segs) >= 2 ? 2 : 1;
    // two tokens per warp round for Switch on <= 2 KiB rows (C4b: 51.3 vs
    // 53.5 us); no gain for k = 2
    const int tpw_dflt = (a.k == 1 && a.row_bytes <= 2048) ? 1 : 0;
    const int T = env_int("MOE_REVERSE_TPW", tpw_dflt) ? std::max(1, per / Uc) : 1;
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
  } else if (a.row_bytes % 32 == 0 && !v16) {
    if (U == 1)
      kern = dtype == MOE_F32 ? (const void*)k_reverse<MOE_F32, 1> : (const void*)k_reverse<MOE_BF16, 1>;
    else
      kern = dtype == MOE_F32 ? (const void*)k_reverse<MOE_F32, 2> : (const void*)k_reverse<MOE_BF16, 2>;
  } else {
    kern = dtype == MOE_F32 ? (const void*)k_reverse16<MOE_F32> : (const void*)k_reverse16<MOE_BF16>;
  }
  void* args[] = {&a};
  const int occ = env_int(E_local != d.E ? "MOE_COMBINE_CTAS_PER_SM" : "MOE_REVERSE_CTAS_PER_SM", 0);
  const int grid = occ > 0 ? occ * device_sm_count() : row_grid(kern);
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(kRowThreads), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_reverse_layout: launch");
  return MOE_OK;
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

}  // namespace moe
