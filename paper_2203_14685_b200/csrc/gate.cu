// gate.cu -- moe_gate: Step 1 of Algorithm 1 on given gate
// logits, fused with capacity slot assignment.
//
// One CTA per tile of tokens; the tile id comes from an atomic ticket, so a
// CTA only ever waits on tiles already claimed by running CTAs (look-back
// always makes progress, whatever else occupies the SMs).
//
//   Phase A  selection + weights (Eq. 1, 123-124, 144-145)
//            L lanes per token; each lane keeps a register top-K of its E/L
//            logits, a shfl_xor butterfly merges the lists (comparator:
//            larger raw fp32 logit, then lower index -- R2, R3).  k > 8 uses
//            a rank-counting path.  Weights are evaluated in fp64 and rounded
//            once to fp32 (R1).
//   Phase B  capacity (R4-R6): in-tile ranks of each item among earlier
//            items of the same expert column (__match_any_sync, 32 items at a
//            time, per-warp histograms), then a decoupled look-back across
//            tiles per column: 64-bit status words (epoch | flag | value)
//            that carry their own payload, so relaxed gpu-scope stores and
//            loads suffice (no fences on the critical path).  slot =
//            tiles-before + warps-before + rank-in-warp; >= cap -> dropped.
//            SLOT priority (j-major) runs the same scan per (j, e) column and
//            k_gate_slot_finalize adds the totals of earlier j afterwards.
#include <cfloat>
#include <climits>

#include "common.cuh"

namespace moe {

constexpr int kGateThreads = 256;
constexpr int kGateWarps = kGateThreads / 32;
constexpr int kMaxTileItems = 2048;  // tile_tokens * k
constexpr int kMaxCols = 2048;       // look-back columns: E or k*E
constexpr size_t kMaxTileLogitBytes = 64 * 1024;
constexpr unsigned kValMask = (1u << 30) - 1;  // counts < 2^30 (S*k < 2^30, checked)

struct GateCtrl {  // 64 bytes at the head of the workspace
  unsigned ticket, done, epoch, bad;
  unsigned pad[12];
};

struct GateArgs {
  const float* logits;
  const int32_t* ids;
  const int32_t* table;
  int vocab;
  int S, E, k, cap, mode, prio;
  int tile_tokens, n_tiles, ncols;
  int lg_words;  // shared-memory words of the staged logits tile (16-byte multiple)
  int32_t* expert_idx;
  int32_t* slot_idx;
  float* weight;
  int32_t* load;
  int32_t* slot_src;
  GateCtrl* ctrl;
  unsigned long long* status;  // [ncols][n_tiles] (column-major: warp look-back)
  int32_t* totals;             // [ncols] (SLOT priority)
  unsigned long long* trace;   // [n_tiles][8] globaltimer stamps (MOE_GATE_TRACE builds)
};

#ifdef MOE_GATE_TRACE
#define GATE_TRACE(k)                                                         \
  do {                                                                        \
    if (threadIdx.x == 0) {                                                   \
      unsigned long long _t;                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                  \
      a.trace[(size_t)s_tile * 8 + (k)] = _t;                                 \
    }                                                                         \
  } while (0)
#else
#define GATE_TRACE(k) \
  do {                \
  } while (0)
#endif

// ------------------------------------------------------------ layout of ws
struct GatePlan {
  int L, K, tile_tokens, n_tiles, ncols, lg_words;
  size_t status_off, totals_off, bytes, smem, trace_off;
};

static int choose_lanes(int E) {
  int L = 1;
  while (L * 2 <= 32 && E % (L * 2) == 0 && E / (L * 2) >= 8) L *= 2;
  return L;
}

static GatePlan gate_plan(const moe_gate_desc_t& d) {
  GatePlan p{};
  p.L = d.kind == MOE_GATE_HASH ? 1 : choose_lanes(d.E);
  p.K = d.k <= 1 ? 1 : d.k <= 2 ? 2 : d.k <= 4 ? 4 : d.k <= 8 ? 8 : 0;
  // >= 256 tiles when S allows (about 1.7 CTAs per SM on 148 SMs), tiles of
  // 32..256 tokens, at most kMaxTileItems items per tile
  int tt = 256;
  while (tt > 32 && (d.S + tt - 1) / tt < 256) tt >>= 1;
  while (tt > 1 && tt * d.k > kMaxTileItems) tt >>= 1;
  // the staged logits tile stays within kMaxTileLogitBytes of shared memory
  if (d.kind != MOE_GATE_HASH)
    while (tt > 1 && (size_t)tt * d.E * 4 > kMaxTileLogitBytes) tt >>= 1;
  p.tile_tokens = tt;
  p.n_tiles = (d.S + tt - 1) / tt;
  p.ncols = d.priority == MOE_PRIO_SLOT ? d.k * d.E : d.E;
  p.status_off = sizeof(GateCtrl);
  p.totals_off = p.status_off + sizeof(unsigned long long) * (size_t)p.n_tiles * p.ncols;
  p.bytes = p.totals_off + sizeof(int32_t) * (size_t)p.ncols;
  p.bytes = (p.bytes + 255) & ~(size_t)255;
#ifdef MOE_GATE_TRACE
  p.trace_off = p.bytes;
  p.bytes += sizeof(unsigned long long) * 8 * (size_t)p.n_tiles;
#endif
  size_t items = (size_t)tt * d.k;
  p.lg_words = d.kind == MOE_GATE_HASH ? 0 : ((tt * d.E + 3) & ~3);
  p.smem = sizeof(int) * (p.lg_words + 2 * items + (size_t)(kGateWarps + 2) * p.ncols);
  return p;
}

// ------------------------------------------------------------ selection
__device__ __forceinline__ bool beats(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

template <int K>
struct TopList {
  float v[K];
  int i[K];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int p = 0; p < K; ++p) {
      v[p] = -INFINITY;
      i[p] = INT_MAX;
    }
  }
  __device__ __forceinline__ void insert(float x, int e) {
    if (!beats(x, e, v[K - 1], i[K - 1])) return;
    v[K - 1] = x;
    i[K - 1] = e;
#pragma unroll
    for (int p = K - 1; p > 0; --p) {
      if (beats(v[p], i[p], v[p - 1], i[p - 1])) {
        float tv = v[p];
        v[p] = v[p - 1];
        v[p - 1] = tv;
        int ti = i[p];
        i[p] = i[p - 1];
        i[p - 1] = ti;
      }
    }
  }
};

// Visit the E/L logits of lane `l` of one token row (in shared memory):
// f(value, expert).
template <typename F>
__device__ __forceinline__ void for_lane_logits(const float* row, int l, int epl, bool vec4,
                                                F&& f) {
  const int base = l * epl;
  if (vec4) {
    const float4* r4 = reinterpret_cast<const float4*>(row + base);
    for (int q = 0; q < epl / 4; ++q) {
      float4 x = r4[q];
      f(x.x, base + 4 * q);
      f(x.y, base + 4 * q + 1);
      f(x.z, base + 4 * q + 2);
      f(x.w, base + 4 * q + 3);
    }
  } else {
    for (int q = 0; q < epl; ++q) f(row[base + q], base + q);
  }
}

template <int L>
__device__ __forceinline__ double group_sum(double x) {
#pragma unroll
  for (int m = 1; m < L; m <<= 1) x += __shfl_xor_sync(0xffffffffu, x, m);
  return x;
}
template <int L>
__device__ __forceinline__ float group_max(float x) {
#pragma unroll
  for (int m = 1; m < L; m <<= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, m));
  return x;
}

// Top-k (Eq. 1), register path, K >= k.
template <int L, int K>
__device__ __forceinline__ void select_topk_reg(const GateArgs& a, const float* row, int t,
                                                bool valid, int l, int epl, bool vec4,
                                                int* s_sel /*[k]*/) {
  TopList<K> top;
  top.init();
  if (valid) for_lane_logits(row, l, epl, vec4, [&](float x, int e) { top.insert(x, e); });
#pragma unroll
  for (int m = 1; m < L; m <<= 1) {
    // snapshot the partner's whole list first: both lanes mutate their own
    float ov[K];
    int oi[K];
#pragma unroll
    for (int p = 0; p < K; ++p) {
      ov[p] = __shfl_xor_sync(0xffffffffu, top.v[p], m);
      oi[p] = __shfl_xor_sync(0xffffffffu, top.i[p], m);
    }
#pragma unroll
    for (int p = 0; p < K; ++p) top.insert(ov[p], oi[p]);
  }
  // weights in fp64 (R1); m = the row maximum = top.v[0], exp(0) = 1 exactly
  const double mx = (double)top.v[0];
  double ex[K];
  ex[0] = 1.0;
#pragma unroll
  for (int p = 1; p < K; ++p) ex[p] = (p < a.k) ? exp((double)top.v[p] - mx) : 0.0;
  double den = 0.0;
  if (a.mode == MOE_W_SOFTMAX) {
    double part = 0.0;
    if (valid) for_lane_logits(row, l, epl, vec4, [&](float x, int) { part += exp((double)x - mx); });
    den = group_sum<L>(part);
  } else {
#pragma unroll
    for (int p = 0; p < K; ++p) den += ex[p];
  }
  if (valid && l == 0) {
    const size_t o = (size_t)t * a.k;
#pragma unroll
    for (int p = 0; p < K; ++p) {
      if (p < a.k) {
        a.expert_idx[o + p] = top.i[p];
        a.weight[o + p] = (float)(ex[p] / den);
        s_sel[p] = top.i[p];
      }
    }
  }
}

// k-top-1 (R11), register path, K >= k prototypes.
template <int L, int K>
__device__ __forceinline__ void select_ktop1_reg(const GateArgs& a, const float* row, int t,
                                                 bool valid, int l, int epl, bool vec4,
                                                 int* s_sel) {
  const int n = a.E / a.k;
  float bv[K];
  int bi[K];
#pragma unroll
  for (int p = 0; p < K; ++p) {
    bv[p] = -INFINITY;
    bi[p] = INT_MAX;
  }
  if (valid)
    for_lane_logits(row, l, epl, vec4, [&](float x, int e) {
      const int pe = e / n;
#pragma unroll
      for (int p = 0; p < K; ++p)
        if (p == pe && beats(x, e, bv[p], bi[p])) {
          bv[p] = x;
          bi[p] = e;
        }
    });
#pragma unroll
  for (int m = 1; m < L; m <<= 1) {
#pragma unroll
    for (int p = 0; p < K; ++p) {
      float ov = __shfl_xor_sync(0xffffffffu, bv[p], m);
      int oi = __shfl_xor_sync(0xffffffffu, bi[p], m);
      if (beats(ov, oi, bv[p], bi[p])) {
        bv[p] = ov;
        bi[p] = oi;
      }
    }
  }
  double den[K];
#pragma unroll
  for (int p = 0; p < K; ++p) den[p] = 1.0;
  if (a.mode == MOE_W_SOFTMAX) {
    double part[K];
#pragma unroll
    for (int p = 0; p < K; ++p) part[p] = 0.0;
    if (valid)
      for_lane_logits(row, l, epl, vec4, [&](float x, int e) {
        const int pe = e / n;
#pragma unroll
        for (int p = 0; p < K; ++p)
          if (p == pe) part[p] += exp((double)x - (double)bv[p]);
      });
#pragma unroll
    for (int p = 0; p < K; ++p) den[p] = group_sum<L>(part[p]);
  }
  if (valid && l == 0) {
    const size_t o = (size_t)t * a.k;
#pragma unroll
    for (int p = 0; p < K; ++p) {
      if (p < a.k) {
        a.expert_idx[o + p] = bi[p];
        a.weight[o + p] = (a.mode == MOE_W_SOFTMAX) ? (float)(1.0 / den[p]) : 1.0f;
        s_sel[p] = bi[p];
      }
    }
  }
}

// Rank-counting path for k > 8: element e is selected at slot j = the number
// of elements of its segment that beat it, if that is < k (top-k: segment =
// row; k-top-1: segment = its prototype slice, selected iff rank == 0).
template <int L, bool KTOP1>
__device__ __forceinline__ void select_rank(const GateArgs& a, const float* row, int t, bool valid,
                                            int l, int epl, int* s_sel) {
  const int n = KTOP1 ? a.E / a.k : a.E;
  float lmax = -INFINITY;
  if (valid)
    for (int q = 0; q < epl; ++q) lmax = fmaxf(lmax, row[l * epl + q]);
  const double mx = (double)group_max<L>(lmax);
  double part = 0.0;
  for (int q = 0; q < epl; ++q) {
    const int e = l * epl + q;
    if (!valid) break;
    const float x = row[e];
    const int seg = KTOP1 ? (e / n) * n : 0;
    int rank = 0;
    for (int u = seg; u < seg + n; ++u) rank += beats(row[u], u, x, e) ? 1 : 0;
    if (!KTOP1 && (a.mode == MOE_W_SOFTMAX || rank < a.k)) part += exp((double)x - mx);
  }
  const double den_topk = KTOP1 ? 1.0 : group_sum<L>(part);
  for (int q = 0; q < epl; ++q) {
    const int e = l * epl + q;
    if (!valid) break;
    const float x = row[e];
    const int seg = KTOP1 ? (e / n) * n : 0;
    int rank = 0;
    for (int u = seg; u < seg + n; ++u) rank += beats(row[u], u, x, e) ? 1 : 0;
    int j = -1;
    float w = 0.f;
    if (KTOP1) {
      if (rank == 0) {
        j = e / n;
        if (a.mode == MOE_W_SOFTMAX) {
          double den = 0.0;
          for (int u = seg; u < seg + n; ++u) den += exp((double)row[u] - (double)x);
          w = (float)(1.0 / den);
        } else {
          w = 1.0f;
        }
      }
    } else if (rank < a.k) {
      j = rank;
      w = (float)(exp((double)x - mx) / den_topk);
    }
    if (j >= 0) {
      a.expert_idx[(size_t)t * a.k + j] = e;
      a.weight[(size_t)t * a.k + j] = w;
      s_sel[j] = e;
    }
  }
}

// ------------------------------------------------------------ the kernel
enum { KIND_TOPK = 0, KIND_KTOP1 = 1, KIND_HASH = 2 };

template <int KIND, int L, int K>
__global__ void __launch_bounds__(kGateThreads) k_gate(GateArgs a) {
  extern __shared__ __align__(16) int smem[];
  const int items = a.tile_tokens * a.k;
  float* s_lg = reinterpret_cast<float*>(smem);  // [tile_tokens][E] staged logits
  int* s_exp = smem + a.lg_words;             // [items] expert of item tt*k+j
  int* s_rank = s_exp + items;                // [items] rank inside its warp
  int* s_hist = s_rank + items;               // [warps][ncols]
  int* s_excl = s_hist + kGateWarps * a.ncols;  // [ncols] tiles-before
  int* s_tot = s_excl + a.ncols;              // [ncols] aggregate, then inclusive
  __shared__ unsigned s_tile, s_epoch, s_bad;
  __shared__ __align__(8) unsigned long long s_mbar;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_wait();     // the producer of the logits / the previous step must be done
  pdl_trigger();  // moe_layout may launch now; it waits for our completion
  if (tid == 0) {
    s_tile = atomicAdd(&a.ctrl->ticket, 1u);
    s_epoch = *((volatile unsigned*)&a.ctrl->epoch) & 0x3FFFFFFFu;
    s_bad = 0;
  }
  for (int i = tid; i < items; i += kGateThreads) s_exp[i] = -1;
  for (int i = tid; i < kGateWarps * a.ncols; i += kGateThreads) s_hist[i] = 0;
  __syncthreads();
  GATE_TRACE(0);
  const int tile = (int)s_tile;
  const unsigned long long epoch = s_epoch;
  const int t0 = tile * a.tile_tokens;
  const int nt = min(a.tile_tokens, a.S - t0);
  if constexpr (KIND != KIND_HASH) {
    // Stage the tile's logits (nt*E contiguous floats) into shared memory
    // with one TMA bulk copy (one DRAM latency for the whole tile); the
    // sub-16-byte tail, if any, with plain loads.
    const unsigned bytes = (unsigned)nt * a.E * 4u, bulk = bytes & ~15u;
    const float* g = a.logits + (size_t)t0 * a.E;
    const unsigned mbar = (unsigned)__cvta_generic_to_shared(&s_mbar);
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bulk)
                   : "memory");
      const unsigned dst = (unsigned)__cvta_generic_to_shared(s_lg);
      for (unsigned o = 0; o < bulk; o += 65536u) {
        const unsigned n = min(65536u, bulk - o);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(dst + o), "l"(reinterpret_cast<const char*>(g) + o), "r"(n), "r"(mbar)
            : "memory");
      }
    }
    for (unsigned i = bulk / 4 + tid; i < bytes / 4; i += kGateThreads) s_lg[i] = __ldg(g + i);
    __syncthreads();  // mbarrier initialised before anyone waits on it
    unsigned done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(mbar)
          : "memory");
  }
  GATE_TRACE(1);

  // ---------------- Phase A: selection + weights
  if constexpr (KIND == KIND_HASH) {
    int nbad = 0;
    for (int tt = tid; tt < nt; tt += kGateThreads) {
      const int t = t0 + tt;
      const int id = __ldg(a.ids + t);
      int e = -1;
      if (id >= 0 && id < a.vocab) e = __ldg(a.table + id);
      if (e < 0 || e >= a.E) {
        e = -1;
        ++nbad;
      }
      a.expert_idx[t] = e;
      a.weight[t] = e < 0 ? 0.f : 1.f;
      s_exp[tt] = e;
    }
    if (nbad) atomicAdd(&s_bad, (unsigned)nbad);
  } else {
    const int g = tid / L, l = tid % L, groups = kGateThreads / L;
    const int epl = a.E / L;
    const bool vec4 = (a.E % 4 == 0) && (epl % 4 == 0);
    for (int base = 0; base < a.tile_tokens; base += groups) {
      const int tt = base + g;
      const bool valid = tt < nt;
      const int t = valid ? t0 + tt : 0;
      int* s_sel = s_exp + (size_t)tt * a.k;
      const float* row = s_lg + (size_t)(valid ? tt : 0) * a.E;
      if constexpr (K == 0) {
        select_rank<L, KIND == KIND_KTOP1>(a, row, t, valid, l, epl, s_sel);
      } else if constexpr (KIND == KIND_TOPK) {
        select_topk_reg<L, K>(a, row, t, valid, l, epl, vec4, s_sel);
      } else {
        select_ktop1_reg<L, K>(a, row, t, valid, l, epl, vec4, s_sel);
      }
    }
  }
  __syncthreads();

  GATE_TRACE(2);
  // ---------------- Phase B1: ranks inside the tile, per warp
  const bool slot_prio = a.prio == MOE_PRIO_SLOT;
  const int per = (items + kGateWarps - 1) / kGateWarps;
  {
    const int wbeg = warp * per, wend = min(items, wbeg + per);
    int* hist = s_hist + warp * a.ncols;
    for (int base = wbeg; base < wend; base += 32) {
      const int pos = base + lane;
      int col = -1, sidx = 0;
      if (pos < wend) {
        int tt, j;
        if (!slot_prio) {
          tt = pos / a.k;
          j = pos - tt * a.k;
        } else {
          j = pos / a.tile_tokens;
          tt = pos - j * a.tile_tokens;
        }
        sidx = tt * a.k + j;
        const int e = s_exp[sidx];
        if (e >= 0) col = slot_prio ? j * a.E + e : e;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, col);
      int r = 0;
      if (col >= 0) r = hist[col] + __popc(peers & lanemask_lt());
      __syncwarp();
      if (col >= 0 && (31 - __clz(peers)) == lane) hist[col] += __popc(peers);
      __syncwarp();
      if (col >= 0) s_rank[sidx] = r;
    }
  }
  __syncthreads();

  // ---------------- Phase B2: warp prefix, then a decoupled look-back per
  // column.  Aggregates are published first (successors never wait on our
  // look-back); the look-back itself reads 256 predecessor tiles per round
  // per column from registers and stops at the nearest tile that already
  // carries an inclusive prefix, so there is no sequential chain across tiles.
  const bool last_tile = tile == a.n_tiles - 1;
  for (int c = tid; c < a.ncols; c += kGateThreads) {
    int run = 0;
#pragma unroll
    for (int w = 0; w < kGateWarps; ++w) {
      const int v = s_hist[w * a.ncols + c];
      s_hist[w * a.ncols + c] = run;
      run += v;
    }
    s_tot[c] = run;  // tile aggregate (the inclusive total after the look-back)
    s_excl[c] = 0;
    st_relaxed_u64(a.status + (size_t)c * a.n_tiles + tile,
                   (epoch << 34) | ((tile == 0 ? 2ull : 1ull) << 32) | (unsigned)run);
  }
  __syncthreads();
  GATE_TRACE(3);
  if (tile > 0) {
    // One warp per column: lane l holds the words of predecessors
    // p = hi - l - 32*u (u < kLB), i.e. 32*kLB tiles per round, loaded
    // before any is consumed; kCB columns are in flight per warp.  The
    // nearest inclusive tile p* is a warp max-reduce; the exclusive prefix
    // is the register sum of the words with p >= p*.  Rounds move to older
    // tiles only while no inclusive word has been seen.
    constexpr int kLB = 8, kCB = 4;
    for (int c0 = warp * kCB; c0 < a.ncols; c0 += kGateWarps * kCB) {
      int hi = tile - 1;
      unsigned excl[kCB];
      bool done[kCB];
#pragma unroll
      for (int cb = 0; cb < kCB; ++cb) {
        excl[cb] = 0;
        done[cb] = c0 + cb >= a.ncols;
      }
      while (true) {
        unsigned long long w[kCB][kLB];
#pragma unroll
        for (int cb = 0; cb < kCB; ++cb)
#pragma unroll
          for (int u = 0; u < kLB; ++u) {
            const int p = hi - lane - 32 * u;
            w[cb][u] = (epoch << 34) | (2ull << 32);  // p < 0: virtual inclusive 0
            if (p >= 0 && !done[cb])
              w[cb][u] = ld_relaxed_u64(a.status + (size_t)(c0 + cb) * a.n_tiles + p);
          }
        bool all_done = true;
#pragma unroll
        for (int cb = 0; cb < kCB; ++cb) {
          if (done[cb]) continue;  // warp-uniform
          int pin = -1;            // nearest inclusive predecessor seen by this lane
#pragma unroll
          for (int u = 0; u < kLB; ++u) {
            const int p = hi - lane - 32 * u;
            while ((w[cb][u] >> 34) != epoch || ((w[cb][u] >> 32) & 3u) == 0)  // rare
              w[cb][u] = ld_relaxed_u64(a.status + (size_t)(c0 + cb) * a.n_tiles + p);
            if (((w[cb][u] >> 32) & 3u) == 2u) pin = max(pin, p);
          }
#pragma unroll
          for (int m = 16; m > 0; m >>= 1) pin = max(pin, __shfl_xor_sync(0xffffffffu, pin, m));
          unsigned sum = 0;
#pragma unroll
          for (int u = 0; u < kLB; ++u) {
            const int p = hi - lane - 32 * u;
            if (p >= pin && p >= 0) sum += (unsigned)w[cb][u];
          }
#pragma unroll
          for (int m = 16; m > 0; m >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, m);
          excl[cb] += sum;
          if (pin >= hi - 32 * kLB + 1 || hi - 32 * kLB + 1 <= 0) done[cb] = true;
          else all_done = false;
        }
        if (all_done) break;
        hi -= 32 * kLB;
      }
      if (lane < kCB && c0 + lane < a.ncols) {
        unsigned ex = 0;
#pragma unroll
        for (int cb = 0; cb < kCB; ++cb)
          if (cb == lane) ex = excl[cb];
        const int c = c0 + lane;
        const unsigned incl = ex + (unsigned)s_tot[c];
        st_relaxed_u64(a.status + (size_t)c * a.n_tiles + tile, (epoch << 34) | (2ull << 32) | incl);
        s_excl[c] = (int)ex;
        s_tot[c] = (int)incl;
      }
    }
  }
  __syncthreads();
  GATE_TRACE(4);
  // ---------------- Phase B3: final slots (coalesced over t*k+j)
  for (int i = tid; i < nt * a.k; i += kGateThreads) {
    const int e = s_exp[i];
    const size_t gi = (size_t)t0 * a.k + i;
    if (e < 0) {
      a.slot_idx[gi] = -1;
      continue;
    }
    const int tt = i / a.k, j = i - tt * a.k;
    const int pos = slot_prio ? j * a.tile_tokens + tt : i;
    const int col = slot_prio ? j * a.E + e : e;
    const int s = s_excl[col] + s_hist[(pos / per) * a.ncols + col] + s_rank[i];
    if (slot_prio) {
      a.slot_idx[gi] = s;  // rank inside the j-stream; finalised by k_gate_slot_finalize
    } else if (s < a.cap) {
      a.slot_idx[gi] = s;
      if (a.slot_src) a.slot_src[(size_t)e * a.cap + s] = (int)gi;
    } else {
      a.slot_idx[gi] = -1;
      a.weight[gi] = 0.f;
    }
  }
  if (last_tile) {
    if (slot_prio) {
      for (int c = tid; c < a.ncols; c += kGateThreads) a.totals[c] = s_tot[c];
    } else {
      for (int e = tid; e < a.E; e += kGateThreads) a.load[e] = s_tot[e];
      if (a.slot_src)
        for (int e = warp; e < a.E; e += kGateWarps)  // warp per expert, coalesced
          for (int s = min(s_tot[e], a.cap) + lane; s < a.cap; s += 32)
            a.slot_src[(size_t)e * a.cap + s] = -1;
    }
  }

  // ---------------- reset the control block for the next call
  __syncthreads();
  GATE_TRACE(5);
  // Every CTA read the epoch before it incremented `done`, so the last one
  // may reset the block without a fence; the next launch sees it.
  if (tid == 0) {
    if (s_bad) atomicAdd(&a.ctrl->bad, s_bad);
    const unsigned prev = atomicAdd(&a.ctrl->done, 1u);
    if (prev == gridDim.x - 1) {
      a.ctrl->ticket = 0;
      a.ctrl->done = 0;
      a.ctrl->epoch = (unsigned)((epoch + 1) & 0x3FFFFFFFu);
    }
  }
}

// SLOT priority: slot = (admitted items of earlier j for this expert) +
// rank inside the j-stream; then capacity, load and slot_src.
__global__ void k_gate_slot_finalize(GateArgs a) {
  const size_t n = (size_t)a.S * a.k;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int e = a.expert_idx[i];
    if (e < 0) continue;
    const int j = (int)(i % a.k);
    int base = 0;
    for (int jj = 0; jj < j; ++jj) base += a.totals[jj * a.E + e];
    const int s = base + a.slot_idx[i];
    if (s < a.cap) {
      a.slot_idx[i] = s;
      if (a.slot_src) a.slot_src[(size_t)e * a.cap + s] = (int)i;
    } else {
      a.slot_idx[i] = -1;
      a.weight[i] = 0.f;
    }
  }
  const size_t nslots = (size_t)a.E * a.cap;
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < nslots || q < (size_t)a.E;
       q += stride) {
    if (q < (size_t)a.E) {
      int ld = 0;
      for (int jj = 0; jj < a.k; ++jj) ld += a.totals[jj * a.E + (int)q];
      a.load[q] = ld;
    }
    if (a.slot_src && q < nslots) {
      const int e = (int)(q / a.cap), s = (int)(q % a.cap);
      int ld = 0;
      for (int jj = 0; jj < a.k; ++jj) ld += a.totals[jj * a.E + e];
      if (s >= min(ld, a.cap)) a.slot_src[q] = -1;
    }
  }
}

// ------------------------------------------------------------ host side
using GateKernel = void (*)(GateArgs);

template <int KIND, int L>
static GateKernel pick_k(int K) {
  switch (K) {
    case 1: return k_gate<KIND, L, 1>;
    case 2: return k_gate<KIND, L, 2>;
    case 4: return k_gate<KIND, L, 4>;
    case 8: return k_gate<KIND, L, 8>;
    default: return k_gate<KIND, L, 0>;
  }
}
template <int KIND>
static GateKernel pick_l(int L, int K) {
  switch (L) {
    case 1: return pick_k<KIND, 1>(K);
    case 2: return pick_k<KIND, 2>(K);
    case 4: return pick_k<KIND, 4>(K);
    case 8: return pick_k<KIND, 8>(K);
    case 16: return pick_k<KIND, 16>(K);
    default: return pick_k<KIND, 32>(K);
  }
}

size_t gate_workspace_bytes(const moe_gate_desc_t& d) { return gate_plan(d).bytes; }

moe_status_t gate_launch(const moe_gate_desc_t& d, const float* logits, const int32_t* ids,
                         const int32_t* table, int32_t vocab, const moe_routing_t& out, void* ws,
                         cudaStream_t stream) {
  const GatePlan p = gate_plan(d);
  if (p.ncols > kMaxCols) {
    set_error("moe_gate: SLOT priority needs k*E <= %d (k=%d, E=%d)", kMaxCols, d.k, d.E);
    return MOE_ERR_UNSUPPORTED;
  }
  GateArgs a{};
  a.logits = logits;
  a.ids = ids;
  a.table = table;
  a.vocab = vocab;
  a.S = d.S;
  a.E = d.E;
  a.k = d.k;
  a.cap = d.capacity;
  a.mode = d.weight_mode;
  a.prio = d.priority;
  a.tile_tokens = p.tile_tokens;
  a.n_tiles = p.n_tiles;
  a.ncols = p.ncols;
  a.lg_words = p.lg_words;
  a.expert_idx = out.expert_idx;
  a.slot_idx = out.slot_idx;
  a.weight = out.weight;
  a.load = out.load;
  a.slot_src = out.slot_src;
  char* w = static_cast<char*>(ws);
  a.ctrl = reinterpret_cast<GateCtrl*>(w);
  a.status = reinterpret_cast<unsigned long long*>(w + p.status_off);
  a.totals = reinterpret_cast<int32_t*>(w + p.totals_off);
  a.trace = p.trace_off ? reinterpret_cast<unsigned long long*>(w + p.trace_off) : nullptr;

  GateKernel kern = d.kind == MOE_GATE_HASH    ? k_gate<KIND_HASH, 1, 1>
                    : d.kind == MOE_GATE_KTOP1 ? pick_l<KIND_KTOP1>(p.L, p.K)
                                               : pick_l<KIND_TOPK>(p.L, p.K);
  if (p.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)p.smem);
    if (e != cudaSuccess) return cuda_status(e, "moe_gate: smem attribute");
  }
  {
    void* args[] = {&a};
    cudaError_t e = launch_pdl((const void*)kern, dim3(p.n_tiles), dim3(kGateThreads), p.smem,
                               stream, args);
    if (e != cudaSuccess) return cuda_status(e, "moe_gate: k_gate launch");
  }
  if (d.priority == MOE_PRIO_SLOT) {
    const size_t n = std::max((size_t)d.S * d.k, (size_t)d.E * d.capacity);
    int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)device_sm_count() * 8);
    k_gate_slot_finalize<<<blocks, 256, 0, stream>>>(a);
    MOE_CHECK_LAUNCH("moe_gate: k_gate_slot_finalize launch");
  }
  return MOE_OK;
}

moe_status_t gate_check(void* ws, cudaStream_t stream, int32_t* bad) {
  GateCtrl* c = static_cast<GateCtrl*>(ws);
  unsigned h = 0;
  cudaError_t e = cudaMemcpyAsync(&h, &c->bad, sizeof h, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(&c->bad, 0, sizeof h, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_status(e, "moe_gate_check");
  *bad = (int32_t)h;
  return MOE_OK;
}

}  // namespace moe
