// gate_impl.cuh -- the gate's device code (selection functions, gate_tile,
// the templated k_gate_select kernel) and the launch plan,
// shared by gate.cu (host side + the non-template kernels) and the picker
// TUs that instantiate the kernel templates (gate_pick_*.cu, compiled in
// parallel).  See gate.cu for the design.
#pragma once
#include <cfloat>
#include <climits>
#include <algorithm>

#include "launch.cuh"

namespace moe {

constexpr int kGateThreads = 256;
constexpr int kGateWarps = kGateThreads / 32;
constexpr int kMaxTileItems = 2048;  // tile_tokens * k
constexpr int kMaxCols = 2048;       // look-back columns: E or k*E
constexpr size_t kMaxTileLogitBytes = 64 * 1024;

struct GateCtrl {  // 64 bytes at the head of the workspace
  unsigned bad;        // invalid hash ids since the last moe_gate_check
  unsigned pad[15];
};

struct GateArgs {
  const float* logits;
  const int32_t* ids;
  const int32_t* table;
  int vocab;
  int S, E, k, cap, mode, prio;
  int tile_tokens, n_tiles, ncols;
  int lg_words;  // shared-memory words of the staged logits tile (16-byte multiple)
  int z_words;   // D2S: shared-memory words of the per-tile z = (l + G)/tau doubles
  // SAM (R17): group logits [S, ngroups], experts in contiguous groups
  const float* glogits;
  int ngroups;
  // Dense-to-Sparse (R18): uniforms [S, E] in (0,1) (NULL = eval), tau, eps
  const float* uniforms;
  double tau, eps;
  int32_t* expert_idx;
  int32_t* slot_idx;
  float* weight;
  int32_t* load;
  int32_t* slot_src;
  GateCtrl* ctrl;
  unsigned long long* status;  // [ncols][n_tiles] u32 tile aggregates, then prefixes
  int32_t* totals;             // [ncols] (SLOT priority)
  // profiling (moe_set_trace, the separate select -> (scan ->) slots path):
  // %globaltimer stamps per tile, NULL = off; see gate_trace
  unsigned long long* trace;
  long long trace_n;
};

// Gate trace layout: [0..3] = n_tiles, 16, 0, 2 (kind: separate gate); tile b's
// stamps at 4 + 16 b + i: k_gate_select i = 0 entry, 1 after pdl_wait, 2 logits
// staged, 3 selection done, 4 in-tile ranks, 5 tile aggregate, 6 end;
// k_gate_slots2 i = 8 entry, 9 after pdl_wait, 10 prefixes reduced, 11 end;
// select -> scan -> slots: k_gate_slots at 8, 9, 11 and k_gate_scan CTA b at
// 12 (entry), 13 (after pdl_wait), 14 (its warp 0 done) of "tile" b.
__device__ __forceinline__ void gate_trace(const GateArgs& a, int tile, int i) {
  const long long w = 4 + 16LL * tile + i;
  if (a.trace && threadIdx.x == 0 && w < a.trace_n) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[w] = t;
    if (tile == 0 && i == 0) {
      a.trace[0] = (unsigned long long)a.n_tiles;
      a.trace[1] = 16;
      a.trace[2] = 0;
      a.trace[3] = 2;
    }
  }
}



// ------------------------------------------------------------ layout of ws
struct GatePlan {
  int L, K, tile_tokens, n_tiles, ncols, lg_words, z_words;
  size_t status_off, totals_off, bytes, smem;
};

inline int choose_lanes(int E) {
  int L = 1;
  while (L * 2 <= 32 && E % (L * 2) == 0 && E / (L * 2) >= 8) L *= 2;
  return L;
}

inline int gate_tiles() { return tuning().gate_tiles; }
// Largest tile of the select -> (scan ->) slots path for the logit gates:
// 128 tokens (S = 64K: 512 tiles; measured C4a gate 22.6 -> 21.4 us, step
// 148 -> 145 us vs 256-token tiles; C2/C3 already get 128-token tiles from the
// >= 256 tiles rule).  The hash gate stages no logits and keeps 256 (C4b: gate
// unchanged, step 97.2 vs 98.3 us with 128).
inline int gate_max_tile(int kind) {
  const int t = tuning().gate_max_tile;
  return t > 0 ? t : kind == MOE_GATE_HASH ? 256 : 128;
}

// want_tiles: >= 256 tiles when S allows (about 1.7 CTAs per SM on 148 SMs)
inline GatePlan gate_plan(const moe_gate_desc_t& d, int want_tiles, int ngroups = 1,
                          int max_tile = 256) {
  GatePlan p{};
  p.L = d.kind == MOE_GATE_HASH ? 1 : choose_lanes(d.kind == MOE_GATE_SAM ? d.E / std::max(1, ngroups) : d.E);
  p.K = d.k <= 1 ? 1 : d.k <= 2 ? 2 : d.k <= 4 ? 4 : d.k <= 8 ? 8 : 0;
  // tiles of 32..256 tokens, at most kMaxTileItems items per tile
  int tt = 256;
  while (tt > 32 && tt > max_tile) tt >>= 1;
  while (tt > 32 && (d.S + tt - 1) / tt < want_tiles) tt >>= 1;
  while (tt > 1 && tt * d.k > kMaxTileItems) tt >>= 1;
  // the staged logits tile stays within kMaxTileLogitBytes of shared memory
  if (d.kind != MOE_GATE_HASH)
    while (tt > 1 && (size_t)tt * d.E * 4 > kMaxTileLogitBytes) tt >>= 1;
  p.tile_tokens = tt;
  p.n_tiles = (d.S + tt - 1) / tt;
  p.ncols = d.priority == MOE_PRIO_SLOT ? d.k * d.E : d.E;
  p.status_off = sizeof(GateCtrl);
  p.totals_off = p.status_off + sizeof(unsigned) * (size_t)p.n_tiles * p.ncols;
  p.bytes = p.totals_off + sizeof(int32_t) * (size_t)p.ncols;
  p.bytes = (p.bytes + 255) & ~(size_t)255;
  size_t items = (size_t)tt * d.k;
  p.lg_words = d.kind == MOE_GATE_HASH ? 0 : ((tt * d.E + 3) & ~3);
  p.z_words = d.kind == MOE_GATE_D2S ? 2 * tt * d.E : 0;
  p.smem = sizeof(int) * (p.lg_words + p.z_words + 2 * items + (size_t)kGateWarps * p.ncols);
  return p;
}

// The plan of the default (non-cooperative) gate launch.
inline GatePlan gate_plan_default(const moe_gate_desc_t& d, int ngroups = 1) {
  return gate_plan(d, gate_tiles(), ngroups, gate_max_tile(d.kind));
}

// ------------------------------------------------------------ selection
// (va, ia) ranks before (vb, ib): larger value, then lower index (R2, R3).
// Bitwise, not short-circuit: predicates and selects, no branches (the
// branchy form cost C4a's k-top-1 selection a reconvergence per logit).
__device__ __forceinline__ bool beats(float va, int ia, float vb, int ib) {
  return (va > vb) | ((va == vb) & (ia < ib));
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
  // Sorted insertion as a select network (no branches): b[p] = x beats
  // entry p is monotone in p (the list is sorted), so entry p becomes entry
  // p-1 where x beats it, x where x beats p but not p-1, else stays.
  __device__ __forceinline__ void insert(float x, int e) {
    bool b[K];
#pragma unroll
    for (int p = 0; p < K; ++p) b[p] = beats(x, e, v[p], i[p]);
#pragma unroll
    for (int p = K - 1; p > 0; --p) {
      v[p] = b[p - 1] ? v[p - 1] : (b[p] ? x : v[p]);
      i[p] = b[p - 1] ? i[p - 1] : (b[p] ? e : i[p]);
    }
    v[0] = b[0] ? x : v[0];
    i[0] = b[0] ? e : i[0];
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
// `row` is the softmax/selection domain (the whole row, or SAM's group
// slice starting at expert `ebase`); SAM SOFTMAX multiplies by `scale` =
// P(group).
template <int L, int K>
__device__ __forceinline__ void select_topk_reg(const GateArgs& a, const float* row, int t,
                                                bool valid, int l, int epl, bool vec4,
                                                int* s_sel /*[k]*/, int ebase = 0,
                                                double scale = 1.0) {
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
        a.expert_idx[o + p] = ebase + top.i[p];
        a.weight[o + p] = (float)(scale * (ex[p] / den));
        s_sel[p] = ebase + top.i[p];
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
  // the lane's experts are consecutive: its prototype pe = e / n is stepped
  // at prototype boundaries instead of divided per logit
  int pe = (l * epl) / n, next = (pe + 1) * n;
  if (valid)
    for_lane_logits(row, l, epl, vec4, [&](float x, int e) {
      const bool adv = e == next;
      pe += adv;
      next += adv ? n : 0;
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const bool take = (p == pe) & beats(x, e, bv[p], bi[p]);
        bv[p] = take ? x : bv[p];
        bi[p] = take ? e : bi[p];
      }
    });
#pragma unroll
  for (int m = 1; m < L; m <<= 1) {
#pragma unroll
    for (int p = 0; p < K; ++p) {
      float ov = __shfl_xor_sync(0xffffffffu, bv[p], m);
      int oi = __shfl_xor_sync(0xffffffffu, bi[p], m);
      const bool take = beats(ov, oi, bv[p], bi[p]);
      bv[p] = take ? ov : bv[p];
      bi[p] = take ? oi : bi[p];
    }
  }
  double den[K];
#pragma unroll
  for (int p = 0; p < K; ++p) den[p] = 1.0;
  if (a.mode == MOE_W_SOFTMAX) {
    double part[K];
#pragma unroll
    for (int p = 0; p < K; ++p) part[p] = 0.0;
    int qe = (l * epl) / n, qnext = (qe + 1) * n;
    if (valid)
      for_lane_logits(row, l, epl, vec4, [&](float x, int e) {
        if (e == qnext) {
          ++qe;
          qnext += n;
        }
#pragma unroll
        for (int p = 0; p < K; ++p)
          if (p == qe) part[p] += exp((double)x - (double)bv[p]);
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

// Hierarchical top-k / SAM (R17), K >= k: the Switch
// Router picks group g = argmax of the group logits (lowest index on ties;
// the L lanes of the token scan strided and merge with a butterfly), then the
// Mixture Router is the top-k register path on the group's n logits.
// SOFTMAX: weight = P(g) * within-group softmax, P(g) in fp64.
template <int L, int K>
__device__ __forceinline__ void select_sam_reg(const GateArgs& a, const float* row, int t,
                                               bool valid, int l, int* s_sel) {
  const int n = a.E / a.ngroups;
  const float* gl = a.glogits + (size_t)t * a.ngroups;
  float bv = -INFINITY;
  int bi = INT_MAX;
  if (valid)
    for (int h = l; h < a.ngroups; h += L) {
      const float x = __ldg(gl + h);
      if (beats(x, h, bv, bi)) {
        bv = x;
        bi = h;
      }
    }
#pragma unroll
  for (int m = 1; m < L; m <<= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, m);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
    if (beats(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  const int g = valid ? bi : 0;
  double pg = 1.0;
  if (a.mode == MOE_W_SOFTMAX) {
    double part = 0.0;
    if (valid)
      for (int h = l; h < a.ngroups; h += L) part += exp((double)__ldg(gl + h) - (double)bv);
    pg = 1.0 / group_sum<L>(part);
  }
  const int epl = n / L;
  const bool vec4 = (n % 4 == 0) && (epl % 4 == 0);
  select_topk_reg<L, K>(a, row + (size_t)g * n, t, valid, l, epl, vec4, s_sel, g * n, pg);
}

template <int L>
__device__ __forceinline__ double group_max_d(double x) {
#pragma unroll
  for (int m = 1; m < L; m <<= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, m));
  return x;
}

// Dense-to-Sparse (R18), k = E slots: z_e = (l_e + G_e)/tau
// in fp64 with G_e = -log(-log(u_e)) (train) or 0 (eval); p = softmax(z);
// survivors p_e >= eps fill slots 0..k'-1 in descending z (ties: lower
// index): each lane ranks its survivors against the token's z row in shared
// memory (pruned entries set to -inf first).  Pruned slots: expert -1,
// weight 0 (not admitted by the capacity pass).
template <int L>
__device__ __forceinline__ void select_d2s(const GateArgs& a, const float* row, double* zrow,
                                           int t, bool valid, int l, int* s_sel) {
  const int E = a.E, epl = E / L;
  const float* u = a.uniforms ? a.uniforms + (size_t)t * E : nullptr;
  double mx = -INFINITY;
  for (int q = 0; q < epl && valid; ++q) {
    const int e = l * epl + q;
    const double g = u ? -log(-log((double)__ldg(u + e))) : 0.0;
    const double z = ((double)row[e] + g) / a.tau;
    zrow[e] = z;
    mx = fmax(mx, z);
  }
  mx = group_max_d<L>(mx);
  double part = 0.0;
  for (int q = 0; q < epl && valid; ++q) part += exp(zrow[l * epl + q] - mx);
  const double den = group_sum<L>(part);
  double psum = 0.0;
  int ns = 0;
  for (int q = 0; q < epl && valid; ++q) {
    const int e = l * epl + q;
    const double p = exp(zrow[e] - mx) / den;
    if (p >= a.eps) {
      psum += p;
      ++ns;
    }
  }
  psum = group_sum<L>(psum);
#pragma unroll
  for (int m = 1; m < L; m <<= 1) ns += __shfl_xor_sync(0xffffffffu, ns, m);
  // survivors keep z, pruned -> -inf (each lane only rewrites its own
  // entries, which no other lane has read yet), then rank against the row
  for (int q = 0; q < epl && valid; ++q) {
    const int e = l * epl + q;
    if (!(exp(zrow[e] - mx) / den >= a.eps)) zrow[e] = -INFINITY;
  }
  __syncwarp();
  if (!valid) return;
  const size_t o = (size_t)t * E;
  for (int q = 0; q < epl; ++q) {
    const int e = l * epl + q;
    const double z = zrow[e];
    if (z == -INFINITY) continue;
    int r = 0;
    for (int e2 = 0; e2 < E; ++e2) {
      const double z2 = zrow[e2];
      r += (z2 > z || (z2 == z && e2 < e)) ? 1 : 0;
    }
    const double p = exp(z - mx) / den;
    a.expert_idx[o + r] = e;
    a.weight[o + r] = (float)(a.mode == MOE_W_RENORM ? p / psum : p);
    s_sel[r] = e;
  }
  for (int j = ns + l; j < E; j += L) {
    a.expert_idx[o + j] = -1;
    a.weight[o + j] = 0.f;
  }
}

// ------------------------------------------------------------ the kernel
enum { KIND_TOPK = 0, KIND_KTOP1 = 1, KIND_HASH = 2, KIND_SAM = 3, KIND_D2S = 4 };

// The logits-tile mbarrier: initialised once per CTA (thread 0, then a
// __syncthreads before its first use); gate_tile's n-th use waits on parity
// n & 1.
__device__ __forceinline__ void gate_mbar_init(unsigned long long& s_mbar) {
  const unsigned mbar = (unsigned)__cvta_generic_to_shared(&s_mbar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Phases A and B of one tile (k_gate_select, k_gate_layout):
// stage the logits, select + weights (expert_idx, weight written), in-tile
// ranks per column (s_exp, s_rank), s_hist[w][c] turned into the exclusive
// prefix over warps, and the tile aggregates written: agg[c][tile] in the
// workspace, or s_agg[c] in shared memory when s_agg is given.  Returns
// with the CTA synchronised.
template <int KIND, int L, int K>
__device__ __forceinline__ void gate_tile(const GateArgs& a, int* smem, unsigned& s_bad,
                                          unsigned long long& s_mbar, int tile, unsigned parity,
                                          int* s_agg = nullptr, bool init_mbar = false) {
  const int items = a.tile_tokens * a.k;
  float* s_lg = reinterpret_cast<float*>(smem);  // [tile_tokens][E] staged logits
  double* s_z = reinterpret_cast<double*>(smem + a.lg_words);  // D2S: [tile_tokens][E]
  int* s_exp = smem + a.lg_words + a.z_words;  // [items] expert of item tt*k+j
  int* s_rank = s_exp + items;                // [items] rank inside its warp
  int* s_hist = s_rank + items;               // [warps][ncols]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t0 = tile * a.tile_tokens;
  const int nt = min(a.tile_tokens, a.S - t0);
  // Stage the tile's logits (nt*E contiguous floats) into shared memory with
  // one TMA bulk copy (one DRAM latency for the whole tile), issued first so
  // the clears below overlap it (the staging area is disjoint from them); the
  // sub-16-byte tail with plain loads.
  const unsigned lg_bytes = KIND != KIND_HASH ? (unsigned)nt * a.E * 4u : 0u;
  const unsigned bulk = lg_bytes & ~15u;
  const float* g = a.logits + (size_t)t0 * a.E;
  const unsigned mbar = (unsigned)__cvta_generic_to_shared(&s_mbar);
  if (KIND != KIND_HASH && tid == 0) {
    if (init_mbar) gate_mbar_init(s_mbar);
    // the previous tile's generic-proxy reads of the buffer come first
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
  if (tid == 0) s_bad = 0;
  for (int i = tid; i < items; i += kGateThreads) s_exp[i] = -1;
  for (int i = tid; i < kGateWarps * a.ncols; i += kGateThreads) s_hist[i] = 0;
  if constexpr (KIND != KIND_HASH)
    for (unsigned i = bulk / 4 + tid; i < lg_bytes / 4; i += kGateThreads) s_lg[i] = __ldg(g + i);
  __syncthreads();  // the clears, the tail's stores (and the mbarrier's init)
  if constexpr (KIND != KIND_HASH) {
    unsigned done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(mbar), "r"(parity)
          : "memory");
  }
  gate_trace(a, tile, 2);

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
      if constexpr (KIND == KIND_D2S) {
        select_d2s<L>(a, row, s_z + (size_t)(valid ? tt : 0) * a.E, t, valid, l, s_sel);
      } else if constexpr (KIND == KIND_SAM) {
        select_sam_reg<L, K>(a, row, t, valid, l, s_sel);
      } else if constexpr (K == 0) {
        select_rank<L, KIND == KIND_KTOP1>(a, row, t, valid, l, epl, s_sel);
      } else if constexpr (KIND == KIND_TOPK) {
        select_topk_reg<L, K>(a, row, t, valid, l, epl, vec4, s_sel);
      } else {
        select_ktop1_reg<L, K>(a, row, t, valid, l, epl, vec4, s_sel);
      }
    }
  }
  __syncthreads();
  gate_trace(a, tile, 3);

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
  gate_trace(a, tile, 4);

  // ---------------- Phase B2: per-column warp prefix and tile aggregate
  unsigned* agg = reinterpret_cast<unsigned*>(a.status);  // [ncols][n_tiles]
  for (int c = tid; c < a.ncols; c += kGateThreads) {
    unsigned run = 0;
#pragma unroll
    for (int w = 0; w < kGateWarps; ++w) {
      const unsigned v = (unsigned)s_hist[w * a.ncols + c];
      s_hist[w * a.ncols + c] = (int)run;
      run += v;
    }
    if (s_agg)
      s_agg[c] = (int)run;
    else
      agg[(size_t)c * a.n_tiles + tile] = run;
  }
  __syncthreads();
  gate_trace(a, tile, 5);
}

template <int KIND, int L, int K>
__global__ void __launch_bounds__(kGateThreads) k_gate_select(GateArgs a) {
  extern __shared__ __align__(16) int smem[];
  __shared__ unsigned s_bad;
  __shared__ __align__(8) unsigned long long s_mbar;
  gate_trace(a, blockIdx.x, 0);
  pdl_wait();     // the producer of the logits / the previous step must be done
  pdl_trigger();  // k_gate_scan may launch now; it waits for our completion
  gate_trace(a, blockIdx.x, 1);
  gate_tile<KIND, L, K>(a, smem, s_bad, s_mbar, blockIdx.x, 0, nullptr, true);
  const int tid = threadIdx.x;
  const int items = a.tile_tokens * a.k;
  const int* s_exp = smem + a.lg_words + a.z_words;
  const int* s_rank = s_exp + items;
  const int* s_hist = s_rank + items;
  const int tile = blockIdx.x;
  const int t0 = tile * a.tile_tokens;
  const int nt = min(a.tile_tokens, a.S - t0);
  const bool slot_prio = a.prio == MOE_PRIO_SLOT;
  const int per = (items + kGateWarps - 1) / kGateWarps;
  // ---------------- provisional slots: rank inside the tile's column
  for (int i = tid; i < nt * a.k; i += kGateThreads) {
    const int e = s_exp[i];
    const size_t gi = (size_t)t0 * a.k + i;
    if (e < 0) {
      a.slot_idx[gi] = -1;  // invalid hash id: routed as dropped
      continue;
    }
    const int tt = i / a.k, j = i - tt * a.k;
    const int pos = slot_prio ? j * a.tile_tokens + tt : i;
    const int col = slot_prio ? j * a.E + e : e;
    a.slot_idx[gi] = s_hist[(pos / per) * a.ncols + col] + s_rank[i];
  }
  if (KIND == KIND_HASH && tid == 0 && s_bad) atomicAdd(&a.ctrl->bad, s_bad);
  if (a.trace) {
    __syncthreads();
    gate_trace(a, tile, 6);
  }
}

// ------------------------------------------------------------ kernel pickers
using GateKernel = void (*)(GateArgs);

template <int KIND, int L>
inline GateKernel pick_k(int K) {
  switch (K) {
    case 1: return k_gate_select<KIND, L, 1>;
    case 2: return k_gate_select<KIND, L, 2>;
    case 4: return k_gate_select<KIND, L, 4>;
    case 8: return k_gate_select<KIND, L, 8>;
    default: return k_gate_select<KIND, L, 0>;
  }
}
template <int KIND>
inline GateKernel pick_l(int L, int K) {
  switch (L) {
    case 1: return pick_k<KIND, 1>(K);
    case 2: return pick_k<KIND, 2>(K);
    case 4: return pick_k<KIND, 4>(K);
    case 8: return pick_k<KIND, 8>(K);
    case 16: return pick_k<KIND, 16>(K);
    default: return pick_k<KIND, 32>(K);
  }
}

// one translation unit each (they dominate the build)
GateKernel pick_topk(int L, int K);   // gate_pick_topk.cu
GateKernel pick_ktop1(int L, int K);  // gate_pick_ktop1.cu
GateKernel pick_hash();               // gate_pick_misc.cu
GateKernel pick_sam(int L, int K);                // gate_pick_misc.cu
GateKernel pick_d2s(int L);                       // gate_pick_misc.cu

}  // namespace moe
