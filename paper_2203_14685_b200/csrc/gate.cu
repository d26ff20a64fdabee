// gate.cu -- moe_gate: Step 1 of Algorithm 1 on given gate
// logits, fused with capacity slot assignment.  Two or three
// kernels, chained with programmatic dependent launch (each one's launch
// overlaps its predecessor's tail), no spin-waits and no co-residency
// assumption: select -> slots2 when tiles x columns <= 4096 (every CTA then
// reduces the tile table itself), else select -> scan -> slots:
//
//   k_gate_select  one CTA per tile of tokens.  The tile's logits come into
//                  shared memory with one TMA bulk copy.  Selection + weights
//                  (Eq. 1, 123-124, 144-145): L lanes per
//                  token, each keeps a register top-K of its E/L logits, a
//                  shfl_xor butterfly merges the lists (larger raw fp32
//                  logit, then lower index -- R2, R3); k > 8 uses a rank-
//                  counting path; weights in fp64, rounded once (R1).  Then
//                  in-tile ranks per expert column (__match_any_sync over 32
//                  items at a time in admission order, per-warp histograms):
//                  provisional slot = warps-before + rank-in-warp, and the
//                  tile's per-column aggregate.
//   k_gate_scan    warp per column: exclusive scan of the tile aggregates
//                  (8 tiles per lane per round, in registers); totals, load.
//   k_gate_slots   slot = earlier tiles + provisional (SLOT priority: + the
//                  items of earlier j); >= cap -> dropped, weight 0 (R4-R6);
//                  slot_src and its empty entries.
//   k_gate_slots2  scan + slots in one pass (per-CTA table reduction).
// SAM (R17) and Dense-to-Sparse (R18) are further selection kinds of
// k_gate_select.  With the layout, gate and scatter run as one persistent
// kernel (gate_layout.cuh, moe_gate_layout / moe_gate_dispatch_p2p).
// Columns are experts (TOKEN priority, t-major admission) or (j, expert)
// pairs (SLOT priority, j-major).  Traffic is O(tiles x columns).
#include "gate_layout.cuh"

namespace moe {

// Exclusive scan of every column's tile aggregates (in place), warp per
// column, 8 consecutive tiles per lane per round of 256; the loads of up to
// kScanRounds rounds are issued before the first is scanned (one L2 round
// trip for <= 1024 tiles instead of one per round: C4a's 512 tiles).
// totals[c] = column total.  TOKEN priority: the column is the expert, so
// load[e] = totals[e].
constexpr int kScanRounds = 4;
__global__ void __launch_bounds__(kGateThreads) k_gate_scan(GateArgs a) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * kGateWarps + (threadIdx.x >> 5);
  gate_trace(a, blockIdx.x, 12);
  pdl_wait();
  pdl_trigger();
  gate_trace(a, blockIdx.x, 13);
  if (c >= a.ncols) return;
  unsigned* col = reinterpret_cast<unsigned*>(a.status) + (size_t)c * a.n_tiles;
  unsigned carry = 0;
  for (int blk = 0; blk < a.n_tiles; blk += 256 * kScanRounds) {
    unsigned v[kScanRounds][8];
#pragma unroll
    for (int r = 0; r < kScanRounds; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = blk + r * 256 + lane * 8 + u;
        v[r][u] = i < a.n_tiles ? __ldcg(col + i) : 0u;
      }
#pragma unroll
    for (int r = 0; r < kScanRounds; ++r) {
      const int base = blk + r * 256;
      if (base >= a.n_tiles) break;
      unsigned run = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const unsigned x = v[r][u];
        v[r][u] = run;
        run += x;
      }
      unsigned incl = run;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const unsigned o = __shfl_up_sync(0xffffffffu, incl, m);
        if (lane >= m) incl += o;
      }
      const unsigned lane_excl = carry + incl - run;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + lane * 8 + u;
        if (i < a.n_tiles) col[i] = lane_excl + v[r][u];
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  if (lane == 0) {
    a.totals[c] = (int)carry;
    if (a.prio != MOE_PRIO_SLOT) a.load[c] = (int)carry;
  }
  gate_trace(a, blockIdx.x, 14);  // warp 0's end
}

// Final slots: slot = (SLOT priority: items of earlier j of this expert) +
// items of earlier tiles in the column + the provisional in-tile rank;
// slot >= cap -> dropped (weight 0).  Then every CTA fills its share of the
// empty slot_src entries [min(load,cap), cap) (warp per expert).
__global__ void __launch_bounds__(kGateThreads) k_gate_slots(GateArgs a) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  const int t0 = tile * a.tile_tokens;
  const int nt = min(a.tile_tokens, a.S - t0);
  const bool slot_prio = a.prio == MOE_PRIO_SLOT;
  gate_trace(a, tile, 8);
  pdl_wait();
  pdl_trigger();
  gate_trace(a, tile, 9);
  const unsigned* pre = reinterpret_cast<const unsigned*>(a.status);
  // (staging this tile's column prefixes in shared memory together with the
  // first item, as k_gate_slots2 does, measured no faster here: C4a gate
  // stage 21.0 -> 22.1 us)
  for (int i = tid; i < nt * a.k; i += kGateThreads) {
    const size_t gi = (size_t)t0 * a.k + i;
    const int e = a.expert_idx[gi];
    if (e < 0) continue;
    const int j = i % a.k;
    int s = a.slot_idx[gi];
    if (slot_prio) {
      for (int jj = 0; jj < j; ++jj) s += a.totals[jj * a.E + e];
      s += (int)pre[(size_t)(j * a.E + e) * a.n_tiles + tile];
    } else {
      s += (int)pre[(size_t)e * a.n_tiles + tile];
    }
    if (s < a.cap) {
      a.slot_idx[gi] = s;
      if (a.slot_src) a.slot_src[(size_t)e * a.cap + s] = (int)gi;
    } else {
      a.slot_idx[gi] = -1;
      a.weight[gi] = 0.f;
    }
  }
  for (int e = tile * kGateWarps + warp; e < a.E; e += gridDim.x * kGateWarps) {
    int ld = 0;
    if (slot_prio) {
      for (int jj = 0; jj < a.k; ++jj) ld += a.totals[jj * a.E + e];
      if (lane == 0) a.load[e] = ld;
    } else {
      ld = a.totals[e];
    }
    if (a.slot_src)
      for (int s = min(ld, a.cap) + lane; s < a.cap; s += 32) a.slot_src[(size_t)e * a.cap + s] = -1;
  }
  if (a.trace) {
    __syncthreads();
    gate_trace(a, tile, 11);
  }
}

// Two-kernel variant of scan + slots: every CTA reduces the column
// aggregates itself (prefix over earlier tiles and the total, warp per
// column, 8 loads in flight per lane; O(tiles x columns) L2 words per CTA),
// then finishes its slots like k_gate_slots.  One launch and one dependency
// fewer than select -> scan -> slots.
__global__ void __launch_bounds__(kGateThreads) k_gate_slots2(GateArgs a) {
  __shared__ int s_pre[kMaxCols], s_tot[kMaxCols];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  const int t0 = tile * a.tile_tokens;
  const int nt = min(a.tile_tokens, a.S - t0);
  const bool slot_prio = a.prio == MOE_PRIO_SLOT;
  gate_trace(a, tile, 8);
  pdl_wait();
  pdl_trigger();
  gate_trace(a, tile, 9);
  // this thread's first item, loaded before the column reduction so the two
  // L2 round trips overlap
  const int n_items = nt * a.k;
  int e0 = -1, s0 = 0;
  if (tid < n_items) {
    e0 = __ldcg(a.expert_idx + (size_t)t0 * a.k + tid);
    s0 = __ldcg(a.slot_idx + (size_t)t0 * a.k + tid);
  }
  const unsigned* agg = reinterpret_cast<const unsigned*>(a.status);
  for (int c = warp; c < a.ncols; c += kGateWarps) {
    const unsigned* col = agg + (size_t)c * a.n_tiles;
    unsigned pre = 0, tot = 0;
    for (int base = 0; base < a.n_tiles; base += 256) {
      unsigned v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * 32 + lane;
        v[u] = i < a.n_tiles ? __ldcg(col + i) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        tot += v[u];
        if (base + u * 32 + lane < tile) pre += v[u];
      }
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
      pre += __shfl_xor_sync(0xffffffffu, pre, m);
      tot += __shfl_xor_sync(0xffffffffu, tot, m);
    }
    if (lane == 0) {
      s_pre[c] = (int)pre;
      s_tot[c] = (int)tot;
    }
  }
  __syncthreads();
  gate_trace(a, tile, 10);
  for (int i = tid; i < n_items; i += kGateThreads) {
    const size_t gi = (size_t)t0 * a.k + i;
    const bool first = i == tid;
    const int e = first ? e0 : a.expert_idx[gi];
    if (e < 0) continue;
    const int j = i % a.k;
    const int col = slot_prio ? j * a.E + e : e;
    int s = (first ? s0 : a.slot_idx[gi]) + s_pre[col];
    if (slot_prio)
      for (int jj = 0; jj < j; ++jj) s += s_tot[jj * a.E + e];
    if (s < a.cap) {
      a.slot_idx[gi] = s;
      if (a.slot_src) a.slot_src[(size_t)e * a.cap + s] = (int)gi;
    } else {
      a.slot_idx[gi] = -1;
      a.weight[gi] = 0.f;
    }
  }
  for (int e = tile * kGateWarps + warp; e < a.E; e += gridDim.x * kGateWarps) {
    int ld = 0;
    if (slot_prio)
      for (int jj = 0; jj < a.k; ++jj) ld += s_tot[jj * a.E + e];
    else
      ld = s_tot[e];
    if (lane == 0) a.load[e] = ld;
    if (a.slot_src)
      for (int s = min(ld, a.cap) + lane; s < a.cap; s += 32) a.slot_src[(size_t)e * a.cap + s] = -1;
  }
  if (a.trace) {
    __syncthreads();
    gate_trace(a, tile, 11);
  }
}

// ------------------------------------------------------------ host side
TraceBuf g_trace;  // moe_set_trace (profiling)

static GateKernel pick_gate(const moe_gate_desc_t& d, const GatePlan& p) {
  if (d.kind == MOE_GATE_SAM) return pick_sam(p.L, p.K);
  if (d.kind == MOE_GATE_D2S) return pick_d2s(p.L);
  return d.kind == MOE_GATE_HASH    ? pick_hash()
         : d.kind == MOE_GATE_KTOP1 ? pick_ktop1(p.L, p.K)
                                    : pick_topk(p.L, p.K);
}

// select -> slots2 (every CTA reduces the tile table itself) when the table
// is small, else select -> scan -> slots.
static bool two_kernels(const GatePlan& p) {
  return (long long)p.n_tiles * p.ncols <= tuning().gate_two_maxw;
}

// Kernels one moe_gate call enqueues for `d`: 2 (select -> slots2) or 3.
int gate_kernel_count(const moe_gate_desc_t& d, int ngroups) {
  return two_kernels(gate_plan_default(d, ngroups)) ? 2 : 3;
}

// The fused gate + layout kernel uses the separate gate's tiles (its phase G
// is the gate's select pass); its control block, status words [n_tiles][E]
// and tile-ready words [n_tiles] follow the gate's own workspace.
struct FusedPlan {
  GatePlan p;
  size_t ctrl_off, st_off, rdy_off, bytes;
};

static FusedPlan fused_plan(const moe_gate_desc_t& d) {
  FusedPlan f;
  f.p = gate_plan_default(d);
  // room for the largest tile count any tuning may pick
  const int most = std::max(f.p.n_tiles, gate_plan(d, 1 << 20, 1, 32).n_tiles);
  const size_t base = std::max({gate_plan_default(d).bytes, gate_plan(d, 1 << 20, 1, 32).bytes});
  f.ctrl_off = (base + 255) & ~(size_t)255;
  f.st_off = f.ctrl_off + 256;
  f.rdy_off = f.st_off + sizeof(unsigned long long) * (size_t)most * d.E;
  f.bytes = (f.rdy_off + sizeof(unsigned) * (size_t)most + 255) & ~(size_t)255;
  return f;
}

size_t gate_workspace_bytes(const moe_gate_desc_t& d) {
  // room for every tile count the tuning may pick (the table is small) and
  // for the fused gate + layout kernel's status words
  return fused_plan(d).bytes;
}

bool gate_layout_supported(const moe_gate_desc_t& d, int row_bytes) {
  return (d.kind == MOE_GATE_TOPK || d.kind == MOE_GATE_KTOP1 || d.kind == MOE_GATE_HASH) &&
         d.priority == MOE_PRIO_TOKEN && d.k <= 8 && d.E <= 256 && row_bytes % 32 == 0;
}

static void fill_args(GateArgs& a, const moe_gate_desc_t& d, const moe_gate_inputs_t& in,
                      const moe_routing_t& out, void* ws, const GatePlan& p, int ng) {
  a = GateArgs{};
  a.logits = in.logits;
  a.ids = in.token_ids;
  a.table = in.table;
  a.vocab = in.vocab;
  a.glogits = in.group_logits;
  a.ngroups = ng;
  a.uniforms = in.uniforms;
  a.tau = in.tau;
  a.eps = in.eps;
  a.z_words = p.z_words;
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
}

static moe_status_t select_launch(const moe_gate_desc_t& d, const GatePlan& p, GateArgs& a,
                                  cudaStream_t stream) {
  if (p.ncols > kMaxCols) {
    set_error("moe_gate: SLOT priority needs k*E <= %d (k=%d, E=%d)", kMaxCols, d.k, d.E);
    return MOE_ERR_UNSUPPORTED;
  }
  void* args[] = {&a};
  GateKernel kern = pick_gate(d, p);
  if (p.smem > 40 * 1024) {  // + static shared memory
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)p.smem);
    if (e != cudaSuccess) return cuda_status(e, "moe_gate: smem attribute");
  }
  cudaError_t e = launch_pdl((const void*)kern, dim3(p.n_tiles), dim3(kGateThreads), p.smem,
                             stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_gate: k_gate_select launch");
  return MOE_OK;
}

// k_gate_select -> (k_gate_slots2 | k_gate_scan -> k_gate_slots), PDL-chained.
// (A single launch -- the fused gate + layout kernel without rows: select,
// look-back prefix, slots -- measured slower, C2 18.0 vs 14.3 us; removed.)
moe_status_t gate_launch(const moe_gate_desc_t& d, const moe_gate_inputs_t& in,
                         const moe_routing_t& out, void* ws, cudaStream_t stream) {
  const int ng = d.kind == MOE_GATE_SAM ? in.n_groups : 1;
  const GatePlan p = gate_plan_default(d, ng);
  GateArgs a;
  fill_args(a, d, in, out, ws, p, ng);
  a.trace = static_cast<unsigned long long*>(g_trace.buf);
  a.trace_n = (long long)(g_trace.bytes / sizeof(unsigned long long));
  moe_status_t s = select_launch(d, p, a, stream);
  if (s != MOE_OK) return s;
  void* args[] = {&a};
  cudaError_t e;
  if (two_kernels(p)) {
    e = launch_pdl((const void*)k_gate_slots2, dim3(p.n_tiles), dim3(kGateThreads), 0, stream,
                   args);
    if (e != cudaSuccess) return cuda_status(e, "moe_gate: k_gate_slots2 launch");
    return MOE_OK;
  }
  e = launch_pdl((const void*)k_gate_scan, dim3((p.ncols + kGateWarps - 1) / kGateWarps),
                 dim3(kGateThreads), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_gate: k_gate_scan launch");
  e = launch_pdl((const void*)k_gate_slots, dim3(p.n_tiles), dim3(kGateThreads), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_gate: k_gate_slots launch");
  return MOE_OK;
}

moe_status_t gate_layout_launch(const moe_gate_desc_t& d, const moe_gate_inputs_t& in,
                                const moe_routing_t& out, void* ws, const void* x,
                                int dtype_size, int dcols, const PeerPtrs& dst, int E_local,
                                int rank, const PeerPtrs* pad_tab, const PeerPtrs* dup_tab,
                                cudaStream_t stream,
                                const PeerPtrs* wt_tab) {
  const int row_bytes = dtype_size * dcols;
  if (!gate_layout_supported(d, row_bytes)) {
    set_error("moe_gate_layout: no fused kernel for this gate (SLOT priority, SAM, D2S, k > 8 "
              "or rows not a multiple of 32 bytes)");
    return MOE_ERR_UNSUPPORTED;
  }
  const FusedPlan fp = fused_plan(d);
  const GatePlan& p = fp.p;
  FusedArgs f{};
  fill_args(f.g, d, in, out, ws, p, 1);
  RowArgs& a = f.r;
  a.src = static_cast<const char*>(x);
  a.expert_idx = out.expert_idx;
  a.slot_idx = out.slot_idx;
  a.weight = out.weight;
  a.load = out.load;
  a.S = d.S;
  a.E = d.E;
  a.k = d.k;
  a.cap = d.capacity;
  a.row_bytes = row_bytes;
  a.d = dcols;
  a.dpeer = dst;
  a.E_local = E_local;
  a.rank = rank;
  a.sys_fence = E_local != d.E;
  if (pad_tab) {
    a.skip_pads = 1;
    a.ptab = *pad_tab;
  }
  if (dup_tab) {
    a.dedupe = 1;
    a.dup = *dup_tab;
    if (wt_tab) a.wt = *wt_tab;
  }
  char* w = static_cast<char*>(ws);
  f.fc = reinterpret_cast<FusedCtrl*>(w + fp.ctrl_off);
  f.st = reinterpret_cast<unsigned long long*>(w + fp.st_off);
  f.tile_ready = reinterpret_cast<unsigned*>(w + fp.rdy_off);
  f.trace = static_cast<unsigned long long*>(g_trace.buf);
  f.trace_n = (long long)(g_trace.bytes / sizeof(unsigned long long));
  const int U = row_bytes <= 2048 ? 2 : 4;  // as k_layout: 2 KiB segments for rows <= 2 KiB
  FusedKernel kern = d.kind == MOE_GATE_HASH    ? pick_fused_hash(U)
                     : d.kind == MOE_GATE_KTOP1 ? pick_fused_ktop1(p.L, p.K, U)
                                                : pick_fused_topk(p.L, p.K, U);
  if (p.smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void*)kern,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    if (e != cudaSuccess) return cuda_status(e, "moe_gate_layout: smem attribute");
  }
  int per_sm = tuning().row_ctas_per_sm;
  if (per_sm <= 0)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kern, kGateThreads, p.smem);
  const int grid = std::max(1, per_sm) * device_sm_count();
  void* args[] = {&f};
  cudaError_t e = launch_pdl((const void*)kern, dim3(grid), dim3(kGateThreads), p.smem, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_gate_layout: k_gate_layout launch");
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
