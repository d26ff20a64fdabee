// p2p.cu -- the one-sided NVLink path: AllToAll steps
// 3/5 of Algorithm 1 done with SM stores straight
// into the owner rank's memory over NVLink 5 / NVSwitch, with the layout
// transform of step 2 fused into the dispatch.
//
//  - symmetric buffers: cudaMalloc + CUDA IPC handles, exchanged over the
//    library's own NCCL communicator (one ncclAllGather of 64-byte handles);
//    every rank maps every peer's allocation;
//  - device-side barrier: each rank bumps a local epoch, stores it (release,
//    system scope) into every peer's flag slot for this rank, and spins
//    (acquire, system scope) until all peers' flags reach it, or until the
//    tuning's barrier_timeout_ms passes (%globaltimer): then it sets this
//    rank's device error word and returns, and moe_comm_check reports
//    MOE_ERR_TIMEOUT instead of the stream hanging forever.  The epoch lives
//    in device memory, so the barrier is CUDA-graph replay safe;
//  - k_a2a_p2p: rank r copies its chunk q into rank q's receive buffer at
//    chunk r; destinations are interleaved so all NVLink ports stay busy;
//  - moe_dispatch_p2p: k_layout in peer mode stores every admitted row (and
//    the zero padding rows) directly into recv[r][e mod E/P][slot] of the
//    expert's owner.  Both end with the barrier, so when the call completes in
//    stream order every rank's receive buffer is complete.
//
// Every entry point is written as a program of steps separated by barriers
// (run_or_queue / comm_barrier): on a real communicator each step launches
// at once; on a simulated rank (sim.cu) the steps are queued and run later,
// all ranks phase by phase on one GPU, so the same code is parity-tested
// for P simulated ranks without NVLink.
#include <cstring>

#include "launch.cuh"
#include "rows.cuh"

namespace moe {

static moe_status_t nccl_st(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return MOE_OK;
  set_error("%s: NCCL error %d (%s)", what, (int)r, ncclGetErrorString(r));
  return MOE_ERR_NCCL;
}

// ------------------------------------------------------------ symmetric memory
moe_status_t sim_symm_alloc(moe_comm* c, size_t bytes, SymmBuf* out);  // sim.cu
moe_status_t sim_symm_release(moe_comm* c, SymmBuf& b);                // sim.cu

static moe_status_t symm_alloc_ipc(moe_comm* c, size_t bytes, SymmBuf* out) {
  const int P = c->nranks, r = c->rank;
  if (P > kMaxRanks) {
    set_error("symmetric memory supports up to %d ranks (got %d)", kMaxRanks, P);
    return MOE_ERR_UNSUPPORTED;
  }
  bytes = (bytes + 4095) & ~(size_t)4095;
  char* base = nullptr;
  cudaError_t e = cudaMalloc(&base, bytes);
  if (e != cudaSuccess) return cuda_status(e, "symmetric alloc: cudaMalloc");
  e = cudaMemset(base, 0, bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, base);
  char* d_h = nullptr;
  cudaStream_t st = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&d_h, (size_t)P * sizeof h);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMemcpy(d_h + (size_t)r * sizeof h, &h, sizeof h, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(base);
    if (d_h) cudaFree(d_h);
    if (st) cudaStreamDestroy(st);
    return cuda_status(e, "symmetric alloc: IPC handle");
  }
  moe_status_t s = nccl_st(ncclAllGather(d_h + (size_t)r * sizeof h, d_h, sizeof h, ncclInt8,
                                         c->nccl, st),
                           "symmetric alloc: handle exchange");
  std::vector<cudaIpcMemHandle_t> all(P);
  if (s == MOE_OK) {
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaMemcpy(all.data(), d_h, (size_t)P * sizeof h, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) s = cuda_status(e, "symmetric alloc: handle exchange");
  }
  cudaFree(d_h);
  cudaStreamDestroy(st);
  if (s != MOE_OK) {
    cudaFree(base);
    return s;
  }
  SymmBuf b{};
  b.base = base;
  b.bytes = bytes;
  for (int q = 0; q < P; ++q) {
    if (q == r) {
      b.peer.p[q] = base;
      continue;
    }
    void* pp = nullptr;
    e = cudaIpcOpenMemHandle(&pp, all[q], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int u = 0; u < q; ++u)
        if (u != r) cudaIpcCloseMemHandle(b.peer.p[u]);
      cudaFree(base);
      return cuda_status(e, "symmetric alloc: cudaIpcOpenMemHandle (no peer access?)");
    }
    b.peer.p[q] = static_cast<char*>(pp);
  }
  *out = b;
  return MOE_OK;
}

moe_status_t symm_alloc(moe_comm* c, size_t bytes, SymmBuf* out) {
  return c->sim ? sim_symm_alloc(c, bytes, out) : symm_alloc_ipc(c, bytes, out);
}

void symm_release(moe_comm* c, SymmBuf& b) {
  for (int q = 0; q < c->nranks; ++q)
    if (q != c->rank && b.peer.p[q]) cudaIpcCloseMemHandle(b.peer.p[q]);
  if (b.base) cudaFree(b.base);
  b.base = nullptr;
}

// A host-side rendezvous of all ranks (used around frees).
static moe_status_t host_barrier(moe_comm* c) {
  int* d = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(int));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_status(e, "barrier");
  moe_status_t s = nccl_st(ncclAllReduce(d, d, 1, ncclInt32, ncclSum, c->nccl, st), "barrier");
  if (s == MOE_OK) {
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) s = cuda_status(e, "barrier");
  }
  cudaFree(d);
  cudaStreamDestroy(st);
  return s;
}

// Collective release: every rank is done with the buffer before anyone
// unmaps or frees it, and nobody allocates again before every rank freed.
moe_status_t symm_release_coll(moe_comm* c, SymmBuf& b) {
  if (c->sim) return sim_symm_release(c, b);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_status(e, "symmetric free: sync");
  moe_status_t s = host_barrier(c);
  if (s != MOE_OK) return s;
  symm_release(c, b);
  return host_barrier(c);
}

// ------------------------------------------------------------ programs
moe_status_t run_or_queue(moe_comm* c, cudaStream_t stream,
                          std::function<moe_status_t(cudaStream_t)> fn) {
  if (!c->sim) return fn(stream);
  SimItem it;
  it.kind = SimItem::FN;
  it.fn = std::move(fn);
  c->queue.push_back(std::move(it));
  return MOE_OK;
}

// ------------------------------------------------------------ device barrier
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_barrier(PeerPtrs sig, int P, int rank, unsigned long long timeout_ns) {
  __shared__ unsigned long long s_e;
  unsigned long long* mine = reinterpret_cast<unsigned long long*>(sig.p[rank]);
  pdl_wait();     // everything before us in the stream is complete
  pdl_trigger();  // the next kernel may be scheduled now; it waits for our completion
  if (threadIdx.x == 0) {
    s_e = mine[kMaxRanks] + 1;
    mine[kMaxRanks] = s_e;
  }
  __syncthreads();
  const unsigned long long e = s_e;
  asm volatile("fence.acq_rel.sys;" ::: "memory");  // one fence, then the releases
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    unsigned long long* flag = reinterpret_cast<unsigned long long*>(sig.p[q]) + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(e) : "memory");
  }
  const unsigned long long t0 = globaltimer_ns();
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine + q) : "memory");
      if (v >= e) break;
      if (timeout_ns && globaltimer_ns() - t0 > timeout_ns) {
        // a peer never arrived: flag it and let the stream go on
        atomicOr(reinterpret_cast<unsigned*>(sig.p[rank] + kErrOff), (unsigned)kErrBarrierTimeout);
        return;
      }
    }
  }
}

moe_status_t barrier_launch(const PeerPtrs& sig, int nranks, int rank, cudaStream_t stream) {
  // PDL by default: re-measured in round 2 at 1-4 us faster per step (C2 at
  // N=2 252.6 vs 254.2 us; N=4 C2/C3/C4a/C4b all 0.3-1.7 us faster)
  unsigned long long to = (unsigned long long)tuning().barrier_timeout_ms * 1000000ull;
  void* args[] = {(void*)&sig, &nranks, &rank, &to};
  cudaError_t e = tuning().barrier_pdl
                      ? launch_pdl((const void*)k_barrier, dim3(1), dim3(32), 0, stream, args)
                      : cudaLaunchKernel((const void*)k_barrier, dim3(1), dim3(32), args, 0, stream);
  if (e != cudaSuccess) return cuda_status(e, "moe_comm_barrier: launch");
  return MOE_OK;
}

moe_status_t sim_barrier(moe_comm* c, cudaStream_t stream);  // sim.cu

moe_status_t comm_barrier(moe_comm* c, cudaStream_t stream) {
  if (c->sim) return sim_barrier(c, stream);
  return barrier_launch(c->sig.peer, c->nranks, c->rank, stream);
}

// ------------------------------------------------------------ P2P AllToAll
// Rank r: for every q, send[q] -> recv_q[r] (recv_q = rank q's buffer).
// Work is cut into 64 KiB pieces, interleaved over destinations.
__global__ void __launch_bounds__(256) k_a2a_p2p(const char* __restrict__ send, PeerPtrs recv,
                                                 size_t off_rank, size_t b, int P, int rank) {
  constexpr size_t kPiece = 64 * 1024;
  constexpr int U = 4;
  pdl_wait();
  const size_t per = (b + kPiece - 1) / kPiece;
  const size_t n = per * (size_t)P;
  for (size_t j = blockIdx.x; j < n; j += gridDim.x) {
    const int q = (rank + 1 + (int)(j % P)) % P;
    const size_t beg = (j / P) * kPiece;
    const size_t len = (b - beg) < kPiece ? (b - beg) : kPiece;
    const char* src = send + (size_t)q * b + beg;
    char* dst = recv.p[q] + off_rank + beg;
    for (size_t o = (size_t)threadIdx.x * 16; o < len; o += (size_t)blockDim.x * 16 * U) {
      V4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t oo = o + (size_t)u * blockDim.x * 16;
        if (oo < len) v[u] = ld_stream_v4(src + oo);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t oo = o + (size_t)u * blockDim.x * 16;
        if (oo < len) st_v4(dst + oo, v[u]);
      }
    }
  }
  __threadfence_system();
}

moe_status_t a2a_p2p_launch(const char* send, const PeerPtrs& recv, size_t recv_off_rank,
                            size_t bytes_per_peer, int nranks, int rank, cudaStream_t stream) {
  const size_t pieces = ((bytes_per_peer + 65535) / 65536) * nranks;
  int grid = (int)std::min<size_t>(pieces, (size_t)device_sm_count() * tuning().a2a_ctas_per_sm);
  if (grid < 1) grid = 1;
  void* args[] = {(void*)&send, (void*)&recv, &recv_off_rank, &bytes_per_peer, &nranks, &rank};
  cudaError_t e = launch_pdl((const void*)k_a2a_p2p, dim3(grid), dim3(256), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "moe_alltoall(P2P): launch");
  return MOE_OK;
}

// ------------------------------------------------------------ local padding
static bool local_pad_on(const moe_gate_desc_t& d) {
  const int t = tuning().p2p_local_pad;
  return t >= 0 ? t != 0 : pad_heavy(d);
}

// After the padded one-sided dispatch's exit barrier: zero this rank's own
// padding rows [cnt, cap) of every (source rank, local expert) block of recv
// ([P][El][cap] rows), cnt from the padding-count table the senders filled.
// The zero rows never cross NVLink (C4b's C = 1.25 makes them ~20% of it).
__global__ void __launch_bounds__(256) k_pad_fill(char* recv, const int* tab, int P, int El,
                                                  int cap, int row_bytes) {
  __shared__ int s_cnt[256];
  pdl_wait();
  pdl_trigger();
  const int n = P * El;  // = E <= 256
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int src = i / El, le = i - src * El;
    const int c = ((const volatile int*)tab)[src * kPadTabStride + le];
    s_cnt[i] = cap - min(max(c, 0), cap);
  }
  __syncthreads();
  __shared__ int s_pre[257];
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int carry = 0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const int v = i < n ? s_cnt[i] : 0;
      int incl = v;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, m);
        if (lane >= m) incl += o;
      }
      if (i < n) s_pre[i] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_pre[n] = carry;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (blockDim.x / 32);
  const V4 z = V4{{0, 0, 0, 0}};
  for (int p = gw; p < s_pre[n]; p += nw) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pre[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const int s = cap - s_cnt[lo] + (p - s_pre[lo]);
    char* row = recv + ((size_t)lo * cap + s) * row_bytes;
    for (int off = lane * 16; off < row_bytes; off += 32 * 16) st_v4(row + off, z);
  }
}

// tab: this rank's padding-count table (RecvTables of recv)
static moe_status_t pad_fill_launch(char* local, const int* tab, int P, int El, int cap,
                                    int row_bytes, cudaStream_t stream) {
  const int nrows_pad_max = P * El * cap;
  const int grid = std::max(1, std::min(device_sm_count() * 4, (nrows_pad_max + 7) / 8));
  void* args[] = {&local, (void*)&tab, &P, &El, &cap, &row_bytes};
  cudaError_t e = launch_pdl((const void*)k_pad_fill, dim3(grid), dim3(256), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "k_pad_fill launch");
  return MOE_OK;
}

// ------------------------------------------------------------ dispatch dedupe
// Owner side: a warp per 32 table entries (coalesced), each nonzero entry
// "= row v-1" copied (16-byte vectors, local HBM), then cleared for the next
// step.  The warp copies up to kDupRows rows at a time, all their loads
// issued before the first store (one HBM latency per group of rows instead
// of per row: a trace of C2 at N=2 showed the serial per-row copy as ~8 us
// between the dispatch and the combine; 4 rows: step 242.4 -> 236.8 us, 8
// rows with the pre-combine at 4 pairs: 225.5 -> 223.1 us).  The entries were stored by the
// senders before their exit barrier (release) and this kernel runs after it
// (acquire).
constexpr int kDupRows = 8;
__global__ void __launch_bounds__(128) k_dup_fill(char* recv, int* tab, long long n, int row_bytes,
                                                  int* pairs) {
  pdl_wait();
  pdl_trigger();
  constexpr int kV = 4;  // 16-byte vectors per lane per row segment: 2 KiB of a row per round
  const int lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;  // warps per CTA
  const long long gw = (long long)blockIdx.x * wpc + (threadIdx.x >> 5), nw = (long long)gridDim.x * wpc;
  for (long long base = gw * 32; base < n; base += nw * 32) {
    const long long i = base + lane;
    const int v = i < n ? tab[i] : 0;
    // the pair table (read by the combine's pre-combine) gets this step's
    // entries, zeros included, so no stale pair survives a step
    if (pairs && i < n) pairs[i] = v;
    unsigned m = __ballot_sync(0xffffffffu, v != 0);
    while (m) {
      const char* sr[kDupRows];
      char* dr[kDupRows];
      int cnt = 0;
#pragma unroll
      for (int q = 0; q < kDupRows; ++q) {
        sr[q] = nullptr;
        dr[q] = nullptr;
        if (m) {
          const int l = __ffs(m) - 1;
          m &= m - 1;
          const long long src = (long long)__shfl_sync(0xffffffffu, v, l) - 1;
          sr[q] = recv + src * row_bytes;
          dr[q] = recv + (base + l) * row_bytes;
          cnt = q + 1;
        }
      }
      for (int o0 = 0; o0 < row_bytes; o0 += 32 * 16 * kV) {
        V4 r[kDupRows][kV];
#pragma unroll
        for (int q = 0; q < kDupRows; ++q)
#pragma unroll
          for (int u = 0; u < kV; ++u) {
            const int off = o0 + (lane + 32 * u) * 16;
            if (q < cnt && off < row_bytes) r[q][u] = ld_stream_v4(sr[q] + off);
          }
#pragma unroll
        for (int q = 0; q < kDupRows; ++q)
#pragma unroll
          for (int u = 0; u < kV; ++u) {
            const int off = o0 + (lane + 32 * u) * 16;
            if (q < cnt && off < row_bytes) st_v4(dr[q] + off, r[q][u]);
          }
      }
    }
    if (v) tab[i] = 0;
  }
}

moe_status_t dup_fill_launch(char* recv, int* tab, long long n_rows, int row_bytes,
                             cudaStream_t stream, int* pairs) {
  const long long groups = (n_rows + 31) / 32;
  // 128-thread CTAs: two fit per SM at ~200 registers, so every warp of
  // the (single) pass is resident at once
  const int grid = (int)std::max<long long>(1, std::min<long long>((groups + 3) / 4,
                                                                    (long long)device_sm_count() * 8));
  void* args[] = {&recv, &tab, &n_rows, &row_bytes, &pairs};
  cudaError_t e = launch_pdl((const void*)k_dup_fill, dim3(grid), dim3(128), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "k_dup_fill launch");
  return MOE_OK;
}

// ------------------------------------------------------------ combine pre-combine
// Owner side, before the combine's entry barrier: for every pair "row B =
// row A" of this step (the pair table k_dup_fill refreshed: one token's two
// slots, both here), pre[B] = the token's combined row, w_A * out[A] + w_B *
// out[B] in fp32 from 0 in slot order, rounded once -- exactly what the
// token's owner would compute from the two rows -- so the combine reads one
// row over NVLink instead of two.  A warp per 32 table entries; the weights
// came with the dispatch (RowArgs::wt).  Rows are 32-byte multiples.
template <int DT>
__global__ void __launch_bounds__(128) k_precombine(const char* recv, const int* pairs,
                                                    const float* wt, char* pre, long long n,
                                                    int row_bytes) {
  pdl_wait();
  pdl_trigger();
  constexpr int NA = DT == MOE_F32 ? 8 : 16;
  constexpr int kS = 2;      // 1 KiB segments per round
  constexpr int kPairs = 4;  // pairs per warp with all their loads in flight
  const int lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;  // warps per CTA
  const long long gw = (long long)blockIdx.x * wpc + (threadIdx.x >> 5), nw = (long long)gridDim.x * wpc;
  for (long long base = gw * 32; base < n; base += nw * 32) {
    const long long i = base + lane;
    const int v = i < n ? pairs[i] : 0;
    unsigned m = __ballot_sync(0xffffffffu, v != 0);
    while (m) {
      const char* xa[kPairs];
      const char* xb[kPairs];
      char* out[kPairs];
      float wa[kPairs], wb[kPairs];
      int cnt = 0;
#pragma unroll
      for (int q = 0; q < kPairs; ++q) {
        xa[q] = xb[q] = nullptr;
        out[q] = nullptr;
        wa[q] = wb[q] = 0.f;
        if (m) {
          const int l = __ffs(m) - 1;
          m &= m - 1;
          const long long ra = (long long)__shfl_sync(0xffffffffu, v, l) - 1, rb = base + l;
          wa[q] = wt[ra];
          wb[q] = wt[rb];
          xa[q] = recv + ra * row_bytes;
          xb[q] = recv + rb * row_bytes;
          out[q] = pre + rb * row_bytes;
          cnt = q + 1;
        }
      }
      for (int o0 = 0; o0 < row_bytes; o0 += 1024 * kS) {
        V8 va[kPairs][kS], vb[kPairs][kS];
#pragma unroll
        for (int q = 0; q < kPairs; ++q)
#pragma unroll
          for (int u = 0; u < kS; ++u) {
            const int off = o0 + (lane + 32 * u) * 32;
            if (q < cnt && off < row_bytes) {
              va[q][u] = ld_stream_v8(xa[q] + off);
              vb[q][u] = ld_stream_v8(xb[q] + off);
            }
          }
#pragma unroll
        for (int q = 0; q < kPairs; ++q)
#pragma unroll
          for (int u = 0; u < kS; ++u) {
            const int off = o0 + (lane + 32 * u) * 32;
            if (q < cnt && off < row_bytes) {
              float acc[NA];
#pragma unroll
              for (int z = 0; z < NA; ++z) acc[z] = 0.f;
              fma_vec<DT>(acc, wa[q], va[q][u]);
              fma_vec<DT>(acc, wb[q], vb[q][u]);
              st_v8(out[q] + off, pack_vec<DT>(acc));
            }
          }
      }
    }
  }
}

static moe_status_t precombine_launch(const char* recv, const int* pairs, const float* wt,
                                      char* pre, long long n_rows, int row_bytes, int dtype,
                                      cudaStream_t stream) {
  const long long groups = (n_rows + 31) / 32;
  // 128-thread CTAs: two fit per SM at ~200 registers, so every warp of
  // the (single) pass is resident at once
  const int grid = (int)std::max<long long>(1, std::min<long long>((groups + 3) / 4,
                                                                    (long long)device_sm_count() * 8));
  void* args[] = {&recv, &pairs, &wt, &pre, &n_rows, &row_bytes};
  const void* kern = dtype == MOE_F32 ? (const void*)k_precombine<MOE_F32>
                                      : (const void*)k_precombine<MOE_BF16>;
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(128), 0, stream, args);
  if (e != cudaSuccess) return cuda_status(e, "k_precombine launch");
  return MOE_OK;
}

// The side tables of receive buffer `recv` (this rank's pointer), with room
// for a duplicate-row table of `dup_rows` rows (0: padding counts only).
// Allocated (collectively: every rank makes the same call) on first use
// outside stream capture, grown the same way; inside a capture without a
// large enough set: nullptr, and the dispatch sends every row, padding
// included (same result).
static RecvTables* recv_tables(moe_comm* c, const void* recv, size_t dup_rows, cudaStream_t stream,
                               moe_status_t* st) {
  *st = MOE_OK;
  RecvTables* t = nullptr;
  for (RecvTables& u : c->tables)
    if (u.recv == recv) t = &u;
  if (t && t->dup_rows >= dup_rows) return t;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
    return nullptr;
  if (t) {  // grow: collectively, after every rank is done with the old set
    *st = symm_release_coll(c, t->buf);
    if (*st == MOE_OK && t->pre.base) *st = symm_release_coll(c, t->pre);
    c->tables.erase(c->tables.begin() + (t - c->tables.data()));
    if (*st != MOE_OK) return nullptr;
  }
  RecvTables n{};
  n.recv = recv;
  n.dup_rows = dup_rows;
  *st = symm_alloc(c, kPadTabBytes + 3 * dup_rows * sizeof(int), &n.buf);  // zero-filled
  if (*st != MOE_OK) return nullptr;
  c->tables.push_back(n);
  return &c->tables.back();
}

// Collective: release the side tables of every receive buffer inside
// [base, base + bytes) (before that buffer is freed).
static moe_status_t release_tables_in(moe_comm* c, const char* base, size_t bytes) {
  moe_status_t s = MOE_OK;
  for (size_t i = 0; i < c->tables.size();) {
    const char* q = static_cast<const char*>(c->tables[i].recv);
    if (q >= base && q < base + bytes) {
      moe_status_t s2 = symm_release_coll(c, c->tables[i].buf);
      if (s == MOE_OK) s = s2;
      if (c->tables[i].pre.base) {
        s2 = symm_release_coll(c, c->tables[i].pre);
        if (s == MOE_OK) s = s2;
      }
      c->tables.erase(c->tables.begin() + i);
    } else {
      ++i;
    }
  }
  return s;
}

// ------------------------------------------------------------ dropless exchange
// counts_q[r][le] = admitted rows of this rank r for q's local expert le
// (stores into every owner's symmetric count table).
__global__ void k_a2av_counts(const int32_t* offsets, PeerPtrs counts, int E, int El, int rank) {
  pdl_wait();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int q = e / El, le = e - q * El;
    reinterpret_cast<int32_t*>(counts.p[q])[rank * El + le] = __ldg(offsets + e + 1) - __ldg(offsets + e);
  }
  __threadfence_system();
}

// peer_base[q] = rows ranks < r put into q's recv (read from q's table);
// recv_offsets = exclusive prefix of this rank's own table [src][le].
__global__ void __launch_bounds__(256) k_a2av_plan(PeerPtrs counts, int P, int El, int rank,
                                                   int32_t* peer_base, int32_t* recv_offsets) {
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = warp; q < P; q += blockDim.x / 32) {
    const volatile int32_t* c = reinterpret_cast<const volatile int32_t*>(counts.p[q]);
    int sum = 0;
    for (int i = lane; i < rank * El; i += 32) sum += c[i];
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, m);
    if (lane == 0) peer_base[q] = sum;
  }
  if (warp == 0) {
    const volatile int32_t* c = reinterpret_cast<const volatile int32_t*>(counts.p[rank]);
    const int n = P * El;
    int carry = 0;
    if (lane == 0) recv_offsets[0] = 0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const int v = i < n ? c[i] : 0;
      int incl = v;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, m);
        if (lane >= m) incl += o;
      }
      if (i < n) recv_offsets[i + 1] = carry + incl;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

// ------------------------------------------------------------ argument checks
static moe_status_t need_p2p(const char* fn, moe_comm_t* comm) {
  if (!comm) {
    set_error("%s: comm is NULL", fn);
    return MOE_ERR_INVALID_ARG;
  }
  if (!comm->p2p_ok) {
    set_error("%s: peer memory is not available between these GPUs", fn);
    return MOE_ERR_UNSUPPORTED;
  }
  return MOE_OK;
}

// The symmetric buffer of `bytes` at p, with its per-rank mappings.
static moe_status_t symm_peers(const char* fn, moe_comm_t* comm, const void* p, size_t bytes,
                               PeerPtrs* out) {
  const SymmBuf* b = find_symm(comm, p, bytes);
  if (!b) {
    set_error("%s: a buffer of %zu bytes is not inside a symmetric buffer (moe_comm_symm_alloc)",
              fn, bytes);
    return MOE_ERR_INVALID_ARG;
  }
  const size_t off = static_cast<const char*>(p) - b->base;
  *out = PeerPtrs{};
  for (int q = 0; q < comm->nranks; ++q) out->p[q] = b->peer.p[q] + off;
  return MOE_OK;
}

// Shared checks of the padded entry points; fills the peer pointers of `buf`.
static moe_status_t p2p_args(const char* fn, moe_comm_t* comm, const moe_gate_desc_t* desc,
                             const moe_routing_t* routing, const void* a, const void* buf,
                             int32_t d, int32_t dtype, PeerPtrs* peers, int* ds) {
  moe_status_t s = need_p2p(fn, comm);
  if (s != MOE_OK) return s;
  if (!desc || !routing || !routing->expert_idx || !routing->slot_idx || !a || !buf || d < 1 ||
      (dtype != MOE_F32 && dtype != MOE_BF16)) {
    set_error("%s: bad arguments", fn);
    return MOE_ERR_INVALID_ARG;
  }
  const int P = comm->nranks;
  if (desc->E % P != 0 || desc->E > 256 || desc->S < 1 || desc->k < 1 || desc->capacity < 1) {
    set_error("%s: E=%d experts must shard over %d ranks (E <= 256, S, k, cap >= 1)", fn, desc->E, P);
    return MOE_ERR_INVALID_ARG;
  }
  *ds = dtype == MOE_F32 ? 4 : 2;
  if (((long long)d * *ds) % 16 != 0 || reinterpret_cast<uintptr_t>(a) % 16 ||
      reinterpret_cast<uintptr_t>(buf) % 16) {
    set_error("%s: rows and pointers must be 16-byte aligned", fn);
    return MOE_ERR_ALIGNMENT;
  }
  return symm_peers(fn, comm, buf, (size_t)desc->E * desc->capacity * d * *ds, peers);
}

static moe_status_t packed_args(const char* fn, moe_comm_t* comm, const moe_gate_desc_t* desc,
                                const moe_routing_t* routing, const int32_t* offsets,
                                const void* a, const void* buf, int64_t rows, int32_t d,
                                int32_t dtype, PeerPtrs* peers, int* ds) {
  moe_status_t s = need_p2p(fn, comm);
  if (s != MOE_OK) return s;
  if (!desc || !routing || !routing->expert_idx || !routing->slot_idx || !offsets || !a || !buf ||
      d < 1 || (dtype != MOE_F32 && dtype != MOE_BF16)) {
    set_error("%s: bad arguments", fn);
    return MOE_ERR_INVALID_ARG;
  }
  const int P = comm->nranks;
  if (desc->E % P != 0 || desc->E > 256) {
    set_error("%s: E=%d experts must shard over %d ranks (E <= 256)", fn, desc->E, P);
    return MOE_ERR_INVALID_ARG;
  }
  if ((int64_t)P * desc->S * desc->k > rows) {
    set_error("%s: buffer of %lld rows < nranks*S*k = %lld (the worst case)", fn, (long long)rows,
              (long long)P * desc->S * desc->k);
    return MOE_ERR_INVALID_ARG;
  }
  *ds = dtype == MOE_F32 ? 4 : 2;
  if (((long long)d * *ds) % 16 != 0 || reinterpret_cast<uintptr_t>(a) % 16 ||
      reinterpret_cast<uintptr_t>(buf) % 16) {
    set_error("%s: rows and pointers must be 16-byte aligned", fn);
    return MOE_ERR_ALIGNMENT;
  }
  return symm_peers(fn, comm, buf, (size_t)rows * d * *ds, peers);
}

// Padded one-sided dispatch after the entry barrier (shared by the dispatch,
// the fused gate + dispatch and the push-form combine adjoint's dy scatter):
// rows into the owners' `dst` by `rows` (k_layout in peer mode, or the fused
// gate + layout kernel), then (unless NO_EXIT) the exit barrier, the owners'
// duplicate-row copies and local padding.  *dup_pending: copies enqueued.
using RowLauncher = std::function<moe_status_t(cudaStream_t, const PeerPtrs* pad_tab,
                                               const PeerPtrs* dup_tab, const PeerPtrs* wt_tab)>;

static moe_status_t dispatch_body(moe_comm* comm, const moe_gate_desc_t& D, int row_bytes,
                                  const PeerPtrs& dst, int32_t flags, cudaStream_t stream,
                                  RowLauncher rows, bool* dup_pending) {
  const int P = comm->nranks, r = comm->rank, El = D.E / P;
  const bool exit_bar = !(flags & MOE_P2P_NO_EXIT_BARRIER);
  // local padding: the zero rows are written by their owner after the exit
  // barrier instead of crossing NVLink (needs that barrier; E/P <= 256).
  // Default when at least ~5% of the rows are padding whatever the routing
  // (E*cap > 1.05*S*k, e.g. the hash config's C = 1.25: C4b dispatch 165 ->
  // 132 us at N=2); with C = 1 the padding is only the imbalance and the
  // extra kernel costs more than it saves (C2: +1.7 us).
  bool local_pad = exit_bar && El <= kPadTabStride && local_pad_on(D);
  // dedupe: k >= 2 and two experts can share an owner; the owners' copies
  // need the exit barrier
  bool dedupe = exit_bar && P >= 2 && D.k >= 2 && El >= 2 && tuning().p2p_dedupe;
  PeerPtrs tab{}, dup{}, wts{};
  int* pairs_mine = nullptr;
  moe_status_t s = MOE_OK;
  if (local_pad || dedupe) {
    const RecvTables* t =
        recv_tables(comm, dst.p[r], dedupe ? (size_t)D.E * D.capacity : 0, stream, &s);
    if (s != MOE_OK) return s;
    if (!t) {
      local_pad = dedupe = false;
    } else {
      for (int q = 0; q < P; ++q) {
        tab.p[q] = t->buf.peer.p[q];
        dup.p[q] = t->dup(q);
        wts.p[q] = t->wts(q);
      }
      pairs_mine = reinterpret_cast<int*>(t->pairs(r));
    }
  }
  s = run_or_queue(comm, stream, [=](cudaStream_t st) {
    return rows(st, local_pad ? &tab : nullptr, dedupe ? &dup : nullptr, dedupe ? &wts : nullptr);
  });
  if (s != MOE_OK) return s;
  *dup_pending = false;
  if (!exit_bar) return MOE_OK;
  s = comm_barrier(comm, stream);  // every row has landed
  if (s != MOE_OK) return s;
  const long long nrows = (long long)D.E * D.capacity;
  char* mine = dst.p[r];
  if (dedupe) {
    int* dtab = reinterpret_cast<int*>(dup.p[r]);
    s = run_or_queue(comm, stream, [=](cudaStream_t st) {
      return dup_fill_launch(mine, dtab, nrows, row_bytes, st, pairs_mine);
    });
    if (s != MOE_OK) return s;
    *dup_pending = true;
  }
  if (!local_pad) return MOE_OK;
  const int* ptab = reinterpret_cast<const int*>(tab.p[r]);
  const int cap = D.capacity;
  return run_or_queue(comm, stream, [=](cudaStream_t st) {
    return pad_fill_launch(mine, ptab, P, El, cap, row_bytes, st);
  });
}

// k_layout in peer mode as the dispatch's row kernel
static RowLauncher layout_rows(const moe_gate_desc_t& D, const moe_routing_t& R, const void* x,
                               int ds, int d, const PeerPtrs& dst, int El, int r) {
  return [=](cudaStream_t st, const PeerPtrs* pad, const PeerPtrs* dup, const PeerPtrs* wt) {
    return layout_launch_peers(D, R, x, ds, d, dst, El, r, st, nullptr, nullptr, pad, dup, wt);
  };
}

}  // namespace moe

using namespace moe;

extern "C" {

moe_status_t moe_comm_symm_alloc(moe_comm_t* comm, size_t bytes, void** out) {
  if (!comm || !out || bytes == 0) {
    set_error("moe_comm_symm_alloc: bad arguments");
    return MOE_ERR_INVALID_ARG;
  }
  moe_status_t s = need_p2p("moe_comm_symm_alloc", comm);
  if (s != MOE_OK) return s;
  SymmBuf b;
  s = symm_alloc(comm, bytes, &b);
  if (s != MOE_OK) return s;
  comm->symm.push_back(b);
  *out = b.base;
  return MOE_OK;
}

moe_status_t moe_comm_symm_free(moe_comm_t* comm, void* p) {
  if (!comm || !p) {
    set_error("moe_comm_symm_free: bad arguments");
    return MOE_ERR_INVALID_ARG;
  }
  for (size_t i = 0; i < comm->symm.size(); ++i) {
    if (comm->symm[i].base == p) {
      // the side tables of receive buffers inside it go first (collective)
      moe_status_t s = release_tables_in(comm, comm->symm[i].base, comm->symm[i].bytes);
      moe_status_t s2 = symm_release_coll(comm, comm->symm[i]);
      comm->symm.erase(comm->symm.begin() + i);
      return s != MOE_OK ? s : s2;
    }
  }
  set_error("moe_comm_symm_free: %p is not a symmetric buffer of this communicator", p);
  return MOE_ERR_INVALID_ARG;
}

moe_status_t moe_comm_barrier(moe_comm_t* comm, moe_stream_t stream) {
  moe_status_t s = need_p2p("moe_comm_barrier", comm);
  if (s != MOE_OK) return s;
  return comm_barrier(comm, reinterpret_cast<cudaStream_t>(stream));
}

moe_status_t moe_dispatch_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                              const moe_routing_t* routing, const void* x, int32_t d,
                              int32_t dtype, void* recv, int32_t flags, moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  PeerPtrs dst;
  int ds = 0;
  moe_status_t s = p2p_args("moe_dispatch_p2p", comm, desc, routing, x, recv, d, dtype, &dst, &ds);
  if (s != MOE_OK) return s;
  if (!routing->load) {
    set_error("moe_dispatch_p2p: routing.load is NULL");
    return MOE_ERR_INVALID_ARG;
  }
  if (!(flags & MOE_P2P_NO_ENTRY_BARRIER)) {  // every owner is ready to receive
    s = comm_barrier(comm, stream);
    if (s != MOE_OK) return s;
  }
  bool dup_pending = false;
  s = dispatch_body(comm, *desc, d * ds, dst, flags, stream,
                    layout_rows(*desc, *routing, x, ds, d, dst, desc->E / comm->nranks, comm->rank),
                    &dup_pending);
  if (s != MOE_OK) return s;
  comm->dup_recv = dup_pending ? recv : nullptr;
  return MOE_OK;
}

moe_status_t moe_combine_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                             const moe_routing_t* routing, const void* expert_out, int32_t d,
                             int32_t dtype, void* y, int32_t flags, moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  PeerPtrs src;
  int ds = 0;
  moe_status_t s = p2p_args("moe_combine_p2p", comm, desc, routing, y, expert_out, d, dtype, &src,
                            &ds);
  if (s != MOE_OK) return s;
  if (!routing->weight) {
    set_error("moe_combine_p2p: routing.weight is NULL");
    return MOE_ERR_INVALID_ARG;
  }
  const int P = comm->nranks, r = comm->rank;
  // A dispatch that sent duplicate rows once left their copies to the owners
  // (k_dup_fill after its exit barrier).  Unless the caller says recv still
  // holds exactly what that dispatch sent (MOE_P2P_RECV_UNMODIFIED: no
  // expert wrote it), those copies must be complete before any read, so the
  // entry barrier is kept even under NO_ENTRY_BARRIER.  With
  // RECV_UNMODIFIED the combine reads such a slot from the row that was sent
  // (alias mode: the bytes are the same) and does not wait for the copies.
  const bool dup_pending = comm->dup_recv && comm->dup_recv == expert_out;
  comm->dup_recv = nullptr;
  const bool no_entry = flags & MOE_P2P_NO_ENTRY_BARRIER;
  const int alias = dup_pending && (flags & MOE_P2P_RECV_UNMODIFIED) ? 1 : 0;
  // Pre-combine (k = 2, an expert may have written the rows): every owner
  // first combines the token pairs the dispatch sent it once (k_precombine,
  // on its own rows, after its expert), so a token whose two slots sit on
  // one remote owner is one row read over NVLink; the symmetric pre-row
  // buffer is allocated with the receive buffer's tables on first use
  // outside capture (collectively).
  PeerPtrs pre{};
  bool pre_on = false;
  const int row_bytes = d * ds;
  if (dup_pending && !alias && desc->k == 2 && tuning().p2p_precombine &&
      reverse_kspec_used(*desc, row_bytes)) {
    RecvTables* t = nullptr;
    for (RecvTables& u : comm->tables)
      if (u.recv == expert_out) t = &u;
    const size_t want = (size_t)desc->E * desc->capacity * row_bytes;
    if (t && t->dup_rows >= (size_t)desc->E * desc->capacity && !(t->pre.base && t->pre_bytes >= want)) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(stream, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
        if (t->pre.base) {
          s = symm_release_coll(comm, t->pre);
          t->pre = SymmBuf{};
          if (s != MOE_OK) return s;
        }
        s = symm_alloc(comm, want, &t->pre);
        if (s != MOE_OK) {
          t->pre = SymmBuf{};
          return s;
        }
        t->pre_bytes = want;
      }
    }
    if (t && t->pre.base && t->pre_bytes >= want) {
      pre_on = true;
      for (int q = 0; q < P; ++q) pre.p[q] = t->pre.peer.p[q];
      const char* mine = static_cast<const char*>(expert_out);
      const int* pairs = reinterpret_cast<const int*>(t->pairs(r));
      const float* wts = reinterpret_cast<const float*>(t->wts(r));
      char* pre_mine = t->pre.peer.p[r];
      const long long nrows = (long long)desc->E * desc->capacity;
      s = run_or_queue(comm, stream, [=](cudaStream_t st) {
        return precombine_launch(mine, pairs, wts, pre_mine, nrows, row_bytes, dtype, st);
      });
      if (s != MOE_OK) return s;
    }
  }
  if (!no_entry || (dup_pending && !alias)) {  // every rank's expert is done
    s = comm_barrier(comm, stream);
    if (s != MOE_OK) return s;
  }
  const moe_gate_desc_t D = *desc;
  const moe_routing_t R = *routing;
  s = run_or_queue(comm, stream, [=](cudaStream_t st) {
    return reverse_launch_peers(D, R, src, D.E / P, r, dtype, ds, d, y, st, nullptr, nullptr,
                                alias, pre_on ? &pre : nullptr);
  });
  if (s != MOE_OK) return s;
  if (flags & MOE_P2P_NO_EXIT_BARRIER) return MOE_OK;
  return comm_barrier(comm, stream);  // nobody reads them any more
}

moe_status_t moe_gate_dispatch_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                   const moe_gate_inputs_t* in, const moe_routing_t* out,
                                   void* ws, size_t ws_bytes, const void* x, int32_t d,
                                   int32_t dtype, void* recv, int32_t flags, moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  moe_status_t s = gate_validate(desc, in, out, ws, ws_bytes);
  if (s != MOE_OK) return s;
  PeerPtrs dst;
  int ds = 0;
  s = p2p_args("moe_gate_dispatch_p2p", comm, desc, out, x, recv, d, dtype, &dst, &ds);
  if (s != MOE_OK) return s;
  if (!out->load) {
    set_error("moe_gate_dispatch_p2p: routing.load is NULL");
    return MOE_ERR_INVALID_ARG;
  }
  const moe_gate_desc_t D = *desc;
  const moe_gate_inputs_t I = *in;
  const moe_routing_t R = *out;
  if (!gate_layout_supported(D, d * ds)) {  // gate, then the dispatch
    s = run_or_queue(comm, stream, [=](cudaStream_t st) { return gate_launch(D, I, R, ws, st); });
    if (s != MOE_OK) return s;
    return moe_dispatch_p2p(comm, desc, out, x, d, dtype, recv, flags, stream_);
  }
  const int P = comm->nranks, r = comm->rank;
  if (!(flags & MOE_P2P_NO_ENTRY_BARRIER)) {
    s = comm_barrier(comm, stream);
    if (s != MOE_OK) return s;
  }
  bool dup_pending = false;
  s = dispatch_body(comm, D, d * ds, dst, flags, stream,
                    [=](cudaStream_t st, const PeerPtrs* pad, const PeerPtrs* dup,
                        const PeerPtrs* wt) {
                      return gate_layout_launch(D, I, R, ws, x, ds, d, dst, D.E / P, r, pad, dup,
                                                st, wt);
                    },
                    &dup_pending);
  if (s != MOE_OK) return s;
  comm->dup_recv = dup_pending ? recv : nullptr;
  return MOE_OK;
}

moe_status_t moe_combine_backward_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                      const moe_routing_t* routing, const void* dy,
                                      const void* expert_out, int32_t d, int32_t dtype,
                                      void* d_expert_out, float* d_weight, int32_t flags,
                                      moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const char* fn = "moe_combine_backward_p2p";
  PeerPtrs src, dst;
  int ds = 0;
  moe_status_t s = p2p_args(fn, comm, desc, routing, dy, expert_out, d, dtype, &src, &ds);
  if (s != MOE_OK) return s;
  s = p2p_args(fn, comm, desc, routing, dy, d_expert_out, d, dtype, &dst, &ds);
  if (s != MOE_OK) return s;
  if (!routing->weight || !routing->load || !d_weight) {
    set_error("%s: routing.weight, routing.load and d_weight are required", fn);
    return MOE_ERR_INVALID_ARG;
  }
  const int P = comm->nranks, r = comm->rank;
  if (!(flags & MOE_P2P_NO_ENTRY_BARRIER)) {
    s = comm_barrier(comm, stream);
    if (s != MOE_OK) return s;
  }
  const moe_gate_desc_t D = *desc;
  const moe_routing_t R = *routing;
  s = run_or_queue(comm, stream, [=](cudaStream_t st) {
    return combine_bwd_launch(D, R, dy, src, dst, D.E / P, r, dtype, ds, d, d_weight, st);
  });
  if (s != MOE_OK) return s;
  if (flags & MOE_P2P_NO_EXIT_BARRIER) return MOE_OK;
  return comm_barrier(comm, stream);
}

moe_status_t moe_combine_backward_push_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                           const moe_routing_t* routing, const void* dy,
                                           const void* expert_out, int32_t d, int32_t dtype,
                                           void* d_expert_out, float* wtab, float* dwtab,
                                           float* d_weight, int32_t flags, moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const char* fn = "moe_combine_backward_push_p2p";
  PeerPtrs src, dst, wt, dwt;
  int ds = 0;
  moe_status_t s = p2p_args(fn, comm, desc, routing, dy, expert_out, d, dtype, &src, &ds);
  if (s != MOE_OK) return s;
  s = p2p_args(fn, comm, desc, routing, dy, d_expert_out, d, dtype, &dst, &ds);
  if (s != MOE_OK) return s;
  if (!routing->weight || !routing->load || !d_weight || !wtab || !dwtab) {
    set_error("%s: routing.weight/load, wtab, dwtab and d_weight are required", fn);
    return MOE_ERR_INVALID_ARG;
  }
  const size_t tb = sizeof(float) * (size_t)desc->E * desc->capacity;
  s = symm_peers(fn, comm, wtab, tb, &wt);
  if (s != MOE_OK) return s;
  s = symm_peers(fn, comm, dwtab, tb, &dwt);
  if (s != MOE_OK) return s;
  const int P = comm->nranks, r = comm->rank;
  if (!(flags & MOE_P2P_NO_ENTRY_BARRIER)) {
    s = comm_barrier(comm, stream);
    if (s != MOE_OK) return s;
  }
  const moe_gate_desc_t D = *desc;
  const moe_routing_t R = *routing;
  // the slot weights to the experts' owners, then dy rows (the dispatch
  // kernel: a top-2 token's dy row goes once to an owner of both its
  // experts; padding rows zero, written by the owners themselves when
  // padding is heavy); exit barrier; the owners' duplicate copies, padding
  s = run_or_queue(comm, stream, [=](cudaStream_t st) {
    return push_bwd_launch(D, R, wt, dwt, nullptr, nullptr, nullptr, P, r, dtype, d * ds, 0, st);
  });
  if (s != MOE_OK) return s;
  bool dup_pending = false;
  s = dispatch_body(comm, D, d * ds, dst, 0, stream, layout_rows(D, R, dy, ds, d, dst, D.E / P, r),
                    &dup_pending);
  if (s != MOE_OK) return s;
  // owners: scale in place, dot with the local expert rows into the token
  // owners' dw tables; barrier; token owners gather d_weight
  char* deo = static_cast<char*>(d_expert_out);
  const char* eo = static_cast<const char*>(expert_out);
  s = run_or_queue(comm, stream, [=](cudaStream_t st) {
    return push_bwd_launch(D, R, wt, dwt, deo, eo, nullptr, P, r, dtype, d * ds, 1, st);
  });
  if (s != MOE_OK) return s;
  s = comm_barrier(comm, stream);  // dots landed, d_expert_out final
  if (s != MOE_OK) return s;
  return run_or_queue(comm, stream, [=](cudaStream_t st) {
    return push_bwd_launch(D, R, wt, dwt, nullptr, nullptr, d_weight, P, r, dtype, d * ds, 2, st);
  });
}

moe_status_t moe_dispatch_backward_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                       const moe_routing_t* routing, const void* d_recv,
                                       int32_t d, int32_t dtype, void* dx, int32_t flags,
                                       moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  PeerPtrs src;
  int ds = 0;
  moe_status_t s = p2p_args("moe_dispatch_backward_p2p", comm, desc, routing, dx, d_recv, d, dtype,
                            &src, &ds);
  if (s != MOE_OK) return s;
  const int P = comm->nranks, r = comm->rank;
  if (!(flags & MOE_P2P_NO_ENTRY_BARRIER)) {
    s = comm_barrier(comm, stream);
    if (s != MOE_OK) return s;
  }
  const moe_gate_desc_t D = *desc;
  moe_routing_t unit = *routing;
  unit.weight = nullptr;  // adjoint of the dispatch copy: unit-weight combine
  s = run_or_queue(comm, stream, [=](cudaStream_t st) {
    return reverse_launch_peers(D, unit, src, D.E / P, r, dtype, ds, d, dx, st);
  });
  if (s != MOE_OK) return s;
  if (flags & MOE_P2P_NO_EXIT_BARRIER) return MOE_OK;
  return comm_barrier(comm, stream);
}

moe_status_t moe_dispatch_packed_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                     const moe_routing_t* routing, const int32_t* offsets,
                                     int32_t* counts, int32_t* peer_base, int32_t* recv_offsets,
                                     const void* x, int32_t d, int32_t dtype, void* recv,
                                     int64_t recv_cap_rows, int32_t flags, moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const char* fn = "moe_dispatch_packed_p2p";
  PeerPtrs dst, cnt;
  int ds = 0;
  moe_status_t s = packed_args(fn, comm, desc, routing, offsets, x, recv, recv_cap_rows, d, dtype,
                               &dst, &ds);
  if (s != MOE_OK) return s;
  if (!counts || !peer_base || !recv_offsets) {
    set_error("%s: counts, peer_base and recv_offsets are required", fn);
    return MOE_ERR_INVALID_ARG;
  }
  s = symm_peers(fn, comm, counts, sizeof(int32_t) * (size_t)desc->E, &cnt);
  if (s != MOE_OK) return s;
  const int P = comm->nranks, r = comm->rank, El = desc->E / P;
  if (!(flags & MOE_P2P_NO_ENTRY_BARRIER)) {  // owners done with the previous step's tables
    s = comm_barrier(comm, stream);
    if (s != MOE_OK) return s;
  }
  const moe_gate_desc_t D = *desc;
  const moe_routing_t R = *routing;
  s = run_or_queue(comm, stream, [=](cudaStream_t st) {
    k_a2av_counts<<<1, 256, 0, st>>>(offsets, cnt, D.E, El, r);
    MOE_CHECK_LAUNCH("moe_dispatch_packed_p2p: counts launch");
    return MOE_OK;
  });
  if (s != MOE_OK) return s;
  s = comm_barrier(comm, stream);  // every table complete
  if (s != MOE_OK) return s;
  s = run_or_queue(comm, stream, [=](cudaStream_t st) {
    k_a2av_plan<<<1, 256, 0, st>>>(cnt, P, El, r, peer_base, recv_offsets);
    MOE_CHECK_LAUNCH("moe_dispatch_packed_p2p: plan launch");
    return layout_launch_peers(D, R, x, ds, d, dst, El, r, st, offsets, peer_base);
  });
  if (s != MOE_OK) return s;
  if (flags & MOE_P2P_NO_EXIT_BARRIER) return MOE_OK;
  return comm_barrier(comm, stream);  // every row has landed
}

moe_status_t moe_combine_packed_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                    const moe_routing_t* routing, const int32_t* offsets,
                                    const int32_t* peer_base, const void* expert_out, int32_t d,
                                    int32_t dtype, int64_t expert_out_rows, void* y,
                                    int32_t flags, moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const char* fn = "moe_combine_packed_p2p";
  PeerPtrs src;
  int ds = 0;
  moe_status_t s = packed_args(fn, comm, desc, routing, offsets, y, expert_out, expert_out_rows, d,
                               dtype, &src, &ds);
  if (s != MOE_OK) return s;
  if (!routing->weight || !peer_base) {
    set_error("%s: routing.weight and peer_base are required", fn);
    return MOE_ERR_INVALID_ARG;
  }
  const int P = comm->nranks, r = comm->rank;
  if (!(flags & MOE_P2P_NO_ENTRY_BARRIER)) {
    s = comm_barrier(comm, stream);
    if (s != MOE_OK) return s;
  }
  const moe_gate_desc_t D = *desc;
  const moe_routing_t R = *routing;
  s = run_or_queue(comm, stream, [=](cudaStream_t st) {
    return reverse_launch_peers(D, R, src, D.E / P, r, dtype, ds, d, y, st, offsets, peer_base);
  });
  if (s != MOE_OK) return s;
  if (flags & MOE_P2P_NO_EXIT_BARRIER) return MOE_OK;
  return comm_barrier(comm, stream);
}

moe_status_t moe_combine_packed_backward_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                            const moe_routing_t* routing, const int32_t* offsets,
                                            const int32_t* peer_base, const void* dy,
                                            const void* expert_out, int32_t d, int32_t dtype,
                                            int64_t rows, void* d_expert_out, float* d_weight,
                                            int32_t flags, moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const char* fn = "moe_combine_packed_backward_p2p";
  PeerPtrs src, dst;
  int ds = 0;
  moe_status_t s = packed_args(fn, comm, desc, routing, offsets, dy, expert_out, rows, d, dtype,
                               &src, &ds);
  if (s != MOE_OK) return s;
  s = packed_args(fn, comm, desc, routing, offsets, dy, d_expert_out, rows, d, dtype, &dst, &ds);
  if (s != MOE_OK) return s;
  if (!routing->weight || !peer_base || !d_weight) {
    set_error("%s: routing.weight, peer_base and d_weight are required", fn);
    return MOE_ERR_INVALID_ARG;
  }
  const int P = comm->nranks, r = comm->rank;
  if (!(flags & MOE_P2P_NO_ENTRY_BARRIER)) {
    s = comm_barrier(comm, stream);
    if (s != MOE_OK) return s;
  }
  const moe_gate_desc_t D = *desc;
  const moe_routing_t R = *routing;
  s = run_or_queue(comm, stream, [=](cudaStream_t st) {
    return combine_bwd_launch(D, R, dy, src, dst, D.E / P, r, dtype, ds, d, d_weight, st, offsets,
                              peer_base);
  });
  if (s != MOE_OK) return s;
  if (flags & MOE_P2P_NO_EXIT_BARRIER) return MOE_OK;
  return comm_barrier(comm, stream);
}

moe_status_t moe_dispatch_packed_backward_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                             const moe_routing_t* routing, const int32_t* offsets,
                                             const int32_t* peer_base, const void* d_recv,
                                             int32_t d, int32_t dtype, int64_t rows, void* dx,
                                             int32_t flags, moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const char* fn = "moe_dispatch_packed_backward_p2p";
  PeerPtrs src;
  int ds = 0;
  moe_status_t s = packed_args(fn, comm, desc, routing, offsets, dx, d_recv, rows, d, dtype, &src,
                               &ds);
  if (s != MOE_OK) return s;
  if (!peer_base) {
    set_error("%s: peer_base is required", fn);
    return MOE_ERR_INVALID_ARG;
  }
  const int P = comm->nranks, r = comm->rank;
  if (!(flags & MOE_P2P_NO_ENTRY_BARRIER)) {
    s = comm_barrier(comm, stream);
    if (s != MOE_OK) return s;
  }
  const moe_gate_desc_t D = *desc;
  moe_routing_t unit = *routing;
  unit.weight = nullptr;
  s = run_or_queue(comm, stream, [=](cudaStream_t st) {
    return reverse_launch_peers(D, unit, src, D.E / P, r, dtype, ds, d, dx, st, offsets, peer_base);
  });
  if (s != MOE_OK) return s;
  if (flags & MOE_P2P_NO_EXIT_BARRIER) return MOE_OK;
  return comm_barrier(comm, stream);
}

}  // extern "C"
