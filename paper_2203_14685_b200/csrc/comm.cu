// comm.cu -- moe_alltoall: Alg. 1 steps 3 and 5 over
// NCCL point-to-point on NVLink 5 / NVSwitch: flat (Fig. 5),
// the paper's hierarchical leader scheme (Fig. 6)
// mimicked with groups of G consecutive ranks on one box (R13), and the
// two-level decoupled form ("fully utilizes the intra-node ...
// and inter-node bandwidth"): an intra-group exchange followed by one
// exchange per group pair between ranks of equal local index (R21).
//
// Every algorithm is a host-side schedule of ops (moe_a2a_op_t): the send /
// recv ops of one `phase` are issued as one NCCL group (comm_group), the
// local copies and chunk permutes of the phase follow in stream order.  The
// schedule is exported (moe_alltoall_plan) so the multi-process tests can
// execute the very same plan over gloo on CPUs, and it runs unchanged on a
// simulated communicator (sim.cu), where the groups are matched across the
// simulated ranks on one GPU.
#include <nccl.h>

#include <cstring>
#include <vector>

#include "comm.cuh"

namespace moe {

moe_status_t chunk_permute_launch(const void* src, void* dst, int N, int G, long long chunk_bytes,
                                  cudaStream_t stream);
moe_status_t chunk_transpose_launch(const void* src, void* dst, int X, int Y, long long chunk_bytes,
                                    cudaStream_t stream);
moe_status_t a2a_p2p_launch(const char* send, const PeerPtrs& recv, size_t recv_off_rank,
                            size_t bytes_per_peer, int nranks, int rank, cudaStream_t stream);
void symm_release(moe_comm* c, SymmBuf& b);

static moe_status_t nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return MOE_OK;
  set_error("%s: NCCL error %d (%s)", what, (int)r, ncclGetErrorString(r));
  return MOE_ERR_NCCL;
}

moe_status_t comm_group(moe_comm* c, std::vector<SimOp> ops, cudaStream_t stream) {
  if (ops.empty()) return MOE_OK;
  if (c->sim) {
    SimItem it;
    it.kind = SimItem::GROUP;
    it.ops = std::move(ops);
    c->queue.push_back(std::move(it));
    return MOE_OK;
  }
  moe_status_t s = nccl_status(ncclGroupStart(), "ncclGroupStart");
  if (s != MOE_OK) return s;
  for (const SimOp& o : ops) {
    ncclResult_t r = o.send ? ncclSend(o.ptr, o.bytes, ncclInt8, o.peer, c->nccl, stream)
                            : ncclRecv(o.ptr, o.bytes, ncclInt8, o.peer, c->nccl, stream);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return nccl_status(r, "ncclSend/ncclRecv");
    }
  }
  return nccl_status(ncclGroupEnd(), "ncclGroupEnd");
}

enum { OP_SEND = 0, OP_RECV = 1, OP_COPY = 2, OP_PERMUTE = 3, OP_TRANSPOSE = 4 };
enum { BUF_SEND = 0, BUF_RECV = 1, BUF_A = 2, BUF_B = 3 };

static void push(std::vector<moe_a2a_op_t>& v, int phase, int op, int peer, int sb, int db,
                 long long so, long long dof, long long n) {
  moe_a2a_op_t o;
  o.phase = phase;
  o.op = op;
  o.peer = peer;
  o.src_buf = sb;
  o.dst_buf = db;
  o.src_off = so;
  o.dst_off = dof;
  o.chunks = n;
  v.push_back(o);
}

// FLAT: one phase; rank r sends chunk q of its send buffer to q and receives
// chunk q of its recv buffer from q (self included: NCCL copies it in the
// same group, overlapped with the peer transfers).
//
// HIER_LEADER (N = P/G groups, leader = local rank 0 of each group):
//  phase 0  (1)+(2) members -> leader: member m of group g sends, for every
//           destination group h, its G chunks [hG, hG+G) into leader staging
//           A[h][m][0..G)  ("reorder by destination node" costs nothing);
//  phase 1  (3) leader g sends A[h] (G*G chunks = B*G/N bytes)
//           to leader h and receives leader h's block into B[h]:
//           B[g'][m][n] = chunk for (dst local n) from source rank g'G+m;
//  phase 2  (4) permute B[g'][m][n] -> A[n][g'][m]   (k_chunk_permute)
//  phase 3  (5) leader sends A[n] (P chunks, ascending source rank) to member
//           n; its own A[0] is copied into its recv buffer.
//
// HIER_2D (rank r = (g, m), N groups of G; every rank works, no leader):
//  phase 0  transpose send [h][m'] -> A [m'][h]           (k_chunk_transpose)
//  phase 1  intra-group: send A[m'] (N chunks: for ranks (h, m')) to (g, m'),
//           receive B[m] from (g, m): B[m][h] = chunk (g,m) -> (h, m_self)
//  phase 2  transpose B [m][h] -> A [h][m]
//  phase 3  inter-group, equal local index: send A[h] (G chunks, B*G/P
//           bytes) to (h, m_self), receive recv[h*G .. h*G+G) from (h, m_self):
//           the chunks of sources (h, 0..G-1), ascending source rank.
static std::vector<moe_a2a_op_t> make_plan(int P, int r, int algo, int G) {
  std::vector<moe_a2a_op_t> v;
  if (algo == MOE_A2A_FLAT || P == 1) {
    for (int q = 0; q < P; ++q) {
      push(v, 0, OP_SEND, q, BUF_SEND, -1, q, 0, 1);
      push(v, 0, OP_RECV, q, -1, BUF_RECV, 0, q, 1);
    }
    return v;
  }
  const int N = P / G, g = r / G, m = r % G, leader = g * G;
  if (algo == MOE_A2A_HIER_2D) {
    push(v, 0, OP_TRANSPOSE, N, BUF_SEND, BUF_A, 0, 0, G);
    for (int mm = 0; mm < G; ++mm) {
      push(v, 1, OP_SEND, g * G + mm, BUF_A, -1, (long long)mm * N, 0, N);
      push(v, 1, OP_RECV, g * G + mm, -1, BUF_B, 0, (long long)mm * N, N);
    }
    push(v, 2, OP_TRANSPOSE, G, BUF_B, BUF_A, 0, 0, N);
    for (int h = 0; h < N; ++h) {
      push(v, 3, OP_SEND, h * G + m, BUF_A, -1, (long long)h * G, 0, G);
      push(v, 3, OP_RECV, h * G + m, -1, BUF_RECV, 0, (long long)h * G, G);
    }
    return v;
  }
  // HIER_LEADER.  G == 1 (every rank a leader) and G == P (one group:
  // gather + scatter only) are valid degenerate forms.
  const long long GG = (long long)G * G;
  // phase 0
  if (m != 0) {
    for (int h = 0; h < N; ++h) push(v, 0, OP_SEND, leader, BUF_SEND, -1, (long long)h * G, 0, G);
  } else {
    for (int mm = 0; mm < G; ++mm)
      for (int h = 0; h < N; ++h) {
        const long long dst = (long long)h * GG + (long long)mm * G;
        if (mm == 0)
          push(v, 0, OP_COPY, -1, BUF_SEND, BUF_A, (long long)h * G, dst, G);
        else
          push(v, 0, OP_RECV, leader + mm, -1, BUF_A, 0, dst, G);
      }
    // phase 1: leader <-> leader
    for (int h = 0; h < N; ++h) {
      if (h == g) {
        push(v, 1, OP_COPY, -1, BUF_A, BUF_B, (long long)h * GG, (long long)g * GG, GG);
      } else {
        push(v, 1, OP_SEND, h * G, BUF_A, -1, (long long)h * GG, 0, GG);
        push(v, 1, OP_RECV, h * G, -1, BUF_B, 0, (long long)h * GG, GG);
      }
    }
    // phase 2: permute B -> A
    push(v, 2, OP_PERMUTE, N, BUF_B, BUF_A, 0, 0, G);
    // phase 3: scatter
    for (int n = 0; n < G; ++n) {
      if (n == 0)
        push(v, 3, OP_COPY, -1, BUF_A, BUF_RECV, 0, 0, P);
      else
        push(v, 3, OP_SEND, leader + n, BUF_A, -1, (long long)n * P, 0, P);
    }
  }
  if (m != 0) push(v, 3, OP_RECV, leader, -1, BUF_RECV, 0, 0, P);
  return v;
}

static bool algo_ok(int algo) {
  return algo == MOE_A2A_FLAT || algo == MOE_A2A_HIER_LEADER || algo == MOE_A2A_P2P ||
         algo == MOE_A2A_HIER_2D;
}

}  // namespace moe

using namespace moe;

extern "C" {

moe_status_t moe_comm_unique_id(uint8_t id[128]) {
  if (!id) {
    set_error("moe_comm_unique_id: id is NULL");
    return MOE_ERR_INVALID_ARG;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  moe_status_t s = nccl_status(ncclGetUniqueId(&u), "moe_comm_unique_id");
  if (s == MOE_OK) std::memcpy(id, &u, 128);
  return s;
}

moe_status_t moe_comm_init(const uint8_t id[128], int32_t nranks, int32_t rank, moe_comm_t** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("moe_comm_init: bad arguments (nranks=%d rank=%d)", nranks, rank);
    return MOE_ERR_INVALID_ARG;
  }
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  int dev = 0;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce != cudaSuccess) return cuda_status(ce, "moe_comm_init: cudaGetDevice");
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 1;
  const moe_tuning_t& tu = tuning();
  if (tu.nccl_max_ctas > 0) cfg.maxCTAs = tu.nccl_max_ctas;
  if (tu.nccl_min_ctas > 0) cfg.minCTAs = tu.nccl_min_ctas;
  if (tu.nccl_cta_policy >= 0) cfg.CTAPolicy = tu.nccl_cta_policy;
  ncclComm_t c;
  moe_status_t s = nccl_status(ncclCommInitRankConfig(&c, nranks, u, rank, &cfg), "moe_comm_init");
  if (s != MOE_OK) return s;
  moe_comm_t* m = new moe_comm_t();
  m->nccl = c;
  m->nranks = nranks;
  m->rank = rank;
  m->device = dev;
  m->sig = SymmBuf{};
  // Signal words of the device-side barrier (one-sided NVLink path).  If the
  // GPUs cannot map each other's memory, that path is reported unsupported;
  // the NCCL path still works.  Every rank tries, so the collective
  // handle exchange inside symm_alloc stays matched.
  m->p2p_ok = false;
  if (nranks <= kMaxRanks && !tuning().disable_p2p) {
    moe_status_t ss = symm_alloc(m, kSigBytes, &m->sig);
    m->p2p_ok = ss == MOE_OK;
  }
  *out = m;
  return MOE_OK;
}

static void release_regs(moe_comm_t* comm) {
  for (auto& pr : comm->regs) {
    if (pr.second) ncclCommDeregister(comm->nccl, pr.second);
    ncclMemFree(pr.first);
  }
  comm->regs.clear();
}

moe_status_t moe_comm_destroy(moe_comm_t* comm) {
  if (!comm) return MOE_OK;
  if (comm->sim) {
    set_error("moe_comm_destroy: a simulated rank is owned by its world (moe_sim_world_destroy)");
    return MOE_ERR_INVALID_ARG;
  }
  cudaDeviceSynchronize();
  release_regs(comm);
  for (SymmBuf& b : comm->symm) symm_release(comm, b);
  if (comm->sig.base) symm_release(comm, comm->sig);
  for (RecvTables& t : comm->tables) {
    symm_release(comm, t.buf);
    if (t.pre.base) symm_release(comm, t.pre);
  }
  moe_status_t s = nccl_status(ncclCommDestroy(comm->nccl), "moe_comm_destroy");
  delete comm;
  return s;
}

moe_status_t moe_comm_check(moe_comm_t* comm, moe_stream_t stream) {
  if (!comm) {
    set_error("moe_comm_check: comm is NULL");
    return MOE_ERR_INVALID_ARG;
  }
  cudaError_t e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_status(e, "moe_comm_check: stream");
  if (comm->sig.base) {
    unsigned w = 0;
    e = cudaMemcpy(&w, comm->sig.base + kErrOff, sizeof w, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_status(e, "moe_comm_check: error word");
    if (w & kErrBarrierTimeout) {
      set_error("moe_comm_check: rank %d: a device barrier gave up after %d ms waiting for a "
                "peer (a rank died, hung, or skipped a matching call); abort the communicator",
                comm->rank, tuning().barrier_timeout_ms);
      return MOE_ERR_TIMEOUT;
    }
  }
  if (comm->nccl) {
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError(comm->nccl, &ar);
    if (r != ncclSuccess) return nccl_status(r, "moe_comm_check: ncclCommGetAsyncError");
    if (ar != ncclSuccess && ar != ncclInProgress)
      return nccl_status(ar, "moe_comm_check: asynchronous NCCL error");
  }
  return MOE_OK;
}

moe_status_t moe_comm_abort(moe_comm_t* comm) {
  if (!comm) return MOE_OK;
  if (comm->sim) {
    set_error("moe_comm_abort: a simulated rank is owned by its world (moe_sim_world_destroy)");
    return MOE_ERR_INVALID_ARG;
  }
  // NCCL first: it unblocks this rank's NCCL kernels, so the device drains
  moe_status_t s = nccl_status(ncclCommAbort(comm->nccl), "moe_comm_abort");
  cudaDeviceSynchronize();
  for (auto& pr : comm->regs) ncclMemFree(pr.first);  // the registrations died with the comm
  comm->regs.clear();
  for (SymmBuf& b : comm->symm) symm_release(comm, b);
  if (comm->sig.base) symm_release(comm, comm->sig);
  for (RecvTables& t : comm->tables) {
    symm_release(comm, t.buf);
    if (t.pre.base) symm_release(comm, t.pre);
  }
  delete comm;
  return s;
}

moe_status_t moe_comm_mem_alloc(moe_comm_t* comm, size_t bytes, void** out) {
  if (!comm || !out || bytes == 0) {
    set_error("moe_comm_mem_alloc: bad arguments");
    return MOE_ERR_INVALID_ARG;
  }
  if (comm->sim) {  // simulated ranks: plain device memory
    cudaError_t e = cudaMalloc(out, bytes);
    if (e != cudaSuccess) return cuda_status(e, "moe_comm_mem_alloc");
    comm->regs.emplace_back(*out, nullptr);
    return MOE_OK;
  }
  void* p = nullptr;
  moe_status_t s = nccl_status(ncclMemAlloc(&p, bytes), "moe_comm_mem_alloc: ncclMemAlloc");
  if (s != MOE_OK) return s;
  void* h = nullptr;
  s = nccl_status(ncclCommRegister(comm->nccl, p, bytes, &h), "moe_comm_mem_alloc: ncclCommRegister");
  if (s != MOE_OK) {
    ncclMemFree(p);
    return s;
  }
  comm->regs.emplace_back(p, h);
  *out = p;
  return MOE_OK;
}

moe_status_t moe_comm_mem_free(moe_comm_t* comm, void* p) {
  if (!comm || !p) {
    set_error("moe_comm_mem_free: bad arguments");
    return MOE_ERR_INVALID_ARG;
  }
  for (size_t i = 0; i < comm->regs.size(); ++i) {
    if (comm->regs[i].first != p) continue;
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_status(e, "moe_comm_mem_free: sync");
    moe_status_t s = MOE_OK;
    if (comm->sim) {
      cudaFree(p);
    } else {
      s = nccl_status(ncclCommDeregister(comm->nccl, comm->regs[i].second),
                      "moe_comm_mem_free: ncclCommDeregister");
      ncclMemFree(p);
    }
    comm->regs.erase(comm->regs.begin() + i);
    return s;
  }
  set_error("moe_comm_mem_free: %p was not allocated by moe_comm_mem_alloc", p);
  return MOE_ERR_INVALID_ARG;
}

moe_status_t moe_comm_size(const moe_comm_t* comm, int32_t* nranks, int32_t* rank) {
  if (!comm || !nranks || !rank) {
    set_error("moe_comm_size: NULL argument");
    return MOE_ERR_INVALID_ARG;
  }
  *nranks = comm->nranks;
  *rank = comm->rank;
  return MOE_OK;
}

size_t moe_alltoall_workspace_bytes(int32_t nranks, int32_t algo, int32_t group_size,
                                    size_t bytes_per_peer) {
  if (nranks < 1 || group_size < 1) return 0;
  if (algo == MOE_A2A_HIER_LEADER)
    return 2 * (size_t)group_size * (size_t)nranks * bytes_per_peer;
  if (algo == MOE_A2A_HIER_2D) return 2 * (size_t)nranks * bytes_per_peer;
  return 0;
}

moe_status_t moe_alltoall_plan(int32_t nranks, int32_t rank, int32_t algo, int32_t group_size,
                               moe_a2a_op_t* ops, int32_t capacity, int32_t* n_ops) {
  const bool hier = algo == MOE_A2A_HIER_LEADER || algo == MOE_A2A_HIER_2D;
  if (nranks < 1 || rank < 0 || rank >= nranks || !n_ops ||
      (algo != MOE_A2A_FLAT && !hier) ||
      (hier && (group_size < 1 || nranks % group_size != 0))) {
    set_error("moe_alltoall_plan: bad arguments (nranks=%d rank=%d algo=%d group_size=%d)", nranks,
              rank, algo, group_size);
    return MOE_ERR_INVALID_ARG;
  }
  std::vector<moe_a2a_op_t> v = make_plan(nranks, rank, algo, group_size);
  *n_ops = (int32_t)v.size();
  if (!ops || capacity < (int32_t)v.size()) {
    set_error("moe_alltoall_plan: need room for %d ops", (int)v.size());
    return MOE_ERR_INVALID_ARG;
  }
  std::memcpy(ops, v.data(), v.size() * sizeof(moe_a2a_op_t));
  return MOE_OK;
}

moe_status_t moe_alltoallv_plan(int32_t nranks, int32_t E, const int32_t* offsets,
                                const int32_t* recv_counts, int64_t* send_rows,
                                int64_t* recv_rows, int32_t* recv_offsets) {
  if (nranks < 1 || E < 1 || E % nranks != 0 || !offsets || !recv_counts || !send_rows ||
      !recv_rows || !recv_offsets) {
    set_error("moe_alltoallv_plan: need E %% nranks == 0 and non-NULL arrays (E=%d, nranks=%d)", E,
              nranks);
    return MOE_ERR_INVALID_ARG;
  }
  const int El = E / nranks;
  for (int e = 0; e < E; ++e)
    if (offsets[e + 1] < offsets[e] || recv_counts[e] < 0) {
      set_error("moe_alltoallv_plan: offsets must be non-decreasing and counts >= 0 (e=%d)", e);
      return MOE_ERR_INVALID_ARG;
    }
  long long acc = 0;
  recv_offsets[0] = 0;
  for (int q = 0; q < nranks; ++q) {
    send_rows[q] = (int64_t)offsets[(q + 1) * El] - offsets[q * El];
    long long rr = 0;
    for (int le = 0; le < El; ++le) {
      const int c = recv_counts[q * El + le];
      rr += c;
      acc += c;
      if (acc > 2147483647LL) {
        set_error("moe_alltoallv_plan: more than 2^31 receive rows");
        return MOE_ERR_UNSUPPORTED;
      }
      recv_offsets[q * El + le + 1] = (int32_t)acc;
    }
    recv_rows[q] = rr;
  }
  return MOE_OK;
}

moe_status_t moe_alltoallv(moe_comm_t* comm, const void* send, const int64_t* send_rows,
                           void* recv, const int64_t* recv_rows, size_t row_bytes,
                           moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (!comm || !send_rows || !recv_rows || row_bytes == 0) {
    set_error("moe_alltoallv: NULL comm/send_rows/recv_rows or row_bytes == 0");
    return MOE_ERR_INVALID_ARG;
  }
  const int P = comm->nranks;
  int64_t ns = 0, nr = 0;
  for (int q = 0; q < P; ++q) {
    if (send_rows[q] < 0 || recv_rows[q] < 0) {
      set_error("moe_alltoallv: negative row count for rank %d", q);
      return MOE_ERR_INVALID_ARG;
    }
    ns += send_rows[q];
    nr += recv_rows[q];
  }
  if ((ns && !send) || (nr && !recv)) {
    set_error("moe_alltoallv: NULL send/recv with rows to move");
    return MOE_ERR_INVALID_ARG;
  }
  std::vector<SimOp> ops;
  int64_t so = 0, ro = 0;
  for (int q = 0; q < P; ++q) {
    ops.push_back(SimOp{1, q, const_cast<char*>(static_cast<const char*>(send)) + so * row_bytes,
                        (size_t)send_rows[q] * row_bytes, 0});
    ops.push_back(SimOp{0, q, static_cast<char*>(recv) + ro * row_bytes,
                        (size_t)recv_rows[q] * row_bytes, 0});
    so += send_rows[q];
    ro += recv_rows[q];
  }
  return comm_group(comm, std::move(ops), stream);
}

moe_status_t moe_alltoall(moe_comm_t* comm, int32_t algo, int32_t group_size, const void* send,
                          void* recv, size_t bytes_per_peer, void* ws, size_t ws_bytes,
                          moe_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (!comm || !send || !recv) {
    set_error("moe_alltoall: NULL comm/send/recv");
    return MOE_ERR_INVALID_ARG;
  }
  const int P = comm->nranks, r = comm->rank;
  if (!algo_ok(algo)) {
    set_error("moe_alltoall: invalid algo %d", algo);
    return MOE_ERR_INVALID_ARG;
  }
  const bool hier = algo == MOE_A2A_HIER_LEADER || algo == MOE_A2A_HIER_2D;
  if (hier && (group_size < 1 || P % group_size != 0)) {
    set_error("moe_alltoall: nranks %d not divisible by group_size %d", P, group_size);
    return MOE_ERR_INVALID_ARG;
  }
  if (bytes_per_peer == 0) return MOE_OK;
  if (P == 1) {
    if (send == recv) return MOE_OK;
    return run_or_queue(comm, stream, [=](cudaStream_t st) {
      cudaError_t e = cudaMemcpyAsync(recv, send, bytes_per_peer, cudaMemcpyDeviceToDevice, st);
      return e == cudaSuccess ? MOE_OK : cuda_status(e, "moe_alltoall: self copy");
    });
  }
  if (send == recv) {
    set_error("moe_alltoall: in-place (send == recv) is not supported for nranks > 1");
    return MOE_ERR_INVALID_ARG;
  }
  if (algo == MOE_A2A_P2P) {
    if (!comm->p2p_ok) {
      set_error("moe_alltoall(P2P): peer memory is not available between these GPUs");
      return MOE_ERR_UNSUPPORTED;
    }
    if (bytes_per_peer % 16 != 0 || reinterpret_cast<uintptr_t>(send) % 16 ||
        reinterpret_cast<uintptr_t>(recv) % 16) {
      set_error("moe_alltoall(P2P): 16-byte aligned buffers and chunks required");
      return MOE_ERR_ALIGNMENT;
    }
    const SymmBuf* sb = find_symm(comm, recv, (size_t)P * bytes_per_peer);
    if (!sb) {
      set_error("moe_alltoall(P2P): recv is not inside a symmetric buffer (moe_comm_symm_alloc)");
      return MOE_ERR_INVALID_ARG;
    }
    PeerPtrs dst{};
    const size_t off = static_cast<const char*>(recv) - sb->base;
    for (int q = 0; q < P; ++q) dst.p[q] = sb->peer.p[q] + off;
    // entry barrier: no rank writes into a receive buffer before its owner's
    // stream has reached this call (the receive semantics of the NCCL path)
    moe_status_t s = comm_barrier(comm, stream);
    if (s != MOE_OK) return s;
    const char* sp = static_cast<const char*>(send);
    s = run_or_queue(comm, stream, [=](cudaStream_t st) {
      return a2a_p2p_launch(sp, dst, (size_t)r * bytes_per_peer, bytes_per_peer, P, r, st);
    });
    if (s != MOE_OK) return s;
    return comm_barrier(comm, stream);
  }
  const size_t need = moe_alltoall_workspace_bytes(P, algo, group_size, bytes_per_peer);
  const bool needs_ws = (algo == MOE_A2A_HIER_LEADER && r % group_size == 0) ||
                        algo == MOE_A2A_HIER_2D;
  if (needs_ws) {
    if (!ws || ws_bytes < need) {
      set_error("moe_alltoall: workspace %zu < %zu bytes", ws_bytes, need);
      return MOE_ERR_WORKSPACE;
    }
    if (bytes_per_peer % 16 != 0) {
      set_error("moe_alltoall: hierarchical algorithms need bytes_per_peer %% 16 == 0 (got %zu)",
                bytes_per_peer);
      return MOE_ERR_ALIGNMENT;
    }
  }
  if (algo == MOE_A2A_FLAT && tuning().nccl_alltoall && !comm->sim) {
    // NCCL's own AllToAll (2.28): the same bytes as the grouped send/recv
    return nccl_status(ncclAlltoAll(send, recv, bytes_per_peer, ncclInt8, comm->nccl, stream),
                       "moe_alltoall: ncclAlltoAll");
  }
  std::vector<moe_a2a_op_t> plan = make_plan(P, r, algo, group_size);
  const size_t b = bytes_per_peer;
  const size_t stage = need / 2;
  char* bufs[4] = {const_cast<char*>(static_cast<const char*>(send)), static_cast<char*>(recv),
                   static_cast<char*>(ws), ws ? static_cast<char*>(ws) + stage : nullptr};
  size_t i = 0;
  while (i < plan.size()) {
    const int phase = plan[i].phase;
    size_t jend = i;
    while (jend < plan.size() && plan[jend].phase == phase) ++jend;
    std::vector<SimOp> ops;
    for (size_t j = i; j < jend; ++j) {
      const moe_a2a_op_t& o = plan[j];
      if (o.op == OP_SEND)
        ops.push_back(SimOp{1, o.peer, bufs[o.src_buf] + o.src_off * b, (size_t)o.chunks * b, 0});
      else if (o.op == OP_RECV)
        ops.push_back(SimOp{0, o.peer, bufs[o.dst_buf] + o.dst_off * b, (size_t)o.chunks * b, 0});
    }
    moe_status_t s = comm_group(comm, std::move(ops), stream);
    if (s != MOE_OK) return s;
    for (size_t j = i; j < jend; ++j) {
      const moe_a2a_op_t o = plan[j];
      char* src = bufs[o.src_buf] + (o.op == OP_COPY ? o.src_off * b : 0);
      char* dst = bufs[o.dst_buf] + (o.op == OP_COPY ? o.dst_off * b : 0);
      if (o.op == OP_COPY) {
        s = run_or_queue(comm, stream, [=](cudaStream_t st) {
          cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)o.chunks * b, cudaMemcpyDeviceToDevice, st);
          return e == cudaSuccess ? MOE_OK : cuda_status(e, "moe_alltoall: local copy");
        });
      } else if (o.op == OP_PERMUTE) {
        s = run_or_queue(comm, stream, [=](cudaStream_t st) {
          return chunk_permute_launch(src, dst, o.peer, (int)o.chunks, (long long)b, st);
        });
      } else if (o.op == OP_TRANSPOSE) {
        s = run_or_queue(comm, stream, [=](cudaStream_t st) {
          return chunk_transpose_launch(src, dst, o.peer, (int)o.chunks, (long long)b, st);
        });
      }
      if (s != MOE_OK) return s;
    }
    i = jend;
  }
  return MOE_OK;
}

}  // extern "C"
