// comm.cuh -- the library-owned communicator (moe_comm_t): the NCCL
// communicator plus the symmetric (peer-mapped) buffers of the one-sided
// NVLink path and the device-side barrier's signal words.
#pragma once
#include <nccl.h>

#include <functional>
#include <vector>

#include "common.cuh"

namespace moe {

constexpr int kMaxRanks = 32;
// The comm's signal buffer: barrier words at offset 0, the device error word
// of this rank (a barrier that timed out sets it) at kErrOff.
constexpr size_t kErrOff = 2048;
constexpr size_t kSigBytes = 4096;
// Side tables of a receive buffer of the padded one-sided dispatch
// (RecvTables): the padding-count table [kMaxRanks source ranks][256 local
// experts] int32 (admitted rows per (source, local expert)), then the
// duplicate-row table (int32 per recv row).
constexpr int kPadTabStride = 256;
constexpr size_t kPadTabBytes = sizeof(int) * kMaxRanks * kPadTabStride;
enum { kErrBarrierTimeout = 1 };

// P pointers to the same symmetric buffer as mapped on every rank
// (peer[r] == this rank's own allocation).  Passed to kernels by value.
struct PeerPtrs {
  char* p[kMaxRanks];
};

struct SymmBuf {
  char* base;
  size_t bytes;
  PeerPtrs peer;
};

// The side tables the senders of a padded one-sided dispatch write into an
// owner and the owner reads after the exit barrier (padding counts, duplicate
// rows), one set PER RECEIVE BUFFER: a caller that alternates two receive
// buffers may then drop the combine's exit barrier (moe.h, MOE_P2P_*).
struct RecvTables {
  const void* recv;   // this rank's receive buffer they belong to
  // [kPadTabBytes padding counts][dup_rows int32 duplicate-row table]
  // [dup_rows int32 pair table][dup_rows float slot weights]
  SymmBuf buf;
  size_t dup_rows;    // capacity of the per-row tables
  SymmBuf pre{};      // pre-combined rows of token pairs (moe_combine_p2p), lazily
  size_t pre_bytes = 0;
  char* dup(int q) const { return buf.peer.p[q] + kPadTabBytes; }
  char* pairs(int q) const { return dup(q) + dup_rows * sizeof(int); }
  char* wts(int q) const { return pairs(q) + dup_rows * sizeof(int); }
};

// One step of a rank's program on a SIMULATED communicator (moe_sim_*):
// calls on a simulated rank do not launch; they append their steps here and
// moe_sim_world_run executes every rank's program on one GPU, phase by
// phase: a BARRIER step waits until every rank reached its matching barrier;
// a GROUP step is one NCCL group of send/recv ops, matched across ranks in
// issue order per (source, destination) pair as NCCL matches them.
struct SimOp {
  int send;  // 1 = send, 0 = recv
  int peer;
  char* ptr;
  size_t bytes;
  int done;
};
struct SimItem {
  enum Kind { FN = 0, BARRIER = 1, GROUP = 2 } kind;
  std::function<moe_status_t(cudaStream_t)> fn;
  std::vector<SimOp> ops;
  int posted = 0, pending_sends = 0;
};

}  // namespace moe

struct moe_sim_world;

struct moe_comm {
  ncclComm_t nccl;
  int nranks, rank, device;
  std::vector<moe::SymmBuf> symm;  // live symmetric buffers
  moe::SymmBuf sig;                // barrier signals: [kMaxRanks] flags + local epoch
  std::vector<moe::RecvTables> tables;  // one-sided dispatch: side tables per receive buffer
  const void* dup_recv = nullptr;  // recv of the last dispatch whose owners fill duplicate rows
                                   // after its exit barrier (the combine must not skip its entry one)
  bool p2p_ok;                     // peer mappings could be made (NVLink / P2P)
  // simulated rank (moe_sim_world): no NCCL; calls queue their steps
  moe_sim_world* sim = nullptr;
  std::vector<moe::SimItem> queue;
  int sim_nalloc = 0;              // symmetric allocations made by this rank so far
  // NCCL-registered buffers of moe_comm_mem_alloc: (pointer, registration)
  std::vector<std::pair<void*, void*>> regs;
};

namespace moe {

// Run `fn` on `stream` now (a real communicator) or append it to a simulated
// rank's program (moe_sim_world_run executes it later, in order).
moe_status_t run_or_queue(moe_comm* c, cudaStream_t stream,
                          std::function<moe_status_t(cudaStream_t)> fn);
// The device barrier of all ranks (k_barrier, bounded by the tuning's
// barrier_timeout_ms), or a barrier step of a simulated rank.
moe_status_t comm_barrier(moe_comm* c, cudaStream_t stream);
// One NCCL group of send/recv ops (ncclGroupStart .. End), or a group step
// of a simulated rank.
moe_status_t comm_group(moe_comm* c, std::vector<SimOp> ops, cudaStream_t stream);
// Symmetric allocation over the communicator's ranks (CUDA IPC), or from the
// simulated world's per-rank buffers; release is collective too.
moe_status_t symm_alloc(moe_comm* c, size_t bytes, SymmBuf* out);
moe_status_t symm_release_coll(moe_comm* c, SymmBuf& b);

// The symmetric buffer containing [p, p + bytes), or nullptr.
inline const SymmBuf* find_symm(const moe_comm* c, const void* p, size_t bytes) {
  const char* q = static_cast<const char*>(p);
  for (const SymmBuf& b : c->symm)
    if (q >= b.base && q + bytes <= b.base + b.bytes) return &b;
  return nullptr;
}

}  // namespace moe
