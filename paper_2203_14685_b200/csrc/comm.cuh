// comm.cuh -- the library-owned communicator (moe_comm_t): the NCCL
// communicator plus the symmetric (peer-mapped) buffers of the one-sided
// NVLink path and the device-side barrier's signal words.
#pragma once
#include <nccl.h>

#include <vector>

#include "common.cuh"

namespace moe {

constexpr int kMaxRanks = 32;
// The comm's signal buffer: barrier words at offset 0, then the padding-count
// table of the padded one-sided dispatch: [kMaxRanks source ranks][256 local
// experts] int32 (admitted rows per (source, local expert)).
constexpr size_t kPadTabOff = 4096;
constexpr int kPadTabStride = 256;
constexpr size_t kSigBytes = kPadTabOff + sizeof(int) * kMaxRanks * kPadTabStride;

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

moe_status_t barrier_launch(const PeerPtrs& sig, int nranks, int rank, cudaStream_t stream);

}  // namespace moe

struct moe_comm {
  ncclComm_t nccl;
  int nranks, rank, device;
  std::vector<moe::SymmBuf> symm;  // live symmetric buffers
  moe::SymmBuf sig;                // barrier signals: [kMaxRanks] flags + local epoch
  moe::SymmBuf dup{};              // one-sided dispatch: duplicate-row table (int32 per recv row)
  const void* dup_recv = nullptr;  // recv of the last dispatch whose owners fill duplicate rows
                                   // after its exit barrier (the combine must not skip its entry one)
  bool p2p_ok;                     // peer mappings could be made (NVLink / P2P)
};

namespace moe {

// The symmetric buffer containing [p, p + bytes), or nullptr.
inline const SymmBuf* find_symm(const moe_comm* c, const void* p, size_t bytes) {
  const char* q = static_cast<const char*>(p);
  for (const SymmBuf& b : c->symm)
    if (q >= b.base && q + bytes <= b.base + b.bytes) return &b;
  return nullptr;
}

}  // namespace moe
