// sim.cu -- simulated ranks (include/moe.h "simulated ranks"): TEST
// INFRASTRUCTURE that runs the multi-GPU path's real kernels for P ranks on
// one GPU, so the exchange steps of Algorithm 1 are
// parity-checked on a single B200.
//
// A simulated rank is an ordinary moe_comm with `sim` set: its symmetric
// buffers are P plain allocations on this device (buffer i of every rank is
// made when the first rank asks for it), and the library's entry points
// queue their steps instead of launching (run_or_queue, comm_barrier,
// comm_group in p2p.cu / comm.cu).  moe_sim_world_run interleaves the
// ranks' programs on one stream:
//   FN      a rank's kernel launch(es), in its call order;
//   BARRIER every rank must reach its next barrier before any goes on (the
//           device barrier becomes a step boundary: no kernel waits on
//           another, which a single GPU could not guarantee);
//   GROUP   one NCCL group: its sends are posted, its receives take the
//           oldest matching posted send of that (source, destination) pair
//           (NCCL's matching order) as a device copy; the group completes
//           when its receives are done and its sends were consumed.
// Stream order then gives every cross-rank dependency the real path gets
// from the barriers and NCCL.
#include <cstring>

#include "launch.cuh"

struct moe_sim_world {
  int P = 0;
  std::vector<moe_comm*> comms;
  // symmetric allocation i of every rank: P device pointers, bytes, and how
  // many ranks still hold it
  struct Slot {
    moe::PeerPtrs peer;
    size_t bytes;
    int held;
  };
  std::vector<Slot> slots;  // slot 0: every rank's signal buffer
};

namespace moe {

moe_status_t barrier_launch(const PeerPtrs& sig, int nranks, int rank, cudaStream_t stream);

moe_status_t sim_symm_alloc(moe_comm* c, size_t bytes, SymmBuf* out) {
  moe_sim_world* w = c->sim;
  bytes = (bytes + 4095) & ~(size_t)4095;
  const int i = c->sim_nalloc;
  if (i == (int)w->slots.size()) {  // the first rank to ask makes every rank's buffer
    moe_sim_world::Slot s{};
    s.bytes = bytes;
    s.held = w->P;
    for (int q = 0; q < w->P; ++q) {
      cudaError_t e = cudaMalloc(&s.peer.p[q], bytes);
      if (e == cudaSuccess) e = cudaMemset(s.peer.p[q], 0, bytes);
      if (e != cudaSuccess) {
        for (int u = 0; u <= q; ++u)
          if (s.peer.p[u]) cudaFree(s.peer.p[u]);
        return cuda_status(e, "simulated symmetric alloc");
      }
    }
    w->slots.push_back(s);
  } else if (i > (int)w->slots.size() || w->slots[i].bytes != bytes) {
    set_error("simulated symmetric alloc: rank %d's allocation #%d (%zu bytes) does not match the "
              "other ranks' (collective calls out of order)", c->rank, i, bytes);
    return MOE_ERR_INVALID_ARG;
  }
  ++c->sim_nalloc;
  const moe_sim_world::Slot& s = w->slots[i];
  SymmBuf b{};
  b.base = s.peer.p[c->rank];
  b.bytes = s.bytes;
  b.peer = s.peer;
  *out = b;
  return MOE_OK;
}

moe_status_t sim_symm_release(moe_comm* c, SymmBuf& b) {
  moe_sim_world* w = c->sim;
  for (moe_sim_world::Slot& s : w->slots) {
    if (s.peer.p[c->rank] != b.base) continue;
    if (--s.held == 0) {
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) return cuda_status(e, "simulated symmetric free");
      for (int q = 0; q < w->P; ++q) {
        cudaFree(s.peer.p[q]);
        s.peer.p[q] = nullptr;
      }
    }
    b.base = nullptr;
    return MOE_OK;
  }
  set_error("simulated symmetric free: not a buffer of rank %d", c->rank);
  return MOE_ERR_INVALID_ARG;
}

moe_status_t sim_barrier(moe_comm* c, cudaStream_t) {
  SimItem it;
  it.kind = SimItem::BARRIER;
  c->queue.push_back(std::move(it));
  return MOE_OK;
}

}  // namespace moe

using namespace moe;

extern "C" {

moe_status_t moe_sim_world_create(int32_t nranks, moe_sim_world_t** out) {
  if (!out || nranks < 1 || nranks > kMaxRanks) {
    set_error("moe_sim_world_create: nranks must be in 1..%d (got %d)", kMaxRanks, nranks);
    return MOE_ERR_INVALID_ARG;
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "moe_sim_world_create: cudaGetDevice");
  moe_sim_world* w = new moe_sim_world();
  w->P = nranks;
  for (int r = 0; r < nranks; ++r) {
    moe_comm* c = new moe_comm();
    c->nccl = nullptr;
    c->nranks = nranks;
    c->rank = r;
    c->device = dev;
    c->sim = w;
    c->p2p_ok = true;
    w->comms.push_back(c);
  }
  // the barrier words, error word and padding-count tables: allocation #0
  for (int r = 0; r < nranks; ++r) {
    moe_status_t s = sim_symm_alloc(w->comms[r], kSigBytes, &w->comms[r]->sig);
    if (s != MOE_OK) {
      moe_sim_world_destroy(w);
      return s;
    }
  }
  *out = w;
  return MOE_OK;
}

moe_status_t moe_sim_world_comm(moe_sim_world_t* w, int32_t rank, moe_comm_t** out) {
  if (!w || !out || rank < 0 || rank >= w->P) {
    set_error("moe_sim_world_comm: bad arguments (rank=%d)", rank);
    return MOE_ERR_INVALID_ARG;
  }
  *out = w->comms[rank];
  return MOE_OK;
}

moe_status_t moe_sim_live_barrier(moe_sim_world_t* w, int32_t rank, moe_stream_t stream) {
  if (!w || rank < 0 || rank >= w->P) {
    set_error("moe_sim_live_barrier: bad arguments (rank=%d)", rank);
    return MOE_ERR_INVALID_ARG;
  }
  moe_comm* c = w->comms[rank];
  return barrier_launch(c->sig.peer, w->P, rank, reinterpret_cast<cudaStream_t>(stream));
}

moe_status_t moe_sim_world_run(moe_sim_world_t* w, moe_stream_t stream_) {
  if (!w) {
    set_error("moe_sim_world_run: world is NULL");
    return MOE_ERR_INVALID_ARG;
  }
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const int P = w->P;
  std::vector<size_t> pos(P, 0);
  // posted, not yet consumed sends per (src, dst): (item, op index)
  struct Posted {
    SimItem* item;
    int op;
  };
  std::vector<std::vector<Posted>> posted((size_t)P * P);
  moe_status_t st = MOE_OK;
  auto fail = [&](moe_status_t s) {
    for (moe_comm* c : w->comms) c->queue.clear();
    return s;
  };
  for (;;) {
    bool progress = false;
    for (int r = 0; r < P; ++r) {
      std::vector<SimItem>& q = w->comms[r]->queue;
      while (pos[r] < q.size()) {
        SimItem& it = q[pos[r]];
        if (it.kind == SimItem::FN) {
          st = it.fn(stream);
          if (st != MOE_OK) return fail(st);
          ++pos[r];
          progress = true;
          continue;
        }
        if (it.kind == SimItem::BARRIER) break;
        // GROUP
        if (!it.posted) {
          it.posted = 1;
          for (int k = 0; k < (int)it.ops.size(); ++k) {
            const SimOp& o = it.ops[k];
            if (o.peer < 0 || o.peer >= P) {
              set_error("moe_sim_world_run: rank %d addresses rank %d of %d", r, o.peer, P);
              return fail(MOE_ERR_INVALID_ARG);
            }
            if (o.send) {
              posted[(size_t)r * P + o.peer].push_back(Posted{&it, k});
              ++it.pending_sends;
            }
          }
          progress = true;
        }
        bool recvs_done = true;
        for (SimOp& o : it.ops) {
          if (o.send || o.done) continue;
          std::vector<Posted>& pq = posted[(size_t)o.peer * P + r];
          if (pq.empty()) {
            recvs_done = false;
            continue;
          }
          Posted ps = pq.front();
          pq.erase(pq.begin());
          const SimOp& so = ps.item->ops[ps.op];
          if (so.bytes != o.bytes) {
            set_error("moe_sim_world_run: rank %d sends %zu bytes to rank %d, which receives %zu",
                      o.peer, so.bytes, r, o.bytes);
            return fail(MOE_ERR_INVALID_ARG);
          }
          if (o.bytes) {
            cudaError_t e = cudaMemcpyAsync(o.ptr, so.ptr, o.bytes, cudaMemcpyDeviceToDevice, stream);
            if (e != cudaSuccess) return fail(cuda_status(e, "moe_sim_world_run: copy"));
          }
          o.done = 1;
          --ps.item->pending_sends;
          progress = true;
        }
        if (recvs_done && it.pending_sends == 0) {
          ++pos[r];
          progress = true;
          continue;
        }
        break;
      }
    }
    // every rank at a barrier: all pass it
    int at_bar = 0, at_end = 0;
    for (int r = 0; r < P; ++r) {
      const std::vector<SimItem>& q = w->comms[r]->queue;
      if (pos[r] == q.size())
        ++at_end;
      else if (q[pos[r]].kind == SimItem::BARRIER)
        ++at_bar;
    }
    if (at_end == P) break;
    if (at_bar == P) {
      for (int r = 0; r < P; ++r) ++pos[r];
      continue;
    }
    if (!progress) {
      set_error("moe_sim_world_run: the ranks' programs do not match (%d of %d ranks wait at a "
                "barrier, %d have finished, the rest wait on a send/recv)", at_bar, P, at_end);
      return fail(MOE_ERR_INVALID_ARG);
    }
  }
  for (moe_comm* c : w->comms) c->queue.clear();
  return MOE_OK;
}

moe_status_t moe_sim_world_destroy(moe_sim_world_t* w) {
  if (!w) return MOE_OK;
  cudaDeviceSynchronize();
  for (moe_sim_world::Slot& s : w->slots)
    for (int q = 0; q < w->P; ++q)
      if (s.peer.p[q]) cudaFree(s.peer.p[q]);
  for (moe_comm* c : w->comms) delete c;
  delete w;
  return MOE_OK;
}

}  // extern "C"
