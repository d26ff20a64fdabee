"""Multi-GPU parity at BASELINE.json's full per-rank sizes, in the launch
configuration bench.py times (RoutePipeline, expert stand-in on): C3 (Switch,
S=32768, d=2048, E=64) and C4a/C4b (k-top-1 / hash, S=65536, d=1024, E=32).

Every rank regenerates all ranks' seeded inputs (synthgen) and runs the
oracle's P-rank simulation of Algorithm 1 itself, then checks its own
outputs: routing and the post-expert receive buffer bit-exact, y within the
north_star tolerance.  Needs >= world GPUs (gpurun --gpus N)."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synthgen

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _rank_main(rank, world, name, algo, port, q):
    import torch.distributed as dist
    import oracle
    import paper_2203_14685_b200 as moe
    from gpu_util import as_f64, combine_bound, dev, host
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synthgen.WORKLOADS[name]
        comm = moe.Comm.from_process_group()
        cap = moe.capacity(w.S, w.E, w.k, w.C)
        inputs = [synthgen.workload_inputs(w, r) for r in range(world)]
        lg, ids, table, x = inputs[rank]
        pipe = moe.RoutePipeline(w.S, w.d, w.E, w.k, cap, torch.bfloat16, w.kind, comm=comm,
                                 algo=algo)
        y = pipe.step(None if lg is None else dev(lg), dev(x), None if ids is None else dev(ids),
                      None if table is None else dev(table), expert=True)
        torch.cuda.synchronize()
        routings, disp, recvs, ys = oracle.route_multi(
            [i[3] for i in inputs], None if w.kind == "hash" else [i[0] for i in inputs],
            E=w.E, k=w.k, cap=cap, kind=w.kind,
            token_ids_list=None if w.kind != "hash" else [i[1] for i in inputs], table=table)
        ro = routings[rank]
        msgs = []
        if not (host(pipe.routing.expert_idx) == ro.expert_idx).all():
            msgs.append("expert_idx")
        if not (host(pipe.routing.slot_idx) == ro.slot_idx).all():
            msgs.append("slot_idx")
        if not (host(pipe.routing.load) == ro.load).all():
            msgs.append("load")
        El = w.E // world
        scaled = oracle.expert_scale(recvs[rank].reshape(world, El, cap, w.d), rank * El)
        if host(pipe.recv).tobytes() != scaled.tobytes():
            msgs.append("recv (post-expert) not bit-exact")
        back = oracle.alltoall_flat([oracle.expert_scale(recvs[p].reshape(world, El, cap, w.d),
                                                         p * El).reshape(w.E, cap, w.d)
                                     for p in range(world)])[rank]
        bound = combine_bound(as_f64(back), ro)
        err = np.abs(as_f64(host(y)) - as_f64(ys[rank]))
        bad = int((err > 1e-2 * bound + 1e-30).sum())
        if bad:
            msgs.append("y: %d elements out of tolerance" % bad)
        q.put((rank, msgs))
        dist.barrier()
        del pipe
        comm.destroy()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, ["exception: %r" % e]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name,algo", [(2, "C3", "p2p"), (2, "C3", "flat"),
                                             (4, "C3", "p2p"), (4, "C4a", "p2p"),
                                             (4, "C4b", "flat")])
def test_fullsize_multi_gpu(world, name, algo):
    if torch.cuda.device_count() < world:
        pytest.skip("needs %d GPUs" % world)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + world * 10 + hash((name, algo)) % 7
    ps = [ctx.Process(target=_rank_main, args=(r, world, name, algo, port, q))
          for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=900) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
    for r in range(world):
        assert res[r] == [], "rank %d: %s" % (r, res[r])
