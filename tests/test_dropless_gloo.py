"""Host logic of the NCCL dropless exchange (NEXT-4) at world_size 2 and 4
over gloo on CPU: every rank builds its routing and packed rows with the
oracle, exchanges the per-expert count table, plans moe_alltoallv with
paper_2203_14685_b200.alltoallv_plan, moves the rows with gloo's all_to_all,
and must receive exactly what orc_alltoallv delivers (bit-exact)."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synthgen

S, D, E, K = 300, 4, 8, 2


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import oracle
    import paper_2203_14685_b200 as moe
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lg = synthgen.logits(70 + rank, S, E, K, skew=1.0 + rank)
    x = synthgen.tokens(80 + rank, S, D, "f32")
    r = oracle.gate(lg, E=E, k=K, cap=S * K)                     # dropless
    off = oracle.expert_offsets(r)
    packed = oracle.layout_packed(x, r, off)
    El = E // world
    cnt = torch.from_numpy(np.diff(off).astype(np.int32))       # [P][El] table
    rc = torch.empty_like(cnt)
    dist.all_to_all_single(rc, cnt)                              # the count exchange
    send_rows, recv_rows, recv_off = moe.alltoallv_plan(off, rc.tolist(), world)
    recv = torch.empty((sum(recv_rows), D), dtype=torch.float32)
    dist.all_to_all_single(recv, torch.from_numpy(packed), recv_rows, send_rows)
    q.put((rank, lg, x, recv.numpy().copy(), recv_off))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_dropless_exchange_plan_over_gloo(orc, world):
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, 29800 + world, qu)) for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    for _ in range(world):
        v = qu.get(timeout=120)
        out[v[0]] = v[1:]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    El = E // world
    ros = [orc.gate(out[r][0], E=E, k=K, cap=S * K) for r in range(world)]
    offs = [orc.expert_offsets(ro) for ro in ros]
    packs = [orc.layout_packed(out[r][1], ros[r], offs[r]) for r in range(world)]
    counts = np.array([[offs[q][(r + 1) * El] - offs[q][r * El] for r in range(world)]
                       for q in range(world)])
    want = orc.alltoallv(packs, counts)
    for r in range(world):
        assert out[r][2].tobytes() == want[r].tobytes()
        table = [offs[q][r * El + le + 1] - offs[q][r * El + le] for q in range(world)
                 for le in range(El)]
        assert out[r][3] == np.concatenate([[0], np.cumsum(table)]).tolist()


def test_alltoallv_plan_rejects_bad_shapes():
    import paper_2203_14685_b200 as moe
    with pytest.raises(ValueError):
        moe.alltoallv_plan([0, 1, 2], [1, 1, 1], 2)       # E = 2, 3 counts
    with pytest.raises(moe.MoeError) as ei:
        moe.alltoallv_plan([0, 1, 2, 3], [1, 1, 1], 2)    # E = 3 not divisible by 2
    assert ei.value.status == 1                           # MOE_ERR_INVALID_ARG, from the C plan
    with pytest.raises(moe.MoeError):
        moe.alltoallv_plan([0, 2, 1, 3, 4], [1, 1, 1, 1], 2)   # offsets must not decrease
