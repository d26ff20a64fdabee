"""The AllToAll schedules libmoe_b200 executes (moe_alltoall_plan), checked
without GPUs two ways:

1. an in-process interpreter runs every rank's plan with the executor's
   semantics (per phase: all matched sends/recvs, then local copies and the
   chunk permute) and must reproduce the oracle's flat AllToAll byte for byte
   (R13) for many (P, G);
2. real processes (world_size 2 and 4, gloo backend) execute their own plan
   with torch.distributed point-to-point ops -- the multi-process host logic
   of the N>1 path.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2203_14685_b200 as moe

SEND, RECV, COPY, PERMUTE, TRANSPOSE = 0, 1, 2, 3, 4


def _bufs(send, P, G, c):
    stage = G * P * c
    return {0: send.copy(), 1: np.zeros(P * c, send.dtype), 2: np.zeros(stage, send.dtype),
            3: np.zeros(stage, send.dtype)}


def _permute(src, dst, N, G, c):
    for n in range(G):
        for g in range(N):
            for m in range(G):
                d = (n * N + g) * G + m
                s = (g * G + m) * G + n
                dst[d * c:(d + 1) * c] = src[s * c:(s + 1) * c]


def _transpose(src, dst, X, Y, c):
    """dst chunk [y][x] <- src chunk [x][y] (HIER_2D's local reorders)."""
    for x in range(X):
        for y in range(Y):
            d, s = y * X + x, x * Y + y
            dst[d * c:(d + 1) * c] = src[s * c:(s + 1) * c]


def interpret(P, algo, G, sends, c):
    plans = [moe.alltoall_plan(P, r, algo, G) for r in range(P)]
    bufs = [_bufs(sends[r], P, G, c) for r in range(P)]
    phases = sorted(set(o["phase"] for p in plans for o in p))
    for ph in phases:
        msgs = {}
        for r in range(P):   # sends read buffers as they are at the phase start
            for o in plans[r]:
                if o["phase"] == ph and o["op"] == SEND:
                    a = o["src_off"] * c
                    msgs.setdefault((r, o["peer"]), []).append(
                        bufs[r][o["src_buf"]][a:a + o["chunks"] * c].copy())
        for r in range(P):
            for o in plans[r]:
                if o["phase"] == ph and o["op"] == RECV:
                    data = msgs[(o["peer"], r)].pop(0)
                    assert data.size == o["chunks"] * c
                    a = o["dst_off"] * c
                    bufs[r][o["dst_buf"]][a:a + data.size] = data
        assert all(not v for v in msgs.values()), "unmatched sends"
        for r in range(P):
            for o in plans[r]:
                if o["phase"] != ph:
                    continue
                if o["op"] == COPY:
                    a, b, n = o["src_off"] * c, o["dst_off"] * c, o["chunks"] * c
                    bufs[r][o["dst_buf"]][b:b + n] = bufs[r][o["src_buf"]][a:a + n]
                elif o["op"] == PERMUTE:
                    _permute(bufs[r][o["src_buf"]], bufs[r][o["dst_buf"]], o["peer"], o["chunks"], c)
                elif o["op"] == TRANSPOSE:
                    _transpose(bufs[r][o["src_buf"]], bufs[r][o["dst_buf"]], o["peer"],
                               o["chunks"], c)
    return [bufs[r][1] for r in range(P)], plans


@pytest.mark.parametrize("P,G", [(1, 1), (2, 1), (2, 2), (4, 2), (4, 4), (6, 3), (8, 4), (8, 2),
                                 (8, 8), (8, 1), (16, 4)])
@pytest.mark.parametrize("algo", ["flat", "hier", "hier2d"])
def test_plan_reproduces_oracle_alltoall(orc, P, G, algo):
    c = 3
    rng = np.random.default_rng(P * 31 + G)
    sends = [rng.integers(0, 255, P * c, dtype=np.uint8) for _ in range(P)]
    got, plans = interpret(P, algo, G, sends, c)
    want = orc.alltoall_flat(sends)
    for a, b in zip(got, want):
        assert a.tobytes() == b.tobytes()
    if algo == "hier" and P > 1:
        N = P // G
        cross = sum(1 for r in range(P) for o in plans[r]
                    if o["op"] == SEND and o["peer"] // G != r // G)
        assert cross == N * (N - 1)
        sizes = set(o["chunks"] for r in range(P) for o in plans[r]
                    if o["op"] == SEND and o["peer"] // G != r // G)
        assert sizes <= {G * G}                   # B*G/N per group pair
    if algo == "hier2d" and P > 1:
        # two-level: inside the group N chunks per peer, across groups one
        # message of G chunks per group pair per local index (B*G/P bytes)
        N = P // G
        for r in range(P):
            for o in plans[r]:
                if o["op"] == SEND:
                    same = o["peer"] // G == r // G
                    assert o["chunks"] == (N if o["phase"] == 1 else G)
                    assert same if o["phase"] == 1 else o["peer"] % G == r % G


# ------------------------------------------------------------ real processes (gloo)
def _worker(rank, world, algo, G, port, c, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1000 + rank)
    send = rng.integers(0, 255, world * c, dtype=np.uint8)
    bufs = {k: torch.from_numpy(v) for k, v in _bufs(send, world, G, c).items()}
    plan = moe.alltoall_plan(world, rank, algo, G)
    for ph in sorted(set(o["phase"] for o in plan)):
        reqs, self_msgs = [], []
        for o in plan:   # gloo has no self send/recv (NCCL does): match those locally
            if o["phase"] == ph and o["op"] == SEND and o["peer"] == rank:
                a = o["src_off"] * c
                self_msgs.append(bufs[o["src_buf"]][a:a + o["chunks"] * c].clone())
        for o in plan:
            if o["phase"] != ph:
                continue
            if o["op"] == SEND and o["peer"] != rank:
                a = o["src_off"] * c
                reqs.append(dist.isend(bufs[o["src_buf"]][a:a + o["chunks"] * c].clone(), o["peer"]))
            elif o["op"] == RECV and o["peer"] == rank:
                a = o["dst_off"] * c
                t = self_msgs.pop(0)
                bufs[o["dst_buf"]][a:a + t.numel()] = t
            elif o["op"] == RECV:
                a = o["dst_off"] * c
                t = torch.empty(o["chunks"] * c, dtype=torch.uint8)
                reqs.append((dist.irecv(t, o["peer"]), o["dst_buf"], a, t))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                bufs[r[1]][r[2]:r[2] + r[3].numel()] = r[3]
            else:
                r.wait()
        for o in plan:
            if o["phase"] != ph:
                continue
            if o["op"] == COPY:
                a, b, n = o["src_off"] * c, o["dst_off"] * c, o["chunks"] * c
                bufs[o["dst_buf"]][b:b + n] = bufs[o["src_buf"]][a:a + n].clone()
            elif o["op"] == PERMUTE:
                dst = bufs[o["dst_buf"]].numpy()
                _permute(bufs[o["src_buf"]].numpy().copy(), dst, o["peer"], o["chunks"], c)
            elif o["op"] == TRANSPOSE:
                dst = bufs[o["dst_buf"]].numpy()
                _transpose(bufs[o["src_buf"]].numpy().copy(), dst, o["peer"], o["chunks"], c)
    q.put((rank, send.tobytes(), bufs[1].numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,algo,G", [(2, "flat", 1), (2, "hier", 1), (2, "hier", 2),
                                          (4, "flat", 1), (4, "hier", 2),
                                          (8, "hier", 4),    # the paper's 4+4 split on 8 ranks
                                          (4, "hier2d", 2), (8, "hier2d", 4)])
def test_plan_executes_over_gloo(orc, world, algo, G):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world * 10 + G + {"flat": 0, "hier": 5, "hier2d": 7}[algo]
    procs = [ctx.Process(target=_worker, args=(r, world, algo, G, port, 4, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (s, v)) for r, s, v in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sends = [np.frombuffer(res[r][0], np.uint8) for r in range(world)]
    want = orc.alltoall_flat(sends)
    for r in range(world):
        assert res[r][1] == want[r].tobytes()
