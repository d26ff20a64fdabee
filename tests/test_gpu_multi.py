"""Multi-GPU parity (needs >= 2 GPUs: run under `gpurun --gpus N`): one
process per GPU, the library-owned NCCL communicator bootstrapped over gloo,
flat and hierarchical AllToAll.  Checked against the oracle's P-rank
simulation of Algorithm 1: recv buffers and routing bit-exact, y within
tolerance, hierarchical byte-identical to flat (R13)."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synthgen

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

S, D, E, K = 1536, 256, 16, 2


def _rank_main(rank, world, algo, G, port, q):
    import torch.distributed as dist
    import paper_2203_14685_b200 as moe
    from gpu_util import dev, host
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = moe.Comm.from_process_group()
    K = int(os.environ.get("MOE_TEST_K", "2"))
    lg = synthgen.logits(synthgen.seed_for(9, rank, 1), S, E, K, skew=0.5)
    dts = os.environ.get("MOE_TEST_DTYPE", "bf16")
    x = synthgen.tokens(synthgen.seed_for(9, rank, 2), S, D, dts)
    cap = moe.capacity(S, E, K, 1.0)
    pipe = moe.RoutePipeline(S, D, E, K, cap, torch.bfloat16 if dts == "bf16" else torch.float32,
                             comm=comm, algo=algo, group_size=G,
                             identity_alias=os.environ.get("MOE_TEST_ALIAS") == "1")
    pipe.step(dev(lg), dev(x), expert=False)     # identity expert: recv = dispatched rows
    torch.cuda.synchronize()
    recv = host(pipe.recv).copy()
    y_id = host(pipe.y).copy()
    y = host(pipe.step(dev(lg), dev(x), expert=True))
    torch.cuda.synchronize()
    y = y.copy()
    # more steps on the same inputs: the double-buffered one-sided path reuses
    # each receive buffer with no entry barrier after combines with no exit
    # barrier; eager steps and graph replays alternate buffers (the results
    # must not change: compared byte for byte with the first two steps)
    lg_d, x_d = dev(lg), dev(x)
    again = []
    for expert in (False, True, False):
        again.append(host(pipe.step(lg_d, x_d, expert=expert)).copy())
    g = pipe.capture(lg_d, x_d)
    for _ in range(3):
        pipe.y.fill_(0)
        g.replay()
        torch.cuda.synchronize()
        again.append(host(pipe.y).copy())
    del g   # a graph holding NCCL work must go before the communicator
    torch.cuda.synchronize()
    ok = [a.tobytes() == (y if i == 1 else y_id).tobytes() for i, a in enumerate(again)]
    q.put((rank, lg, x, recv, y_id, y, host(pipe.routing.slot_idx), ok))
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


def _run(world, algo, G, port):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank_main, args=(r, world, algo, G, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    for _ in range(world):
        r = q.get(timeout=300)
        out[r[0]] = r[1:]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world,algo,G,env", [(2, "flat", 1, None), (2, "hier", 2, None),
                                              (2, "p2p", 1, None), (2, "p2p", 1, "local_pad"),
                                              (2, "p2p", 1, "f32"), (2, "p2p", 1, "rev"),
                                              (2, "p2p", 1, "nodedupe"),
                                              (2, "p2p", 1, "f32_alias"), (2, "p2p", 1, "alias"),
                                              (4, "p2p", 1, "f32"), (2, "p2p", 1, "k4"),
                                              (2, "p2p", 1, "k4_f32"), (2, "p2p", 1, "k4_alias"),
                                              (4, "flat", 1, None), (4, "hier", 2, None),
                                              (4, "hier", 4, None), (4, "p2p", 1, None),
                                              (4, "p2p", 1, "alias"),
                                              (4, "p2p", 1, "local_pad"),
                                              (2, "p2p", 1, "no_precombine")])
def test_multi_gpu_route(orc, world, algo, G, env, monkeypatch):
    if torch.cuda.device_count() < world:
        pytest.skip("needs %d GPUs" % world)
    if env == "local_pad":   # the owners zero their own padding rows (inherited by the ranks)
        monkeypatch.setenv("MOE_P2P_LOCAL_PAD", "1")
    if env == "no_precombine":  # the combine reads both rows of a token's pair
        monkeypatch.setenv("MOE_P2P_PRECOMBINE", "0")
    if env == "nodedupe":    # every row sent, even when a token's two experts share an owner
        monkeypatch.setenv("MOE_P2P_DEDUPE", "0")
    if env == "rev":         # peer combine walking the tokens last to first
        monkeypatch.setenv("MOE_REVERSE_BACKWARDS", "1")
        monkeypatch.setenv("MOE_REVERSE_Y_EF", "1")
    if env in ("alias", "f32_alias", "k4_alias"):   # identity step: RECV_UNMODIFIED combine
        monkeypatch.setenv("MOE_TEST_ALIAS", "1")
    K = 2
    if env in ("k4", "k4_f32", "k4_alias"):  # k = 4: the generic peer combine
        K = 4
        monkeypatch.setenv("MOE_TEST_K", "4")
    f32 = env in ("f32", "f32_alias", "k4_f32")
    if f32:                  # fp32 rows through the one-sided path
        monkeypatch.setenv("MOE_TEST_DTYPE", "f32")
    out = _run(world, algo, G, 29600 + world * 10 + G + {"flat": 0, "hier": 3, "p2p": 6}[algo] +
               {None: 0, "local_pad": 1, "f32": 2, "rev": 3, "nodedupe": 5, "f32_alias": 7,
                "alias": 8, "k4": 9, "k4_f32": 10, "k4_alias": 11, "no_precombine": 12}[env] +
               (40 if env and world == 4 else 0))
    lgs = [out[r][0] for r in range(world)]
    xs = [out[r][1] for r in range(world)]
    cap = orc.capacity(S, E, K, 1.0)
    routings, disp, recvs, ys = orc.route_multi(xs, lgs, E=E, k=K, cap=cap)
    _, _, _, ys_id = orc.route_multi(xs, lgs, E=E, k=K, cap=cap, scale=False)
    for r in range(world):
        _, _, recv, y_id, y, slots, again_ok = out[r]
        assert all(again_ok), "rank %d: repeated steps / graph replays differ: %s" % (r, again_ok)
        assert (slots == routings[r].slot_idx).all()
        assert recv.tobytes() == recvs[r].tobytes()          # AllToAll bit-exact
        # identity expert, k=2 RENORM: y == combine of the original rows
        from gpu_util import as_f64, assert_y_close, combine_bound
        assert_y_close(y_id, ys_id[r], combine_bound(as_f64(disp[r]), routings[r]), not f32)
        back = orc.alltoall_flat([orc.expert_scale(recvs[q].reshape(world, E // world, cap, D),
                                                   q * (E // world)).reshape(E, cap, D)
                                  for q in range(world)])[r]
        assert_y_close(y, ys[r], combine_bound(as_f64(back), routings[r]), not f32)


def _bwd_rank_main(rank, world, port, q):
    """Backward over NVLink: combine_backward_p2p + dispatch_backward_p2p."""
    import torch.distributed as dist
    import paper_2203_14685_b200 as moe
    from gpu_util import dev, host
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = moe.Comm.from_process_group()
    lg = synthgen.logits(synthgen.seed_for(9, rank, 5), S, E, K, skew=0.5)
    cap = moe.capacity(S, E, K, 0.8)
    r = moe.Gate(S, E, K, cap)(dev(lg))
    eo = synthgen.tokens(synthgen.seed_for(9, rank, 6), E * cap, D, "bf16").reshape(E, cap, D)
    dr = synthgen.tokens(synthgen.seed_for(9, rank, 7), E * cap, D, "bf16").reshape(E, cap, D)
    dy = synthgen.tokens(synthgen.seed_for(9, rank, 8), S, D, "bf16")
    expert_out = comm.symm_empty((E, cap, D), torch.bfloat16)
    d_expert_out = comm.symm_empty((E, cap, D), torch.bfloat16)
    d_recv = comm.symm_empty((E, cap, D), torch.bfloat16)
    expert_out.copy_(dev(eo))
    d_recv.copy_(dev(dr))
    d_expert_out.fill_(7.0)  # every row must be overwritten (admitted or padding)
    torch.cuda.synchronize()
    _, dw = comm.combine_backward_p2p(dev(dy), expert_out, r, d_expert_out)
    dx = comm.dispatch_backward_p2p(d_recv, r)
    torch.cuda.synchronize()
    deo_pull = host(d_expert_out).copy()
    # the push form: the same d_expert_out bytes and d_weight (same lane order)
    wtab = comm.symm_empty((E * cap,), torch.float32)
    dwtab = comm.symm_empty((E * cap,), torch.float32)
    d_expert_out.fill_(5.0)
    _, dw2 = comm.combine_backward_push_p2p(dev(dy), expert_out, r, d_expert_out, wtab, dwtab)
    torch.cuda.synchronize()
    assert host(d_expert_out).tobytes() == deo_pull.tobytes(), "push d_expert_out"
    assert host(dw2).tobytes() == host(dw).tobytes(), "push d_weight"
    q.put((rank, lg, eo, dr, dy, deo_pull, host(dw).copy(), host(dx).copy()))
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,env", [(2, None), (2, "local_pad"), (4, None)])
def test_multi_gpu_backward_p2p(orc, world, env, monkeypatch):
    if torch.cuda.device_count() < world:
        pytest.skip("needs %d GPUs" % world)
    if env == "local_pad":   # owners zero their own padding rows of the dy scatter
        monkeypatch.setenv("MOE_P2P_LOCAL_PAD", "1")
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = 29700 + world + (10 if env else 0)
    ps = [ctx.Process(target=_bwd_rank_main, args=(r, world, port, qu)) for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    for _ in range(world):
        v = qu.get(timeout=300)
        out[v[0]] = v[1:]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    from gpu_util import as_f64, assert_y_close, combine_bound
    cap = orc.capacity(S, E, K, 0.8)
    ros = [orc.gate(out[r][0], E=E, k=K, cap=cap) for r in range(world)]
    backs = orc.alltoall_flat([out[q][1] for q in range(world)])      # rows each rank combines
    d_backs, dws = [], []
    for r in range(world):
        db, dw = orc.reverse_layout_bwd(out[r][3], backs[r], ros[r])
        d_backs.append(db)
        dws.append(dw)
    d_eo = orc.alltoall_flat(d_backs)                                   # lands at the owners
    d_disp = orc.alltoall_flat([out[q][2] for q in range(world)])
    for r in range(world):
        assert out[r][4].tobytes() == d_eo[r].tobytes()
        dwb = np.abs(out[r][5].astype(np.float64) - dws[r].astype(np.float64))
        rows = as_f64(backs[r])
        bound = np.zeros_like(dwb)
        for j in range(K):
            ok = ros[r].slot_idx[:, j] >= 0
            bound[ok, j] = np.abs(as_f64(out[r][3])[ok] *
                                  rows[ros[r].expert_idx[ok, j], ros[r].slot_idx[ok, j]]).sum(1)
        assert (dwb <= (D / 32 + 6) * 2.0 ** -24 * bound + 1e-30).all()
        dx_o = orc.layout_bwd(d_disp[r], ros[r])
        unit = type(ros[r])(**{**ros[r].__dict__,
                               "weight": (ros[r].slot_idx >= 0).astype(np.float32)})
        assert_y_close(out[r][6], dx_o, combine_bound(as_f64(d_disp[r]), unit), True, "dx")


def _packed_rank_main(rank, world, port, q):
    """Dropless exchange: device-side (NVLink) and NCCL alltoallv."""
    import torch.distributed as dist
    import paper_2203_14685_b200 as moe
    from gpu_util import dev, host
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = moe.Comm.from_process_group()
    lg = synthgen.logits(synthgen.seed_for(9, rank, 11), S, E, K, skew=1.0 + rank)
    x = synthgen.tokens(synthgen.seed_for(9, rank, 12), S, D, "bf16")
    r = moe.Gate(S, E, K, S * K)(dev(lg), slot_src=False)            # dropless
    off = moe.expert_offsets(r)
    rows = world * S * K
    counts = comm.symm_empty((E,), torch.int32)
    recv = comm.symm_empty((rows, D), torch.bfloat16)
    eo = comm.symm_empty((rows, D), torch.bfloat16)
    pb, roff = comm.dispatch_packed_p2p(dev(x), r, off, counts, recv)
    torch.cuda.synchronize()
    R_in = int(host(roff)[-1])
    recv_h = host(recv)[:R_in].copy()
    # expert stand-in: an independent synthetic output per received row
    out_h = synthgen.tokens(synthgen.seed_for(9, rank, 13), R_in, D, "bf16")
    eo[:R_in].copy_(dev(out_h))
    torch.cuda.synchronize()
    y = host(comm.combine_packed_p2p(eo, r, off, pb)).copy()
    # NCCL path: count table exchange, host counts, alltoallv of the packed rows
    El = E // world
    off_h = host(off)
    send_cnt = np.diff(off_h).astype(np.int32)                     # [E] = [world][El]
    cnt_recv = torch.empty((E,), dtype=torch.int32, device="cuda")
    comm.alltoall(dev(send_cnt), cnt_recv)
    rc = host(cnt_recv).reshape(world, El).sum(1)
    sc = send_cnt.reshape(world, El).sum(1)
    packed = moe.layout_packed(dev(x), r, off)
    recv2 = torch.empty((int(rc.sum()), D), dtype=torch.bfloat16, device="cuda")
    comm.alltoallv(packed, sc, recv2, rc)
    torch.cuda.synchronize()
    # the adjoints of the dropless exchange (NEXT-1 x NEXT-4)
    dy = synthgen.tokens(synthgen.seed_for(9, rank, 14), S, D, "bf16")
    d_eo = comm.symm_empty((rows, D), torch.bfloat16)
    _, dw = comm.combine_packed_backward_p2p(dev(dy), eo, r, off, pb, d_eo)
    dr_h = synthgen.tokens(synthgen.seed_for(9, rank, 15), R_in, D, "bf16")
    d_recv = comm.symm_empty((rows, D), torch.bfloat16)
    d_recv[:R_in].copy_(dev(dr_h))
    torch.cuda.synchronize()
    dx = comm.dispatch_packed_backward_p2p(d_recv, r, off, pb)
    torch.cuda.synchronize()
    bwd = (dy, host(d_eo)[:R_in].copy(), host(dw).copy(), dr_h, host(dx).copy())
    q.put((rank, lg, x, host(roff).copy(), recv_h, out_h, y, host(recv2).copy(), bwd))
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_dropless(orc, world):
    if torch.cuda.device_count() < world:
        pytest.skip("needs %d GPUs" % world)
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = 29750 + world
    ps = [ctx.Process(target=_packed_rank_main, args=(r, world, port, qu)) for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    for _ in range(world):
        v = qu.get(timeout=300)
        out[v[0]] = v[1:]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    from gpu_util import as_f64, assert_y_close
    El = E // world
    ros = [orc.gate(out[r][0], E=E, k=K, cap=S * K) for r in range(world)]
    offs = [orc.expert_offsets(ro) for ro in ros]
    packs = [orc.layout_packed(out[r][1], ros[r], offs[r]) for r in range(world)]
    counts = np.array([[offs[q][(r + 1) * El] - offs[q][r * El] for r in range(world)]
                       for q in range(world)])
    recvs = orc.alltoallv(packs, counts)
    outs = [out[r][4] for r in range(world)]
    backs = orc.alltoallv(outs, counts.T)
    for r in range(world):
        roff, recv_h, _, y, recv2 = out[r][2], out[r][3], out[r][4], out[r][5], out[r][6]
        table = np.array([[offs[q][r * El + le + 1] - offs[q][r * El + le] for le in range(El)]
                          for q in range(world)]).reshape(-1)
        assert roff.tolist() == np.concatenate([[0], np.cumsum(table)]).tolist()
        assert recv_h.tobytes() == recvs[r].tobytes()         # device-side exchange
        assert recv2.tobytes() == recvs[r].tobytes()          # NCCL alltoallv
        y_o = orc.reverse_layout_packed(backs[r], ros[r], offs[r])
        b64 = as_f64(backs[r])
        bound = np.zeros((S, D))
        for j in range(K):
            ok = ros[r].slot_idx[:, j] >= 0
            rows = offs[r][ros[r].expert_idx[ok, j]] + ros[r].slot_idx[ok, j]
            bound[ok] += np.abs(ros[r].weight[ok, j].astype(np.float64)[:, None] * b64[rows])
        assert_y_close(y, y_o, bound, True, "y")
    # adjoints: the token owner's packed d_back rows (padded oracle adjoint
    # minus padding) travel to the owners like the forward rows
    d_backs, dws = [], []
    for r in range(world):
        dy = out[r][7][0]
        ro, off = ros[r], offs[r]
        cap = S * K
        back_pad = np.zeros((E, cap, D), np.uint16)
        for e in range(E):
            back_pad[e, :off[e + 1] - off[e]] = backs[r][off[e]:off[e + 1]]
        db, dw = orc.reverse_layout_bwd(dy, back_pad, ro)
        d_backs.append(np.concatenate([db[e, :off[e + 1] - off[e]] for e in range(E)]))
        dws.append(dw)
    d_eo_want = orc.alltoallv(d_backs, counts)
    d_disp = orc.alltoallv([out[q][7][3] for q in range(world)], counts.T)
    for r in range(world):
        _, d_eo, dw, _, dx = out[r][7]
        assert d_eo.tobytes() == d_eo_want[r].tobytes()
        err = np.abs(dw.astype(np.float64) - dws[r].astype(np.float64))
        b64 = as_f64(backs[r])
        dy64 = as_f64(out[r][7][0])
        bound = np.zeros_like(err)
        for j in range(K):
            ok = ros[r].slot_idx[:, j] >= 0
            rows_ = offs[r][ros[r].expert_idx[ok, j]] + ros[r].slot_idx[ok, j]
            bound[ok, j] = np.abs(dy64[ok] * b64[rows_]).sum(1)
        assert (err <= (D / 32 + 6) * 2.0 ** -24 * bound + 1e-30).all()
        g_pad = np.zeros((E, S * K, D), np.uint16)
        off = offs[r]
        for e in range(E):
            g_pad[e, :off[e + 1] - off[e]] = d_disp[r][off[e]:off[e + 1]]
        dx_o = orc.layout_bwd(g_pad, ros[r])
        from gpu_util import combine_bound
        unit = type(ros[r])(**{**ros[r].__dict__,
                               "weight": (ros[r].slot_idx >= 0).astype(np.float32)})
        assert_y_close(dx, dx_o, combine_bound(as_f64(g_pad), unit), True, "dx")


def _timeout_rank_main(rank, world, port, q):
    """Rank 0 enters a device barrier that rank 1 never enters."""
    import torch.distributed as dist
    import paper_2203_14685_b200 as moe
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    moe.set_tuning(barrier_timeout_ms=200)
    comm = moe.Comm.from_process_group()
    comm.check()
    status = 0
    if rank == 0:
        comm.barrier()
        try:
            comm.check()
        except moe.MoeError as e:
            status = e.status
    q.put((rank, status))
    dist.barrier()            # rank 1 waits here (host side) until rank 0 has its answer
    comm.abort()
    dist.destroy_process_group()


def test_multi_gpu_barrier_timeout():
    """SURVEY §5 failure detection: a rank that never arrives makes the
    peer's bounded device barrier give up; moe_comm_check reports
    MOE_ERR_TIMEOUT; moe_comm_abort releases the communicator."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    ps = [ctx.Process(target=_timeout_rank_main, args=(r, 2, 29790, qu)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(qu.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got[0] == 7 and got[1] == 0     # MOE_ERR_TIMEOUT on the waiting rank only
