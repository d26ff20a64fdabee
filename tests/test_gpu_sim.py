"""The multi-GPU path on ONE GPU: P simulated ranks (moe.SimWorld; include/
moe.h "simulated ranks") run the library's real exchange kernels -- the
one-sided NVLink dispatch/combine with its dedupe, alias and local-padding
forms, the dropless device-side exchange, the backward adjoints, and the NCCL
schedules (flat, the paper's leader scheme, the two-level form) -- phase by
phase, barriers as step boundaries.  Every receive buffer must equal the
oracle's P-rank simulation of Algorithm 1 steps 3 and 5 (PAPER.md:53-54,
62-63) byte for byte; y within the north_star tolerance.

No `multigpu` marker: these run on a single-GPU box.  Calls on a simulated
rank are queued until SimWorld.run(): every tensor they use must stay alive
until then."""
import numpy as np
import pytest
import torch

import paper_2203_14685_b200 as moe
import synthgen
from gpu_util import as_f64, assert_routing_equal, assert_y_close, combine_bound, dev, host

pytestmark = pytest.mark.gpu

TORCH_DT = {"bf16": torch.bfloat16, "f32": torch.float32}


class Ranks:
    """Per-rank seeded inputs, gates and routings of one simulated job."""

    def __init__(self, orc, P, S, d, E, k, C=1.0, dtype="bf16", kind="topk", skew=0.5, seed=11):
        self.P, self.S, self.d, self.E, self.k, self.dtype, self.kind = P, S, d, E, k, dtype, kind
        self.cap = orc.capacity(S, E, k, C)
        self.El = E // P
        self.lgs = [synthgen.logits(synthgen.seed_for(seed, r, 1), S, E, k, kind, skew=skew)
                    for r in range(P)]
        self.xs = [synthgen.tokens(synthgen.seed_for(seed, r, 2), S, d, dtype) for r in range(P)]
        self.gates = [moe.Gate(S, E, k, self.cap, kind) for _ in range(P)]
        self.routings = [g(dev(lg)) for g, lg in zip(self.gates, self.lgs)]
        self.x_dev = [dev(x) for x in self.xs]
        torch.cuda.synchronize()
        self.orc_routings = [orc.gate(lg, E=E, k=k, cap=self.cap, kind=kind) for lg in self.lgs]
        for r in range(P):
            assert_routing_equal(self.routings[r], self.orc_routings[r], "rank %d" % r)
        self.disp = [orc.layout(x, ro) for x, ro in zip(self.xs, self.orc_routings)]

    def symm(self, world, shape, dtype=None):
        return [world.comm(r).symm_empty(shape, dtype or TORCH_DT[self.dtype])
                for r in range(self.P)]


def _expert_outputs(orc, R, recvs):
    return [orc.expert_scale(recvs[q].reshape(R.P, R.El, R.cap, R.d), q * R.El)
            .reshape(R.E, R.cap, R.d) for q in range(R.P)]


def _check_y(R, ys, backs):
    for r in range(R.P):
        assert_y_close(host(ys[r]), backs[r][1], combine_bound(as_f64(backs[r][0]),
                                                               R.orc_routings[r]),
                       R.dtype == "bf16", "rank %d" % r)


# ------------------------------------------------------------ one-sided padded path
P2P_CASES = [
    dict(P=2, S=1536, d=256, E=16, k=2),
    dict(P=4, S=1200, d=256, E=16, k=2),
    dict(P=8, S=1000, d=128, E=32, k=2),
    dict(P=8, S=777, d=256, E=64, k=1),                  # Switch, C3-like expert count
    dict(P=4, S=900, d=128, E=16, k=4),                  # k = 4: the generic combine
    dict(P=2, S=1000, d=64, E=8, k=2, dtype="f32"),
    dict(P=4, S=1500, d=128, E=32, k=1, C=1.25, kind="topk"),  # padding-heavy: local padding
    dict(P=4, S=1024, d=128, E=32, k=2, kind="ktop1"),
    dict(P=2, S=999, d=96, E=8, k=2, C=0.6, skew=3.0),   # heavy drops, ragged
]
P2P_MODES = {"default": {}, "nodedupe": {"p2p_dedupe": 0}, "local_pad": {"p2p_local_pad": 1},
             "no_local_pad": {"p2p_local_pad": 0}, "no_precombine": {"p2p_precombine": 0}}


def _route_p2p(orc, R, world, mode, expert):
    """dispatch_p2p on every rank; run; (expert in place); combine; run."""
    recvs = R.symm(world, (R.E, R.cap, R.d))
    ys = [torch.empty((R.S, R.d), dtype=TORCH_DT[R.dtype], device="cuda") for _ in range(R.P)]
    for r in range(R.P):
        world.comm(r).dispatch_p2p(R.x_dev[r], R.routings[r], recvs[r])
    world.run()
    torch.cuda.synchronize()
    got_recv = [host(t).copy() for t in recvs]
    want_recv = orc.alltoall_flat(R.disp)
    for r in range(R.P):
        assert got_recv[r].tobytes() == want_recv[r].tobytes(), "recv of rank %d" % r
    if mode == "expert":                  # s_e in place, a barrier, combine without its own
        for r in range(R.P):
            moe.expert_scale(recvs[r], R.P, R.El, r * R.El, out=recvs[r])
        for r in range(R.P):
            c = world.comm(r)
            c.barrier()
            c.combine_p2p(recvs[r], R.routings[r], ys[r], flags=c.NO_ENTRY_BARRIER)
        outs = _expert_outputs(orc, R, want_recv)
    elif expert:                           # s_e in place, then the default combine
        for r in range(R.P):
            moe.expert_scale(recvs[r], R.P, R.El, r * R.El, out=recvs[r])
        for r in range(R.P):
            world.comm(r).combine_p2p(recvs[r], R.routings[r], ys[r])
        outs = _expert_outputs(orc, R, want_recv)
    else:                                  # identity expert, RECV_UNMODIFIED (alias mode)
        for r in range(R.P):
            c = world.comm(r)
            c.combine_p2p(recvs[r], R.routings[r], ys[r],
                          flags=c.NO_ENTRY_BARRIER | c.RECV_UNMODIFIED)
        outs = want_recv
    world.run()
    torch.cuda.synchronize()
    backs = orc.alltoall_flat(outs)
    _check_y(R, ys, [(backs[r], orc.reverse_layout(backs[r], R.orc_routings[r]))
                     for r in range(R.P)])


@pytest.mark.parametrize("mode", sorted(P2P_MODES))
@pytest.mark.parametrize("c", P2P_CASES, ids=lambda c: "-".join("%s=%s" % kv for kv in c.items()))
def test_sim_dispatch_combine_p2p(orc, c, mode):
    with moe.tuned(**P2P_MODES[mode]), moe.SimWorld(c["P"]) as world:
        R = Ranks(orc, **c)
        _route_p2p(orc, R, world, mode, expert=True)


@pytest.mark.parametrize("c", [c for c in P2P_CASES if c["k"] == 2],
                         ids=lambda c: "-".join("%s=%s" % kv for kv in c.items()))
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_sim_precombine_bit_identical(orc, c, dtype):
    """The owners' pre-combine of token pairs (k = 2, both slots on one
    remote owner, MOE_P2P_PRECOMBINE) gives y byte for byte equal to reading
    both rows (same fp32 FMA order, one rounding), with the s_e expert in
    place between the dispatch and the combine."""
    ys = {}
    for pre in (1, 0):
        with moe.tuned(p2p_precombine=pre), moe.SimWorld(c["P"]) as world:
            R = Ranks(orc, **{**c, "dtype": dtype})
            recvs = R.symm(world, (R.E, R.cap, R.d))
            out = [torch.empty((R.S, R.d), dtype=TORCH_DT[R.dtype], device="cuda")
                   for _ in range(R.P)]
            for r in range(R.P):
                world.comm(r).dispatch_p2p(R.x_dev[r], R.routings[r], recvs[r])
            world.run()
            torch.cuda.synchronize()
            for r in range(R.P):
                moe.expert_scale(recvs[r], R.P, R.El, r * R.El, out=recvs[r])
            for r in range(R.P):
                world.comm(r).combine_p2p(recvs[r], R.routings[r], out[r])
            world.run()
            torch.cuda.synchronize()
            ys[pre] = [host(t).tobytes() for t in out]
    assert ys[1] == ys[0]


@pytest.mark.parametrize("c", P2P_CASES[:4] + P2P_CASES[5:6],
                         ids=lambda c: "-".join("%s=%s" % kv for kv in c.items()))
@pytest.mark.parametrize("seq", ["alias", "expert_barrier_noentry"])
def test_sim_combine_sequences(orc, c, seq):
    """alias: identity expert, combine(NO_ENTRY | RECV_UNMODIFIED) reads a
    row sent once for two slots once.  expert_barrier_noentry: dispatch ->
    in-place expert -> moe_comm_barrier -> combine(NO_ENTRY_BARRIER); the
    combine must read the expert outputs of BOTH slots."""
    with moe.SimWorld(c["P"]) as world:
        R = Ranks(orc, **c)
        _route_p2p(orc, R, world, "expert" if seq != "alias" else "alias", expert=False)


def test_sim_route_pipeline_p2p(orc):
    """RoutePipeline on simulated ranks: its gate and dispatch, then run."""
    P, S, d, E, k = 4, 1024, 128, 16, 2
    with moe.SimWorld(P) as world:
        R = Ranks(orc, P, S, d, E, k)
        pipes = [moe.RoutePipeline(S, d, E, k, R.cap, torch.bfloat16, comm=world.comm(r),
                                   algo="p2p", identity_alias=True) for r in range(P)]
        lg_dev = [dev(lg) for lg in R.lgs]   # alive until run(): the fused gate + dispatch is queued
        ys = [pipes[r].step(lg_dev[r], R.x_dev[r]) for r in range(P)]
        world.run()
        torch.cuda.synchronize()
        want = orc.alltoall_flat(R.disp)
        for r in range(P):
            assert host(pipes[r].recv).tobytes() == want[r].tobytes()
        backs = orc.alltoall_flat(want)
        _check_y(R, ys, [(backs[r], orc.reverse_layout(backs[r], R.orc_routings[r]))
                         for r in range(P)])


@pytest.mark.parametrize("double_buffer", [True, False])
@pytest.mark.parametrize("P,E", [(4, 16), (8, 8), (8, 32)])
def test_sim_route_pipeline_p2p_steps(orc, double_buffer, P, E):
    """Four RoutePipeline steps on simulated ranks over two alternating token
    sets: with double buffering the steps alternate two receive buffers,
    every combine skips its exit barrier and every dispatch after a buffer's
    first skips its entry barrier (include/moe.h MOE_P2P_*); each step's
    receive buffer and y equal the oracle's for that step's tokens.  (Identity
    expert: on a simulated rank only the library's calls are queued, so an
    in-place expert would run before its dispatch; the multi-GPU test covers
    the s_e expert.)"""
    S, d, k = 768, 64, 2
    with moe.SimWorld(P) as world:
        R = Ranks(orc, P, S, d, E, k)
        xs_b = [synthgen.tokens(synthgen.seed_for(29, r, 2), S, d, "bf16") for r in range(P)]
        sets = [(R.x_dev, R.disp),
                ([dev(x) for x in xs_b], [orc.layout(x, ro) for x, ro in zip(xs_b, R.orc_routings)])]
        pipes = [moe.RoutePipeline(S, d, E, k, R.cap, torch.bfloat16, comm=world.comm(r),
                                   algo="p2p", double_buffer=double_buffer) for r in range(P)]
        lg_dev = [dev(lg) for lg in R.lgs]
        recv_ptrs = set()
        for i in range(4):
            x_dev, disp = sets[i % 2]
            ys = [pipes[r].step(lg_dev[r], x_dev[r]) for r in range(P)]
            world.run()
            torch.cuda.synchronize()
            recv_ptrs.add(pipes[0].recv.data_ptr())
            want = orc.alltoall_flat(disp)
            for r in range(P):
                assert host(pipes[r].recv).tobytes() == want[r].tobytes(), (i, r)
            backs = orc.alltoall_flat(want)
            _check_y(R, ys, [(backs[r], orc.reverse_layout(backs[r], R.orc_routings[r]))
                             for r in range(P)])
        assert len(recv_ptrs) == (2 if double_buffer else 1)


# ------------------------------------------------------------ AllToAll algorithms
A2A_CASES = [(2, "flat", 1), (4, "flat", 1), (8, "flat", 1), (2, "hier", 2), (4, "hier", 2),
             (4, "hier", 4), (8, "hier", 4), (8, "hier", 2), (8, "hier", 1), (4, "hier2d", 2),
             (8, "hier2d", 4), (8, "hier2d", 2), (8, "hier2d", 8), (8, "hier2d", 1), (2, "p2p", 1),
             (4, "p2p", 1), (8, "p2p", 1)]


@pytest.mark.parametrize("P,algo,G", A2A_CASES)
def test_sim_alltoall(orc, P, algo, G):
    """moe_alltoall byte-identical to the oracle's flat AllToAll for every
    algorithm (R13, R21); the leader scheme also equals the oracle's
    explicit five phases."""
    chunk = 4096 + 16 * P           # bytes per peer, 16-byte multiple
    rng = np.random.default_rng(P * 100 + G)
    sends = [rng.integers(0, 256, P * chunk, dtype=np.uint8) for _ in range(P)]
    want = orc.alltoall_flat(sends)
    if algo == "hier":
        assert [h.tobytes() for h in orc.alltoall_hier(sends, G)[0]] == [w.tobytes() for w in want]
    with moe.SimWorld(P) as world:
        comms = [world.comm(r) for r in range(P)]
        if algo == "p2p":
            recvs = [comms[r].symm_empty((P * chunk,), torch.uint8) for r in range(P)]
        else:
            recvs = [torch.empty(P * chunk, dtype=torch.uint8, device="cuda") for _ in range(P)]
        send_d = [torch.from_numpy(s).cuda() for s in sends]
        wss = [torch.empty(max(1, comms[r].workspace_bytes(algo, G, chunk)), dtype=torch.uint8,
                           device="cuda") for r in range(P)]
        for _ in range(2):           # twice: buffers and barrier epochs reused
            for r in range(P):
                recvs[r].fill_(7)
                comms[r].alltoall(send_d[r], recvs[r], algo, G, wss[r])
            world.run()
            torch.cuda.synchronize()
            for r in range(P):
                assert host(recvs[r]).tobytes() == want[r].tobytes(), "rank %d" % r


def test_sim_alltoallv_nccl(orc):
    """The NCCL dropless exchange: count AllToAll, the C host plan
    (moe_alltoallv_plan), moe_alltoallv -- equal to the oracle's alltoallv of
    the packed layouts."""
    P, S, d, E, k = 4, 800, 64, 16, 2
    with moe.SimWorld(P) as world:
        R = Ranks(orc, P, S, d, E, k, C=8.0, skew=1.5)
        offs = [moe.expert_offsets(R.routings[r]) for r in range(P)]
        packed = [moe.layout_packed(R.x_dev[r], R.routings[r], offs[r]) for r in range(P)]
        cnt = [(o[1:] - o[:-1]).contiguous() for o in offs]
        cnt_recv = [torch.empty_like(c) for c in cnt]
        comms = [world.comm(r) for r in range(P)]
        for r in range(P):
            comms[r].alltoall(cnt[r], cnt_recv[r], "flat")
        world.run()
        torch.cuda.synchronize()
        plans = [moe.alltoallv_plan(host(offs[r]), host(cnt_recv[r]), P) for r in range(P)]
        recvs = [torch.empty((P * S * k, d), dtype=torch.bfloat16, device="cuda") for _ in range(P)]
        for r in range(P):
            comms[r].alltoallv(packed[r], plans[r][0], recvs[r], plans[r][1])
        world.run()
        torch.cuda.synchronize()
        o_offs = [orc.expert_offsets(ro) for ro in R.orc_routings]
        o_packed = [orc.layout_packed(x, ro, o) for x, ro, o in zip(R.xs, R.orc_routings, o_offs)]
        El = E // P
        counts = np.array([[o_offs[q][(r + 1) * El] - o_offs[q][r * El] for r in range(P)]
                           for q in range(P)])
        want = orc.alltoallv([op[:o[-1]] for op, o in zip(o_packed, o_offs)], counts)
        for r in range(P):
            n = want[r].shape[0]
            assert host(recvs[r])[:n].tobytes() == want[r].tobytes(), "rank %d" % r
            assert plans[r][2][-1] == n


# ------------------------------------------------------------ dropless device-side exchange
@pytest.mark.parametrize("P,E,k", [(2, 8, 2), (4, 16, 1), (8, 32, 2)])
def test_sim_dropless_p2p(orc, P, E, k):
    S, d = 700, 128
    with moe.SimWorld(P) as world:
        R = Ranks(orc, P, S, d, E, k, C=float(E), skew=1.0)   # cap >= S*k/E*E: dropless
        comms = [world.comm(r) for r in range(P)]
        rows = P * S * k
        recvs = R.symm(world, (rows, d))
        counts = [comms[r].symm_empty((E,), torch.int32) for r in range(P)]
        offs = [moe.expert_offsets(R.routings[r]) for r in range(P)]
        pb = [None] * P
        for r in range(P):
            pb[r] = comms[r].dispatch_packed_p2p(R.x_dev[r], R.routings[r], offs[r], counts[r],
                                                 recvs[r])
        world.run()
        torch.cuda.synchronize()
        o_offs = [orc.expert_offsets(ro) for ro in R.orc_routings]
        o_packed = [orc.layout_packed(x, ro, o) for x, ro, o in zip(R.xs, R.orc_routings, o_offs)]
        El = E // P
        cnts = np.array([[o_offs[q][(r + 1) * El] - o_offs[q][r * El] for r in range(P)]
                         for q in range(P)])
        want = orc.alltoallv([op[:o[-1]] for op, o in zip(o_packed, o_offs)], cnts)
        for r in range(P):
            n = want[r].shape[0]
            assert host(recvs[r])[:n].tobytes() == want[r].tobytes(), "rank %d" % r
            assert host(pb[r][1])[-1] == n
        ys = [torch.empty((S, d), dtype=torch.bfloat16, device="cuda") for _ in range(P)]
        for r in range(P):
            comms[r].combine_packed_p2p(recvs[r], R.routings[r], offs[r], pb[r][0], ys[r])
        world.run()
        torch.cuda.synchronize()
        for r in range(P):   # identity expert: y = sum_j w_j x_t (weights of one token)
            bound = combine_bound(as_f64(R.disp[r]), R.orc_routings[r])
            y_o = orc.reverse_layout(R.disp[r], R.orc_routings[r])
            assert_y_close(host(ys[r]), y_o, bound, True, "rank %d" % r)


# ------------------------------------------------------------ backward over the exchange
@pytest.mark.parametrize("form", ["pull", "push"])
@pytest.mark.parametrize("P,E,k,C,local_pad", [(2, 16, 2, 0.8, -1), (4, 16, 2, 1.0, -1),
                                               (8, 32, 1, 1.25, -1), (4, 32, 1, 1.25, 0),
                                               (2, 8, 2, 1.25, 1),
                                               (8, 8, 2, 1.0, -1)])   # C2 at N=8: 1 expert per rank
def test_sim_backward_p2p(orc, form, P, E, k, C, local_pad):
    """combine_backward (pull: reads expert rows and stores w*dy at the owner;
    push: dy rows + weights to the owners, dots there) and the dispatch
    adjoint, against the oracle's per-rank adjoints around its AllToAlls."""
    S, d = 900, 128
    with moe.tuned(p2p_local_pad=local_pad), moe.SimWorld(P) as world:
        R = Ranks(orc, P, S, d, E, k, C=C, skew=0.5)
        comms = [world.comm(r) for r in range(P)]
        eo = [synthgen.tokens(synthgen.seed_for(31, r, 6), E * R.cap, d, "bf16")
              .reshape(E, R.cap, d) for r in range(P)]
        dr = [synthgen.tokens(synthgen.seed_for(31, r, 7), E * R.cap, d, "bf16")
              .reshape(E, R.cap, d) for r in range(P)]
        dy = [synthgen.tokens(synthgen.seed_for(31, r, 8), S, d, "bf16") for r in range(P)]
        expert_out = R.symm(world, (E, R.cap, d))
        d_eo = R.symm(world, (E, R.cap, d))
        d_recv = R.symm(world, (E, R.cap, d))
        wt = R.symm(world, (E * R.cap,), torch.float32)
        dwt = R.symm(world, (E * R.cap,), torch.float32)
        for r in range(P):
            expert_out[r].copy_(dev(eo[r]))
            d_recv[r].copy_(dev(dr[r]))
            d_eo[r].fill_(3.0)
        dws = [torch.empty((S, k), dtype=torch.float32, device="cuda") for _ in range(P)]
        dxs = [torch.empty((S, d), dtype=torch.bfloat16, device="cuda") for _ in range(P)]
        dy_dev = [dev(v) for v in dy]   # alive until run(): the queued kernels read them
        for r in range(P):
            if form == "pull":
                comms[r].combine_backward_p2p(dy_dev[r], expert_out[r], R.routings[r], d_eo[r],
                                              dws[r])
            else:
                comms[r].combine_backward_push_p2p(dy_dev[r], expert_out[r], R.routings[r],
                                                   d_eo[r], wt[r], dwt[r], dws[r])
            comms[r].dispatch_backward_p2p(d_recv[r], R.routings[r], dxs[r])
        world.run()
        torch.cuda.synchronize()
        backs = orc.alltoall_flat(eo)            # the rows each rank's tokens combined
        d_backs, dw_o = [], []
        for r in range(P):
            db, dw = orc.reverse_layout_bwd(dy[r], backs[r], R.orc_routings[r])
            d_backs.append(db)
            dw_o.append(dw)
        want_deo = orc.alltoall_flat(d_backs)    # lands at the experts' owners
        d_disp = orc.alltoall_flat(dr)
        for r in range(P):
            assert host(d_eo[r]).tobytes() == want_deo[r].tobytes(), "d_expert_out rank %d" % r
            err = np.abs(host(dws[r]).astype(np.float64) - dw_o[r].astype(np.float64))
            bound = np.zeros_like(err)
            rows = as_f64(backs[r])
            ro = R.orc_routings[r]
            for j in range(k):
                ok = ro.slot_idx[:, j] >= 0
                bound[ok, j] = np.abs(as_f64(dy[r])[ok] *
                                      rows[ro.expert_idx[ok, j], ro.slot_idx[ok, j]]).sum(1)
            assert (err <= (d / 32 + 6) * 2.0 ** -24 * bound + 1e-30).all(), "d_weight rank %d" % r
            unit = type(ro)(**{**ro.__dict__, "weight": (ro.slot_idx >= 0).astype(np.float32)})
            assert_y_close(host(dxs[r]), orc.layout_bwd(d_disp[r], ro),
                           combine_bound(as_f64(d_disp[r]), unit), True, "dx rank %d" % r)


# ------------------------------------------------------------ failure handling
def test_sim_barrier_timeout_reports_error():
    """One rank reaches a device barrier and no peer ever does: the bounded
    barrier gives up after barrier_timeout_ms and moe_comm_check reports
    MOE_ERR_TIMEOUT instead of the stream hanging."""
    with moe.tuned(barrier_timeout_ms=50), moe.SimWorld(2) as world:
        c0 = world.comm(0)
        c0.check()                       # healthy before
        world.live_barrier(0)            # rank 1 never arrives
        with pytest.raises(moe.MoeError) as ei:
            c0.check()
        assert ei.value.status == 7      # MOE_ERR_TIMEOUT
        assert "gave up" in str(ei.value)
        world.comm(1).check()            # the other rank saw nothing


def test_sim_mismatched_programs_are_rejected():
    """A rank that skips a collective call: run() reports it, nothing hangs."""
    with moe.SimWorld(2) as world:
        world.comm(0).barrier()
        with pytest.raises(moe.MoeError) as ei:
            world.run()
        assert ei.value.status == 1
        world.run()                      # the queues were cleared: usable again


@pytest.mark.parametrize("mode", ["default", "nodedupe", "local_pad"])
@pytest.mark.parametrize("c", [P2P_CASES[i] for i in (0, 2, 3, 6, 7)],
                         ids=lambda c: "-".join("%s=%s" % kv for kv in c.items()))
def test_sim_gate_dispatch_fused(orc, c, mode):
    """moe_gate_dispatch_p2p (gate + NVLink row scatter as one persistent
    kernel, per simulated rank): routing bit-exact, receive buffers equal the
    oracle's AllToAll of the per-rank layouts, byte for byte."""
    with moe.tuned(**P2P_MODES[mode]), moe.SimWorld(c["P"]) as world:
        R = Ranks(orc, **c)
        recvs = R.symm(world, (R.E, R.cap, R.d))
        lg_dev = [dev(lg) for lg in R.lgs]
        outs = []
        gates = [moe.Gate(R.S, R.E, R.k, R.cap, R.kind) for _ in range(R.P)]  # alive until run()
        for r in range(R.P):
            outs.append(gates[r].with_dispatch_p2p(world.comm(r), R.x_dev[r], recvs[r], lg_dev[r]))
        world.run()
        torch.cuda.synchronize()
        want = orc.alltoall_flat(R.disp)
        for r in range(R.P):
            assert_routing_equal(outs[r], R.orc_routings[r], "rank %d" % r)
            assert host(recvs[r]).tobytes() == want[r].tobytes(), "recv of rank %d" % r


FULL = [("C2", 2), ("C2", 8), ("C3", 8), ("C4a", 8), ("C4b", 8)]


@pytest.mark.parametrize("wname,P", FULL, ids=lambda v: str(v))
def test_sim_full_size(orc, wname, P):
    """BASELINE.json's full per-rank sizes on P simulated ranks, the bench's
    launch configuration (RoutePipeline, one-sided path, s_e expert in place):
    every receive buffer byte-exact against the oracle's AllToAll, y within
    tolerance on a sample of 2048 tokens per rank (the oracle's combine of
    those tokens, from the oracle's own expert outputs)."""
    w = synthgen.WORKLOADS[wname]
    S, d, E, k = w.S, w.d, w.E, w.k
    cap = orc.capacity(S, E, k, w.C)
    El = E // P
    with moe.SimWorld(P) as world:
        ins = [synthgen.workload_inputs(w, r) for r in range(P)]
        pipes = [moe.RoutePipeline(S, d, E, k, cap, torch.bfloat16, w.kind, comm=world.comm(r),
                                   algo="p2p") for r in range(P)]
        dins = [[None if v is None else dev(v) for v in inp] for inp in ins]
        for r in range(P):   # gate (immediate) + dispatch (queued)
            lg, ids, table, x = dins[r]
            pipes[r].gate(lg, ids, table, out=pipes[r].routing)
            world.comm(r).dispatch_p2p(x, pipes[r].routing, pipes[r].recv)
        world.run()
        torch.cuda.synchronize()
        ros = [orc.gate(ins[r][0], E=E, k=k, cap=cap, kind=w.kind, token_ids=ins[r][1],
                        table=ins[r][2]) for r in range(P)]
        for r in range(P):
            assert_routing_equal(pipes[r].routing, ros[r], "rank %d" % r)
        recvs = orc.alltoall_flat([orc.layout(ins[r][3], ros[r]) for r in range(P)])
        for r in range(P):
            assert host(pipes[r].recv).tobytes() == recvs[r].tobytes(), "recv of rank %d" % r
        for r in range(P):   # the s_e stand-in, then the combine
            moe.expert_scale(pipes[r].recv, P, El, r * El, out=pipes[r].recv)
        for r in range(P):
            world.comm(r).combine_p2p(pipes[r].recv, pipes[r].routing, pipes[r].y)
        world.run()
        torch.cuda.synchronize()
        backs = orc.alltoall_flat([orc.expert_scale(recvs[q].reshape(P, El, cap, d), q * El)
                                   .reshape(E, cap, d) for q in range(P)])
        rng = np.random.default_rng(P * 7 + len(wname))
        for r in range(P):
            t = np.sort(rng.choice(S, 2048, replace=False))
            ro = ros[r]
            sub = type(ro)(**{**ro.__dict__, "expert_idx": ro.expert_idx[t], "slot_idx": ro.slot_idx[t],
                              "weight": ro.weight[t], "S": len(t)})
            y_o = orc.reverse_layout(backs[r], sub)
            assert_y_close(host(pipes[r].y)[t], y_o, combine_bound(as_f64(backs[r]), sub), True,
                           "rank %d" % r)
