"""GPU parity: libmoe_b200 (through its C ABI, via the thin binding) against
the CPU oracle on identical seeded inputs.

Bar: routing (expert ids, slots, drop mask, load, slot_src),
dispatch buffers and the expert stand-in bit-exact; weights within 2 ulp;
y within 1e-6 (fp32) / 1e-2 (bf16) of sum_j |w_j a_j|, bit-exact for k=1.
"""
import numpy as np
import pytest
import torch

import synthgen
from gpu_util import (as_f64, assert_routing_equal, assert_y_close, combine_bound, dev, host)

pytestmark = pytest.mark.gpu

import paper_2203_14685_b200 as moe  # noqa: E402


def _inputs(case):
    kind, S, E, k = case["kind"], case["S"], case["E"], case["k"]
    seed = case.get("seed", S * 131 + E * 7 + k)
    if kind == "hash":
        ids, table = synthgen.hash_inputs(seed, S, case.get("V", 4096), E)
        if "bad_ids" in case:
            ids[case["bad_ids"]] = case.get("bad_val", -5)
        return None, ids, table
    if case.get("ties"):
        rng = np.random.default_rng(seed)
        lg = rng.integers(-2, 3, size=(S, E)).astype(np.float32)
        lg[rng.random((S, E)) < 0.05] = -0.0
    elif case.get("equal"):
        lg = np.zeros((S, E), np.float32)
    else:
        lg = synthgen.logits(seed, S, E, k, kind, skew=case.get("skew", 0.0))
    return lg, None, None


def _run_gate(orc, case):
    kind, S, E, k = case["kind"], case["S"], case["E"], case["k"]
    cap = case.get("cap") or orc.capacity(S, E, k, case.get("C", 1.0))
    mode, prio = case.get("mode", "renorm"), case.get("prio", "token")
    lg, ids, table = _inputs(case)
    ro = orc.gate(lg, E=E, k=k, cap=cap, kind=kind, weight_mode=mode, priority=prio,
                  token_ids=ids, table=table)
    g = moe.Gate(S, E, k, cap, kind, mode, prio)
    rg = g(None if lg is None else dev(lg), None if ids is None else dev(ids),
           None if table is None else dev(table))
    torch.cuda.synchronize()
    return rg, ro, g, (lg, ids, table)


GATE_CASES = [
    # headline shapes (C1, C2, C3, C4a, C4b) at reduced S
    dict(kind="topk", S=1024, E=4, k=1),
    dict(kind="topk", S=4096, E=8, k=2),
    dict(kind="topk", S=4096, E=64, k=1),
    dict(kind="ktop1", S=4096, E=32, k=2),
    dict(kind="hash", S=4096, E=32, k=1, C=1.25),
    # ragged tails, S=1, tiny and odd E, all k paths (register K=1,2,4,8; rank path)
    dict(kind="topk", S=1, E=8, k=2),
    dict(kind="topk", S=257, E=3, k=2),
    dict(kind="topk", S=1000, E=5, k=5),
    dict(kind="topk", S=999, E=1, k=1),
    dict(kind="topk", S=777, E=16, k=3),
    dict(kind="topk", S=3000, E=24, k=4),
    dict(kind="topk", S=2049, E=128, k=8),
    dict(kind="topk", S=600, E=256, k=2),
    dict(kind="topk", S=500, E=32, k=12),      # rank path
    dict(kind="topk", S=300, E=16, k=16),      # k = E, rank path
    dict(kind="topk", S=513, E=33, k=2),       # E not a multiple of 4 / 8
    # weight modes and priorities
    dict(kind="topk", S=3001, E=64, k=2, mode="softmax"),
    dict(kind="topk", S=3001, E=8, k=2, prio="slot"),
    dict(kind="topk", S=2500, E=16, k=4, prio="slot", C=0.7, skew=1.0),
    dict(kind="topk", S=700, E=8, k=12 - 4, prio="slot", mode="softmax"),
    dict(kind="ktop1", S=2000, E=32, k=4, mode="softmax"),
    dict(kind="ktop1", S=1500, E=64, k=16),     # rank path
    dict(kind="ktop1", S=1500, E=64, k=16, mode="softmax"),
    dict(kind="ktop1", S=800, E=6, k=3, prio="slot"),
    dict(kind="ktop1", S=800, E=8, k=8),        # one expert per prototype
    # capacity pressure: cap=1, heavy skew, everyone to one expert, ties
    dict(kind="topk", S=1000, E=8, k=2, cap=1),
    dict(kind="topk", S=5000, E=8, k=1, C=0.5, skew=3.0),
    dict(kind="topk", S=5000, E=8, k=2, skew=50.0),
    dict(kind="topk", S=2048, E=8, k=2, ties=True),
    dict(kind="topk", S=2048, E=64, k=4, ties=True, prio="slot"),
    dict(kind="ktop1", S=2048, E=32, k=2, ties=True),
    dict(kind="topk", S=1024, E=4, k=2, equal=True, C=0.5),
    dict(kind="hash", S=3000, E=8, k=1, C=0.5),
    dict(kind="hash", S=3000, E=16, k=1, bad_ids=[0, 7, 2999], bad_val=1 << 20),
]


# kernel variants selected by the library's tuning table (moe.tuned)
GATE_PATHS = {"two": {}, "three": {"gate_two_maxw": 0},
              "two_forced": {"gate_two_maxw": 1000000},
              "tile256": {"gate_max_tile": 256, "gate_tiles": 1},
              "tile32": {"gate_max_tile": 32}}
ROW_PATHS = {"default": {}, "layout_u4_rev_ku4": {"layout_u": 4, "reverse_ku": 4},
             "layout_u1": {"layout_u": 1},
             "reverse_tpw_off": {"reverse_tpw": 0}, "reverse_tpw_on": {"reverse_tpw": 1},
             "reverse_generic": {"reverse_kspec": 0}, "reverse_u2": {"reverse_ku": 2},
             "forward_order": {"reverse_backwards": 0, "reverse_y_ef": 0},
             "reverse_generic_fwd": {"reverse_kspec": 0, "reverse_backwards": 0},
             "pads_first": {"layout_pads_first": 1}, "pads_last": {"layout_pads_first": 0},
             "one_cta_per_sm": {"row_ctas_per_sm": 1},
             "layout_persistent": {"layout_tokens_per_warp": 0},
             "layout_one_token_per_warp": {"layout_tokens_per_warp": 1}}


@pytest.mark.parametrize("path", sorted(GATE_PATHS))
@pytest.mark.parametrize("case", GATE_CASES, ids=lambda c: "-".join(
    "%s=%s" % (k, v) for k, v in c.items() if k not in ("bad_ids",)))
def test_gate_parity(orc, case, path):
    with moe.tuned(**GATE_PATHS[path]):
        rg, ro, g, _ = _run_gate(orc, case)
    assert_routing_equal(rg, ro, str(case))
    if case["kind"] == "hash":
        assert g.check() == ro.bad


@pytest.mark.parametrize("path", sorted(GATE_PATHS))
def test_gate_workspace_reuse_and_graph_replay(orc, path):
    """The workspace resets itself (counters): repeated calls, and CUDA-graph
    replays with new inputs, each match the oracle."""
    with moe.tuned(**GATE_PATHS[path]):
        _gate_reuse_and_replay(orc)


def _gate_reuse_and_replay(orc):
    S, E, k = 3000, 16, 2
    cap = orc.capacity(S, E, k, 1.0)
    g = moe.Gate(S, E, k, cap)
    lg_dev = torch.empty((S, E), dtype=torch.float32, device="cuda")
    out = moe.Routing.empty(S, E, k, cap, "cuda")
    for it in range(3):
        lg = synthgen.logits(900 + it, S, E, k, skew=0.3 * it)
        lg_dev.copy_(dev(lg))
        g(lg_dev, out=out)
        torch.cuda.synchronize()
        assert_routing_equal(out, orc.gate(lg, E=E, k=k, cap=cap), "call %d" % it)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            g(lg_dev, out=out)
    torch.cuda.current_stream().wait_stream(s)
    for it in range(3):
        lg = synthgen.logits(950 + it, S, E, k)
        lg_dev.copy_(dev(lg))
        graph.replay()
        torch.cuda.synchronize()
        assert_routing_equal(out, orc.gate(lg, E=E, k=k, cap=cap), "replay %d" % it)


LAYOUT_CASES = [
    dict(kind="topk", S=1024, E=4, k=1, d=64, dtype="f32"),
    dict(kind="topk", S=3001, E=8, k=2, d=1024, dtype="bf16"),
    dict(kind="topk", S=2000, E=64, k=1, d=2048, dtype="bf16"),
    dict(kind="ktop1", S=1999, E=32, k=2, d=1024, dtype="bf16"),
    dict(kind="hash", S=2000, E=32, k=1, d=1024, dtype="bf16", C=1.25),
    dict(kind="topk", S=777, E=5, k=3, d=8, dtype="bf16", C=0.6),     # 16-byte rows
    dict(kind="topk", S=500, E=8, k=2, d=12, dtype="f32", cap=3),     # 48-byte rows
    dict(kind="topk", S=1500, E=16, k=4, d=2056, dtype="bf16", prio="slot", skew=1.0),
    dict(kind="topk", S=300, E=8, k=2, d=4096, dtype="f32", skew=40.0),
    dict(kind="topk", S=64, E=1, k=1, d=96, dtype="bf16"),
    dict(kind="topk", S=1000, E=16, k=6, d=256, dtype="bf16", C=0.8),          # k > 4: inline dsts
    dict(kind="ktop1", S=900, E=32, k=8, d=128, dtype="f32", mode="softmax"),  # 8 prototypes
]


@pytest.mark.parametrize("path", sorted(ROW_PATHS))
@pytest.mark.parametrize("case", LAYOUT_CASES, ids=lambda c: "-".join(
    "%s=%s" % (k, v) for k, v in c.items()))
def test_layout_and_reverse_parity(orc, case, path):
    with moe.tuned(**ROW_PATHS[path]):
        _layout_and_reverse(orc, case)


def _layout_and_reverse(orc, case):
    rg, ro, _, _ = _run_gate(orc, case)
    assert_routing_equal(rg, ro)
    S, d, bf16 = case["S"], case["d"], case["dtype"] == "bf16"
    x = synthgen.tokens(S + d, S, d, case["dtype"])
    disp_o = orc.layout(x, ro)
    disp_g = moe.layout(dev(x), rg)
    torch.cuda.synchronize()
    assert host(disp_g).tobytes() == disp_o.tobytes()   # incl. zeroed padding rows
    # combine on an independent synthetic expert output
    back = synthgen.tokens(d * 3 + 1, ro.E * ro.cap, d, case["dtype"]).reshape(ro.E, ro.cap, d)
    y_o = orc.reverse_layout(back, ro)
    y_g = host(moe.reverse_layout(dev(back), rg))
    assert_y_close(y_g, y_o, combine_bound(as_f64(back), ro), bf16, str(case))
    if ro.k == 1 and case.get("mode", "renorm") == "renorm":
        assert y_g.tobytes() == y_o.tobytes()            # w = 1: bit-exact
    # fully dropped tokens are exactly zero
    dead = (ro.slot_idx < 0).all(1)
    assert (y_g[dead] == 0).all()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_round_trip_bitwise(orc, dtype):
    """k=1, no drops, unit weights -> reverse(layout(x)) == x."""
    S, E, d = 4097, 8, 256
    lg = synthgen.logits(77, S, E, 1)
    rg = moe.gate(dev(lg), k=1, capacity_=S)
    x = synthgen.tokens(78, S, d, dtype)
    y = moe.reverse_layout(moe.layout(dev(x), rg), rg)
    assert host(y).tobytes() == x.tobytes()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_expert_scale_bit_exact(orc, dtype):
    nsrc, El, cap, d, e_base = 3, 4, 37, 128, 5
    buf = synthgen.tokens(79, nsrc * El * cap, d, dtype).reshape(nsrc, El, cap, d)
    want = orc.expert_scale(buf, e_base)
    got = moe.expert_scale(dev(buf), nsrc, El, e_base, out=torch.empty_like(dev(buf)))
    assert host(got).tobytes() == want.tobytes()


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4a", "C4b"])
def test_pipeline_full_size_p1(orc, name):
    """Every BASELINE config at its full per-rank size, one rank, in the
    launch configuration bench.py times (RoutePipeline), expert stand-in on:
    routing and dispatch bit-exact, y within tolerance."""
    w = synthgen.WORKLOADS[name]
    lg, ids, table, x = synthgen.workload_inputs(w, 0)
    cap = orc.capacity(w.S, w.E, w.k, w.C)
    dt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    pipe = moe.RoutePipeline(w.S, w.d, w.E, w.k, cap, dt, w.kind)
    y = pipe.step(None if lg is None else dev(lg), dev(x), None if ids is None else dev(ids),
                  None if table is None else dev(table), expert=True)
    torch.cuda.synchronize()
    routings, disp, recvs, ys = orc.route_multi([x], None if lg is None else [lg], E=w.E, k=w.k,
                                                cap=cap, kind=w.kind,
                                                token_ids_list=None if ids is None else [ids],
                                                table=table)
    ro = routings[0]
    assert_routing_equal(pipe.routing, ro, name)
    # after the in-place expert stand-in the dispatch buffer holds s_e * rows
    back_o = orc.expert_scale(disp[0].reshape(1, w.E, cap, w.d), 0).reshape(w.E, cap, w.d)
    assert host(pipe.dispatch).tobytes() == back_o.tobytes()
    assert_y_close(host(y), ys[0], combine_bound(as_f64(back_o), ro), w.dtype == "bf16", name)
    if name == "C4b":
        assert (ro.slot_idx >= 0).all()      # C=1.25: the hash config drops nothing (R12)


def test_determinism(orc):
    w = synthgen.WORKLOADS["C2"]
    lg, _, _, x = synthgen.workload_inputs(w, 0, S=8192)
    cap = orc.capacity(8192, w.E, w.k, w.C)
    pipe = moe.RoutePipeline(8192, w.d, w.E, w.k, cap, torch.bfloat16)
    a = host(pipe.step(dev(lg), dev(x))).copy()
    r1 = [host(t).copy() for t in (pipe.routing.slot_idx, pipe.routing.slot_src)]
    b = host(pipe.step(dev(lg), dev(x)))
    r2 = [host(t) for t in (pipe.routing.slot_idx, pipe.routing.slot_src)]
    assert a.tobytes() == b.tobytes()
    assert all(u.tobytes() == v.tobytes() for u, v in zip(r1, r2))


def test_run_host_pipelined_matches_step(orc):
    """RoutePipeline.run_host (copies on their own streams, double-buffered
    staging) returns, for every batch, exactly the y that step() gives for
    that batch alone -- no buffer is overwritten while in use -- and the
    oracle's y within the north_star bar."""
    S, d, E, k = 4096, 512, 8, 2
    cap = orc.capacity(S, E, k, 1.0)
    pipe = moe.RoutePipeline(S, d, E, k, cap, torch.bfloat16)
    batches, want = [], []
    for i in range(5):
        lg = synthgen.logits(300 + i, S, E, k)
        x = synthgen.tokens(400 + i, S, d, "bf16")
        batches.append({"logits": torch.from_numpy(lg).pin_memory(),
                        "x": torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).pin_memory()})
        want.append(host(pipe.step(dev(lg), dev(x))).copy())
        _, disp, _, ys = orc.route_multi([x], [lg], E=E, k=k, cap=cap, scale=False)
        ro = orc.gate(lg, E=E, k=k, cap=cap)
        assert_y_close(want[-1], ys[0], combine_bound(as_f64(disp[0]), ro), True)
    torch.cuda.synchronize()
    outs = [torch.empty((S, d), dtype=torch.bfloat16).pin_memory() for _ in range(5)]
    pipe.run_host(batches, outs)
    torch.cuda.synchronize()
    for i in range(5):
        assert host(outs[i]).tobytes() == want[i].tobytes(), "batch %d" % i


@pytest.mark.parametrize("case", [c for c in LAYOUT_CASES] + [
    dict(kind="topk", S=4096, E=64, k=1, d=2048, dtype="bf16", prio="slot"),
    dict(kind="topk", S=65536, E=32, k=2, d=256, dtype="bf16"),             # scanned table
    dict(kind="topk", S=3000, E=16, k=2, d=256, dtype="bf16", prio="slot", C=0.8),
    dict(kind="topk", S=65536, E=32, k=2, d=128, dtype="f32", prio="slot", C=0.9),  # scanned, SLOT
    dict(kind="ktop1", S=5000, E=32, k=4, d=64, dtype="f32", mode="softmax", C=0.7),
    dict(kind="hash", S=3000, E=16, k=1, d=128, dtype="f32", bad_ids=[0, 7], bad_val=1 << 20),
], ids=lambda c: "-".join("%s=%s" % kv for kv in c.items() if kv[0] != "bad_ids"))
def test_gate_layout_fused_equals_gate_then_layout(orc, case):
    """moe_gate_layout (the capacity pass inside the layout kernel) gives the
    same routing and dispatch as the oracle (and thus as gate + layout)."""
    kind, S, E, k, d = case["kind"], case["S"], case["E"], case["k"], case["d"]
    cap = case.get("cap") or orc.capacity(S, E, k, case.get("C", 1.0))
    mode, prio = case.get("mode", "renorm"), case.get("prio", "token")
    lg, ids, table = _inputs(case)
    ro = orc.gate(lg, E=E, k=k, cap=cap, kind=kind, weight_mode=mode, priority=prio,
                  token_ids=ids, table=table)
    x = synthgen.tokens(S + d + 1, S, d, case["dtype"])
    g = moe.Gate(S, E, k, cap, kind, mode, prio)
    xd = dev(x)
    disp = torch.empty((E, cap, d), dtype=xd.dtype, device="cuda")
    rg = g.with_layout(xd, disp, None if lg is None else dev(lg),
                       None if ids is None else dev(ids), None if table is None else dev(table))
    torch.cuda.synchronize()
    assert_routing_equal(rg, ro, str(case))
    assert host(disp).tobytes() == orc.layout(x, ro).tobytes()
    if kind == "hash":
        assert g.check() == ro.bad


@pytest.mark.parametrize("tile", [32, 64, 0, 256])   # gate_max_tile (0: the default)
@pytest.mark.parametrize("case", [
    dict(kind="topk", S=32768, E=8, k=2, d=1024),           # C2 shape
    dict(kind="topk", S=8192, E=64, k=1, d=2048),           # C3 rows (4 KiB, U = 4)
    dict(kind="ktop1", S=20000, E=32, k=2, d=512),
    dict(kind="hash", S=20000, E=32, k=1, d=512, C=1.25),
    dict(kind="topk", S=3333, E=256, k=8, d=128, C=0.7),     # widest gate, K = 8
    dict(kind="topk", S=1, E=4, k=2, d=64),                  # one token
], ids=lambda c: "-".join("%s=%s" % kv for kv in c.items()))
def test_gate_layout_fused_replays(orc, case, tile):
    """The fused kernel's device-side tile counter, epoch-tagged look-back
    words and ready word reset themselves: eager calls and CUDA-graph replays
    with new inputs each match the oracle, for every tile size."""
    kind, S, E, k, d = case["kind"], case["S"], case["E"], case["k"], case["d"]
    cap = orc.capacity(S, E, k, case.get("C", 1.0))
    with moe.tuned(gate_max_tile=tile):
        g = moe.Gate(S, E, k, cap, kind)
        xd = torch.empty((S, d), dtype=torch.bfloat16, device="cuda")
        lgd = torch.empty((S, E), dtype=torch.float32, device="cuda")
        idd = torch.empty((S,), dtype=torch.int32, device="cuda")
        disp = torch.empty((E, cap, d), dtype=torch.bfloat16, device="cuda")
        out = moe.Routing.empty(S, E, k, cap, "cuda", g.kind, g.mode, g.prio)
        table = None
        if kind == "hash":
            ids, table = synthgen.hash_inputs(4242, S, 32768, E)
            table_d = dev(table)

        def fill(it):
            x = synthgen.tokens(700 + it, S, d, "bf16")
            xd.copy_(dev(x))
            if kind == "hash":
                ids = synthgen.hash_inputs(4300 + it, S, 32768, E)[0]
                idd.copy_(dev(ids))
                return x, None, ids
            lg = synthgen.logits(800 + it, S, E, k, kind, skew=0.2 * it)
            lgd.copy_(dev(lg))
            return x, lg, None

        def call():
            if kind == "hash":
                g.with_layout(xd, disp, None, idd, table_d, out=out)
            else:
                g.with_layout(xd, disp, lgd, out=out)

        def check(x, lg, ids, what):
            ro = orc.gate(lg, E=E, k=k, cap=cap, kind=kind, token_ids=ids, table=table)
            assert_routing_equal(out, ro, what)
            assert host(disp).tobytes() == orc.layout(x, ro).tobytes(), what

        for it in range(2):
            v = fill(it)
            call()
            torch.cuda.synchronize()
            check(*v, "eager %d" % it)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                call()
        torch.cuda.current_stream().wait_stream(s)
        for it in range(2, 5):
            v = fill(it)
            graph.replay()
            torch.cuda.synchronize()
            check(*v, "replay %d" % it)


@pytest.mark.parametrize("fuse", [False, True])
def test_route_pipeline_nvtx_and_fuse(orc, fuse):
    """RoutePipeline with NVTX ranges and with / without the fused gate +
    layout: the same routing, dispatch and y as the oracle."""
    S, d, E, k = 3000, 256, 16, 2
    cap = orc.capacity(S, E, k, 1.0)
    lg = synthgen.logits(4242, S, E, k)
    x = synthgen.tokens(4343, S, d, "bf16")
    pipe = moe.RoutePipeline(S, d, E, k, cap, torch.bfloat16, nvtx=True, fuse_gate_layout=fuse)
    y = host(pipe.step(dev(lg), dev(x)))
    torch.cuda.synchronize()
    ro = orc.gate(lg, E=E, k=k, cap=cap)
    assert_routing_equal(pipe.routing, ro)
    disp = orc.layout(x, ro)
    assert host(pipe.dispatch).tobytes() == disp.tobytes()
    assert_y_close(y, orc.reverse_layout(disp, ro), combine_bound(as_f64(disp), ro), True)
