"""GPU parity of the routing path's backward through
the C ABI, against the oracle's adjoints on the same seeded inputs.

Bars (derived from the arithmetic):
  - d_back: bit-exact (one rounding of an exact product on both sides);
  - d_weight: fp32 dot product, per-lane sequential FMA over d/32 columns then
    a 5-level tree: |err| <= (d/32 + 6) * 2^-24 * sum_c |dy_c back_c|;
  - dx: the combine with unit weights: the y bar (1e-6 fp32 / 1e-2 bf16 of
    sum |a|), bit-exact for k = 1;
  - d_logits: both sides fp64 with a different summation order and exp, one
    rounding: |err| <= 2.4e-7 |ref| + 1e-12 sum_j |g_j|.
"""
import numpy as np
import pytest
import torch

import synthgen
from gpu_util import as_f64, assert_routing_equal, assert_y_close, dev, host

pytestmark = pytest.mark.gpu

import paper_2203_14685_b200 as moe  # noqa: E402
from paper_2203_14685_b200 import autograd as ag  # noqa: E402

CASES = [
    dict(kind="topk", S=1024, E=4, k=1, d=64, dtype="f32"),
    dict(kind="topk", S=3001, E=8, k=2, d=1024, dtype="bf16"),
    dict(kind="topk", S=2000, E=64, k=1, d=2048, dtype="bf16", C=0.8),
    dict(kind="ktop1", S=1999, E=32, k=2, d=1024, dtype="bf16", mode="softmax"),
    dict(kind="topk", S=777, E=5, k=3, d=8, dtype="bf16", C=0.6),        # 16-byte rows
    dict(kind="topk", S=500, E=8, k=2, d=12, dtype="f32", cap=3),        # 48-byte rows
    dict(kind="topk", S=1500, E=16, k=4, d=2056, dtype="bf16", prio="slot", skew=1.0),
    dict(kind="topk", S=600, E=32, k=8, d=256, dtype="f32", mode="softmax", skew=2.0),
    dict(kind="topk", S=300, E=16, k=12, d=128, dtype="f32", C=0.5),     # rank-path gate
    dict(kind="ktop1", S=400, E=8, k=8, d=64, dtype="f32", mode="softmax"),
    dict(kind="hash", S=2000, E=32, k=1, d=1024, dtype="bf16", C=1.25),
]


def _setup(orc, c):
    S, E, k, d = c["S"], c["E"], c["k"], c["d"]
    cap = c.get("cap") or orc.capacity(S, E, k, c.get("C", 1.0))
    mode, prio = c.get("mode", "renorm"), c.get("prio", "token")
    if c["kind"] == "hash":
        ids, table = synthgen.hash_inputs(S + 5, S, 4096, E)
        lg = None
        ro = orc.gate(None, E=E, k=k, cap=cap, kind="hash", token_ids=ids, table=table)
        rg = moe.Gate(S, E, k, cap, "hash")(None, dev(ids), dev(table))
    else:
        lg = synthgen.logits(S * 3 + E, S, E, k, c["kind"], skew=c.get("skew", 0.0))
        ro = orc.gate(lg, E=E, k=k, cap=cap, kind=c["kind"], weight_mode=mode, priority=prio)
        rg = moe.Gate(S, E, k, cap, c["kind"], mode, prio)(dev(lg))
    torch.cuda.synchronize()
    assert_routing_equal(rg, ro)
    return lg, ro, rg, cap


def _dot_bound(dy64, back64, ro):
    S, k = ro.expert_idx.shape
    d = dy64.shape[1]
    out = np.zeros((S, k))
    for j in range(k):
        ok = ro.slot_idx[:, j] >= 0
        rows = back64[ro.expert_idx[ok, j], ro.slot_idx[ok, j]]
        out[ok, j] = np.abs(dy64[ok] * rows).sum(1)
    return (d / 32 + 6) * 2.0 ** -24 * out


@pytest.mark.parametrize("pads_first", [0, 1])   # padding rows of d_back zeroed last / first
@pytest.mark.parametrize("c", CASES, ids=lambda c: "-".join("%s=%s" % kv for kv in c.items()))
def test_combine_and_layout_backward(orc, c, pads_first):
    with moe.tuned(layout_pads_first=pads_first):
        _combine_and_layout_backward(orc, c)


def _combine_and_layout_backward(orc, c):
    lg, ro, rg, cap = _setup(orc, c)
    S, E, d, bf16 = c["S"], c["E"], c["d"], c["dtype"] == "bf16"
    dy = synthgen.tokens(S * 7 + d, S, d, c["dtype"])
    back = synthgen.tokens(S * 11 + d, E * cap, d, c["dtype"]).reshape(E, cap, d)
    db_o, dw_o = orc.reverse_layout_bwd(dy, back, ro)
    db_g, dw_g = moe.reverse_layout_backward(dev(dy), dev(back), rg)
    torch.cuda.synchronize()
    assert host(db_g).tobytes() == db_o.tobytes()            # incl. zeroed padding rows
    err = np.abs(host(dw_g).astype(np.float64) - dw_o.astype(np.float64))
    tol = _dot_bound(as_f64(dy), as_f64(back), ro) + 1e-30
    assert (err <= tol).all(), "d_weight: worst %.3g" % (err - tol).max()
    assert (host(dw_g)[ro.slot_idx < 0] == 0).all()
    # adjoint of the layout on an independent gradient buffer
    g = synthgen.tokens(S * 13 + d, E * cap, d, c["dtype"]).reshape(E, cap, d)
    dx_o = orc.layout_bwd(g, ro)
    dx_g = host(moe.layout_backward(dev(g), rg))
    unit = type(ro)(**{**ro.__dict__, "weight": (ro.slot_idx >= 0).astype(np.float32)})
    from gpu_util import combine_bound
    assert_y_close(dx_g, dx_o, combine_bound(as_f64(g), unit), bf16, "dx")
    if ro.k == 1:
        assert dx_g.tobytes() == dx_o.tobytes()
    assert (dx_g[(ro.slot_idx < 0).all(1)] == 0).all()


def _gate_tol(ref, g, ro):
    gs = np.abs(g.astype(np.float64) * (ro.slot_idx >= 0)).sum(1, keepdims=True)
    return 2.4e-7 * np.abs(ref.astype(np.float64)) + 1e-12 * gs


@pytest.mark.parametrize("c", [c for c in CASES if c["kind"] != "hash"] + [
    dict(kind="topk", S=257, E=256, k=2, d=0, dtype="f32", mode="softmax"),
    dict(kind="topk", S=257, E=3, k=2, d=0, dtype="f32"),
    dict(kind="ktop1", S=300, E=256, k=256, d=0, dtype="f32", mode="softmax"),
    dict(kind="ktop1", S=300, E=64, k=4, d=0, dtype="f32"),
], ids=lambda c: "-".join("%s=%s" % kv for kv in c.items()))
def test_gate_backward(orc, c):
    lg, ro, rg, cap = _setup(orc, c)
    mode = c.get("mode", "renorm")
    g = np.random.default_rng(c["S"]).standard_normal((c["S"], c["k"])).astype(np.float32)
    ref = orc.gate_bwd(lg, ro, g, kind=c["kind"], weight_mode=mode)
    got = host(moe.gate_backward(dev(lg), rg, dev(g)))
    err = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    tol = _gate_tol(ref, g, ro)
    assert (err <= tol).all(), "d_logits: %d bad, worst %.3g" % ((err > tol).sum(), (err - tol).max())


def test_gate_backward_rejects_hash():
    with pytest.raises(moe.MoeError):
        r = moe.Routing.empty(8, 4, 1, 8, "cuda", kind=2)
        moe.gate_backward(torch.zeros((8, 4), device="cuda"), r, torch.zeros((8, 1), device="cuda"))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_autograd_chain(orc, dtype):
    """gate_weights -> dispatch -> (identity expert) -> combine, loss = <y, dy>:
    torch autograd through the library's adjoint kernels matches the oracle's
    adjoint chain."""
    S, E, k, d = 2048, 8, 2, 256
    cap = orc.capacity(S, E, k, 0.9)
    lg = synthgen.logits(41, S, E, k, skew=0.5)
    x = synthgen.tokens(42, S, d, dtype)
    dy = synthgen.tokens(43, S, d, dtype)
    g = moe.Gate(S, E, k, cap)
    lg_t = dev(lg).requires_grad_(True)
    x_t = dev(x).requires_grad_(True)
    rs = []
    w = ag.gate_weights(lg_t, g, rs)
    r = rs[0]
    disp = ag.dispatch(x_t, r)
    y = ag.combine(disp, w, r)
    y.backward(dev(dy))
    torch.cuda.synchronize()
    ro = orc.gate(lg, E=E, k=k, cap=cap)
    assert_routing_equal(r, ro)
    disp_o = orc.layout(x, ro)
    assert host(disp).tobytes() == disp_o.tobytes()
    db_o, dw_o = orc.reverse_layout_bwd(dy, disp_o, ro)
    dx_o = orc.layout_bwd(db_o, ro)
    dl_o = orc.gate_bwd(lg, ro, dw_o)
    # dx: d_back is bit-exact, so only the layout adjoint's bar applies
    from gpu_util import combine_bound
    unit = type(ro)(**{**ro.__dict__, "weight": (ro.slot_idx >= 0).astype(np.float32)})
    assert_y_close(host(x_t.grad), dx_o, combine_bound(as_f64(db_o), unit), dtype == "bf16", "dx")
    # d_logits: the gate bar plus the propagated d_weight error
    # (|d d_l / d g_j| <= p_j (1 + p_e) <= 2)
    dw_tol = _dot_bound(as_f64(dy), as_f64(disp_o), ro)
    tol = _gate_tol(dl_o, dw_o, ro) + 2.0 * dw_tol.sum(1, keepdims=True)
    err = np.abs(host(lg_t.grad).astype(np.float64) - dl_o.astype(np.float64))
    assert (err <= tol).all()
