"""GPU parity of the dropless packed layout through
the C ABI: expert offsets and the packed rows bit-exact, the packed combine
within the y bar (bit-exact for k = 1)."""
import numpy as np
import pytest
import torch

import synthgen
from gpu_util import as_f64, assert_routing_equal, assert_y_close, dev, host

pytestmark = pytest.mark.gpu

import paper_2203_14685_b200 as moe  # noqa: E402

CASES = [
    dict(kind="topk", S=4096, E=8, k=2, d=1024, dtype="bf16", dropless=True, skew=1.0),
    dict(kind="topk", S=3001, E=64, k=1, d=2048, dtype="bf16", dropless=True),
    dict(kind="topk", S=2000, E=16, k=4, d=256, dtype="f32", C=0.7, skew=1.5),
    dict(kind="hash", S=5000, E=32, k=1, d=1024, dtype="bf16", dropless=True),
    dict(kind="ktop1", S=1999, E=32, k=2, d=512, dtype="bf16", dropless=True),
    dict(kind="topk", S=777, E=5, k=3, d=8, dtype="bf16", dropless=True),      # 16-byte rows
    dict(kind="topk", S=1, E=4, k=1, d=64, dtype="f32", dropless=True),
]


def _routing(orc, c):
    S, E, k = c["S"], c["E"], c["k"]
    cap = S * k if c.get("dropless") else orc.capacity(S, E, k, c.get("C", 1.0))
    if c["kind"] == "hash":
        ids, table = synthgen.hash_inputs(S + 3, S, 4096, E)
        ro = orc.gate(None, E=E, k=1, cap=cap, kind="hash", token_ids=ids, table=table)
        rg = moe.Gate(S, E, 1, cap, "hash")(None, dev(ids), dev(table), slot_src=False)
    else:
        lg = synthgen.logits(S + 17, S, E, k, c["kind"], skew=c.get("skew", 0.0))
        ro = orc.gate(lg, E=E, k=k, cap=cap, kind=c["kind"])
        rg = moe.Gate(S, E, k, cap, c["kind"])(dev(lg), slot_src=False)
    torch.cuda.synchronize()
    return ro, rg


@pytest.mark.parametrize("c", CASES, ids=lambda c: "-".join("%s=%s" % kv for kv in c.items()))
def test_packed_layout_and_combine(orc, c):
    ro, rg = _routing(orc, c)
    ro.slot_src = None
    assert (host(rg.slot_idx) == ro.slot_idx).all() and (host(rg.load) == ro.load).all()
    off_o = orc.expert_offsets(ro)
    off_g = moe.expert_offsets(rg)
    assert (host(off_g) == off_o).all()
    if c.get("dropless"):
        assert (ro.slot_idx >= 0).sum() == off_o[-1] == (ro.expert_idx >= 0).sum()
    S, d, bf16 = c["S"], c["d"], c["dtype"] == "bf16"
    x = synthgen.tokens(S * 3 + d, S, d, c["dtype"])
    R = int(off_o[-1])
    packed = host(moe.layout_packed(dev(x), rg, off_g))
    assert packed[:R].tobytes() == orc.layout_packed(x, ro, off_o).tobytes()
    back = synthgen.tokens(S * 5 + d, R, d, c["dtype"])
    y_o = orc.reverse_layout_packed(back, ro, off_o)
    back_pad = np.concatenate([back, np.zeros((S * c["k"] - R, d), back.dtype)])
    y_g = host(moe.reverse_layout_packed(dev(back_pad), rg, off_g))
    # the bound sum_j |w_j a_j| over the packed rows
    bound = np.zeros((S, d))
    b64 = as_f64(back)
    for j in range(c["k"]):
        ok = ro.slot_idx[:, j] >= 0
        rows = off_o[ro.expert_idx[ok, j]] + ro.slot_idx[ok, j]
        bound[ok] += np.abs(ro.weight[ok, j].astype(np.float64)[:, None] * b64[rows])
    assert_y_close(y_g, y_o, bound, bf16)
    if c["k"] == 1:
        assert y_g.tobytes() == y_o.tobytes()


@pytest.mark.parametrize("c", [c for c in CASES if c["S"] > 1],
                         ids=lambda c: "-".join("%s=%s" % kv for kv in c.items()))
def test_packed_backward(orc, c):
    """Adjoints of the packed form against the padded oracle adjoints with
    the padding removed (the packed form IS the padded one minus padding)."""
    ro, rg = _routing(orc, c)
    S, E, k, d = c["S"], c["E"], c["k"], c["d"]
    cap = ro.cap
    off_o = orc.expert_offsets(ro)
    off_g = moe.expert_offsets(rg)
    R = int(off_o[-1])
    dy = synthgen.tokens(S * 7 + d, S, d, c["dtype"])
    back_pk = synthgen.tokens(S * 9 + d, R, d, c["dtype"])
    # the same rows in the padded form (padding rows zero)
    back_pad = np.zeros((E, cap, d), back_pk.dtype)
    for e in range(E):
        back_pad[e, :off_o[e + 1] - off_o[e]] = back_pk[off_o[e]:off_o[e + 1]]
    db_o, dw_o = orc.reverse_layout_bwd(dy, back_pad, ro)
    db_o_pk = np.concatenate([db_o[e, :off_o[e + 1] - off_o[e]] for e in range(E)])
    pad_rows = np.concatenate([back_pk, np.zeros((S * k - R, d), back_pk.dtype)])
    db_g, dw_g = moe.reverse_layout_packed_backward(dev(dy), dev(pad_rows), rg, off_g)
    torch.cuda.synchronize()
    assert host(db_g)[:R].tobytes() == db_o_pk.tobytes()
    err = np.abs(host(dw_g).astype(np.float64) - dw_o.astype(np.float64))
    bound = np.zeros_like(err)
    b64, dy64 = as_f64(back_pad), as_f64(dy)
    for j in range(k):
        ok = ro.slot_idx[:, j] >= 0
        bound[ok, j] = np.abs(dy64[ok] * b64[ro.expert_idx[ok, j], ro.slot_idx[ok, j]]).sum(1)
    assert (err <= (d / 32 + 6) * 2.0 ** -24 * bound + 1e-30).all()
    # layout adjoint: gradient rows in the packed form
    g_pk = synthgen.tokens(S * 11 + d, R, d, c["dtype"])
    g_pad = np.zeros((E, cap, d), g_pk.dtype)
    for e in range(E):
        g_pad[e, :off_o[e + 1] - off_o[e]] = g_pk[off_o[e]:off_o[e + 1]]
    dx_o = orc.layout_bwd(g_pad, ro)
    dx_g = host(moe.layout_packed_backward(
        dev(np.concatenate([g_pk, np.zeros((S * k - R, d), g_pk.dtype)])), rg, off_g))
    unit = type(ro)(**{**ro.__dict__, "weight": (ro.slot_idx >= 0).astype(np.float32)})
    from gpu_util import combine_bound
    assert_y_close(dx_g, dx_o, combine_bound(as_f64(g_pad), unit), c["dtype"] == "bf16")
