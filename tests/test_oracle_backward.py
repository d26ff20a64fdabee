"""Pins of the oracle's backward of the routing path:
orc_reverse_layout_bwd, orc_layout_bwd, orc_gate_bwd.

None of these re-types the formula under test.  Each gradient is pinned by
what the mathematics fixes independently of its implementation:
  - adjoint identities against the (already pinned) forward oracle:
    <layout(x), g> == <x, layout_bwd(g)> and <reverse(back), dy> ==
    <back, d_back>, exact on small-integer data;
  - per-entry finite differences of the forward oracle (the combine is
    linear in each weight, so one unit step is exact on integer data);
  - central finite differences of Eq. 1's weights computed with
    scipy.special.softmax (a library routine) in float64;
  - closed forms: k=1 RENORM and k-top-1 RENORM weights are constants (zero
    gradient), softmax shift invariance (each softmax block's gradient sums to
    zero), dropped slots carry no gradient.
"""
import numpy as np
import pytest
from scipy.special import softmax

import synthgen


def _int_data(seed, shape, lo=-4, hi=5):
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi, size=shape).astype(np.float32)


def _routing(orc, S, E, k, C=1.0, kind="topk", mode="renorm", prio="token", skew=0.0, seed=5):
    lg = synthgen.logits(seed, S, E, k, kind, skew=skew)
    cap = orc.capacity(S, E, k, C)
    return lg, orc.gate(lg, E=E, k=k, cap=cap, kind=kind, weight_mode=mode, priority=prio)


# ------------------------------------------------------------ layout adjoint
@pytest.mark.parametrize("S,E,k,C", [(64, 4, 1, 1.0), (97, 8, 2, 0.6), (50, 6, 3, 0.5)])
def test_layout_bwd_is_the_adjoint(orc, S, E, k, C):
    """<layout(x), g> == <x, layout_bwd(g)> exactly (integers in fp32)."""
    _, r = _routing(orc, S, E, k, C, skew=1.0)
    d = 8
    x = _int_data(1, (S, d))
    g = _int_data(2, (E, r.cap, d))
    lhs = float((orc.layout(x, r).astype(np.float64) * g).sum())
    rhs = float((x.astype(np.float64) * orc.layout_bwd(g, r)).sum())
    assert lhs == rhs


def test_layout_bwd_one_hot(orc):
    """A unit gradient on slot (e, s) lands on exactly the token that filled
    it (slot_src), nowhere else; an empty slot's gradient is lost."""
    S, E, k, d = 40, 4, 2, 2
    _, r = _routing(orc, S, E, k, 0.5, skew=2.0)
    for e in range(E):
        for s in range(r.cap):
            g = np.zeros((E, r.cap, d), np.float32)
            g[e, s, 0] = 1.0
            dx = orc.layout_bwd(g, r)
            src = r.slot_src[e * r.cap + s]
            if src < 0:
                assert not dx.any()
            else:
                want = np.zeros((S, d), np.float32)
                want[src // k, 0] = 1.0
                assert (dx == want).all()


def test_layout_bwd_dropped_token_zero_bf16(orc):
    S, E, k, d = 200, 4, 2, 16
    _, r = _routing(orc, S, E, k, 0.3, skew=3.0)
    dead = (r.slot_idx < 0).all(1)
    assert dead.any()
    g = synthgen.tokens(3, E * r.cap, d, "bf16").reshape(E, r.cap, d)
    dx = orc.layout_bwd(g, r)
    assert dx.dtype == np.uint16 and (dx[dead] == 0).all()


# ------------------------------------------------------------ combine adjoint
@pytest.mark.parametrize("S,E,k,C,prio", [(80, 4, 1, 1.0, "token"), (120, 8, 2, 0.7, "token"),
                                          (90, 6, 3, 0.6, "slot")])
def test_reverse_bwd_d_back_is_the_adjoint(orc, S, E, k, C, prio):
    """<reverse(back), dy> == <back, d_back> for the fixed weights; d_back of
    every empty slot is zero."""
    _, r = _routing(orc, S, E, k, C, prio=prio, skew=1.0)
    d = 12
    back = _int_data(4, (E, r.cap, d))
    dy = _int_data(5, (S, d))
    d_back, _ = orc.reverse_layout_bwd(dy, back, r)
    y = orc.reverse_layout(back, r)
    lhs = float((y.astype(np.float64) * dy).sum())
    rhs = float((back.astype(np.float64) * d_back).sum())
    assert abs(lhs - rhs) <= 1e-5 * max(1.0, abs(lhs))
    empty = r.slot_src.reshape(E, r.cap) < 0
    assert (d_back[empty] == 0).all()


def test_reverse_bwd_d_weight_finite_difference(orc):
    """y is linear in each weight: raising w[t,j] by 1 changes <y, dy> by
    exactly d_weight[t,j] (integer data, exact in fp32).  Dropped slots: 0."""
    S, E, k, d = 30, 4, 2, 6
    _, r = _routing(orc, S, E, k, 0.6, skew=1.5)
    back = _int_data(6, (E, r.cap, d))
    dy = _int_data(7, (S, d))
    _, d_w = orc.reverse_layout_bwd(dy, back, r)
    import copy
    base = copy.copy(r)
    base.weight = np.ones_like(r.weight) * (r.slot_idx >= 0)
    f0 = float((orc.reverse_layout(back, base).astype(np.float64) * dy).sum())
    for t in range(S):
        for j in range(k):
            if r.slot_idx[t, j] < 0:
                assert d_w[t, j] == 0.0
                continue
            rr = copy.copy(base)
            rr.weight = base.weight.copy()
            rr.weight[t, j] += 1.0
            f1 = float((orc.reverse_layout(back, rr).astype(np.float64) * dy).sum())
            assert f1 - f0 == d_w[t, j]


def test_reverse_bwd_d_back_bf16_rounds_once(orc):
    """bf16: d_back = RNE(w * dy) with the product exact in double -- equal to
    torch's bf16 rounding of the exact float64 product."""
    import torch
    S, E, k, d = 64, 4, 2, 32
    _, r = _routing(orc, S, E, k, 1.0)
    dy = synthgen.tokens(8, S, d, "bf16")
    back = synthgen.tokens(9, E * r.cap, d, "bf16").reshape(E, r.cap, d)
    d_back, _ = orc.reverse_layout_bwd(dy, back, r)
    dyf = torch.from_numpy(dy.view(np.int16)).view(torch.bfloat16).double().numpy()
    for t in range(S):
        for j in range(k):
            s = r.slot_idx[t, j]
            if s < 0:
                continue
            prod = torch.from_numpy(np.float64(r.weight[t, j]) * dyf[t])  # exact
            want = prod.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
            assert (d_back[r.expert_idx[t, j], s] == want).all()


# ------------------------------------------------------------ gate adjoint
def _loss_weights(lg, r, kind, mode):
    """Eq. 1 weights of the FIXED selection as a function of the logits, via
    scipy.special.softmax in float64 (library routine), masked by capacity."""
    S, E = lg.shape
    k = r.k
    w = np.zeros((S, k))
    for t in range(S):
        sel = r.expert_idx[t]
        if kind == "topk" and mode == "renorm":
            w[t] = softmax(lg[t, sel])
        elif kind == "topk":
            w[t] = softmax(lg[t])[sel]
        elif mode == "softmax":
            n = E // k
            for j in range(k):
                w[t, j] = softmax(lg[t, j * n:(j + 1) * n])[sel[j] - j * n]
        else:
            w[t] = 1.0
    return w * (r.slot_idx >= 0)


@pytest.mark.parametrize("kind,mode,E,k,C", [
    ("topk", "renorm", 8, 2, 0.7), ("topk", "renorm", 16, 4, 1.0), ("topk", "softmax", 8, 2, 0.7),
    ("topk", "softmax", 32, 3, 1.0), ("ktop1", "softmax", 16, 2, 0.8), ("ktop1", "softmax", 12, 3, 1.0)])
def test_gate_bwd_central_difference(orc, kind, mode, E, k, C):
    S = 24
    lg, r = _routing(orc, S, E, k, C, kind=kind, mode=mode, skew=0.5, seed=11)
    g = np.random.default_rng(12).standard_normal((S, k)).astype(np.float32)
    dl = orc.gate_bwd(lg, r, g, kind=kind, weight_mode=mode)
    x = lg.astype(np.float64)
    h = 1e-6
    for t in range(S):
        for e in range(E):
            xp, xm = x.copy(), x.copy()
            xp[t, e] += h
            xm[t, e] -= h
            fd = ((_loss_weights(xp, r, kind, mode)[t] - _loss_weights(xm, r, kind, mode)[t])
                  * g[t]).sum() / (2 * h)
            assert abs(dl[t, e] - fd) <= 1e-7 + 1e-6 * abs(fd), (t, e, dl[t, e], fd)


def test_gate_bwd_constant_weights_have_zero_gradient(orc):
    """k=1 RENORM (w = softmax of one logit = 1) and k-top-1 RENORM (w = 1)."""
    S, E = 50, 8
    for kind, k in (("topk", 1), ("ktop1", 2)):
        lg, r = _routing(orc, S, E, k, 1.0, kind=kind)
        g = np.random.default_rng(13).standard_normal((S, k)).astype(np.float32)
        assert not orc.gate_bwd(lg, r, g, kind=kind, weight_mode="renorm").any()


def test_gate_bwd_shift_invariance_and_support(orc):
    """Softmax is shift invariant, so each softmax block's gradient sums to 0;
    RENORM top-k puts gradient on the k selected logits only; a token whose
    slots were all dropped gets no gradient."""
    S, E, k = 300, 8, 2
    lg, r = _routing(orc, S, E, k, 0.4, skew=2.0, seed=14)
    g = np.random.default_rng(15).standard_normal((S, k)).astype(np.float32)
    dl = orc.gate_bwd(lg, r, g).astype(np.float64)
    assert np.abs(dl.sum(1)).max() < 1e-6
    for t in range(S):
        off = np.setdiff1d(np.arange(E), r.expert_idx[t])
        assert not dl[t, off].any()
    dead = (r.slot_idx < 0).all(1)
    assert dead.any() and not dl[dead].any()
    dls = orc.gate_bwd(lg, r, g, weight_mode="softmax")  # routing reused: same selection
    assert np.abs(dls.astype(np.float64).sum(1)).max() < 1e-6


def test_gate_bwd_rejects_hash(orc):
    S, E = 10, 4
    ids, table = synthgen.hash_inputs(1, S, 64, E)
    r = orc.gate(None, E=E, k=1, cap=S, kind="hash", token_ids=ids, table=table)
    with pytest.raises(ValueError):
        orc.gate_bwd(np.zeros((S, E), np.float32), r, np.zeros((S, 1), np.float32), kind="hash")


# ------------------------------------------------------------ SAM / Dense-to-Sparse adjoints
def _sam_weights(gl, lg, r, G, mode):
    S, E = lg.shape
    n = E // G
    w = np.zeros((S, r.k))
    for t in range(S):
        sel = r.expert_idx[t]
        g = sel[0] // n
        if mode == "renorm":
            w[t] = softmax(lg[t, sel])
        else:
            w[t] = softmax(gl[t])[g] * softmax(lg[t, g * n:(g + 1) * n])[sel - g * n]
    return w * (r.slot_idx >= 0)


@pytest.mark.parametrize("mode,G,k", [("softmax", 4, 2), ("renorm", 4, 2), ("softmax", 2, 3)])
def test_sam_bwd_central_difference(orc, mode, G, k):
    S, E = 16, 16
    gl, lg = synthgen.group_logits_and_logits(51 + G, S, E, k, G)
    cap = orc.capacity(S, E, k, 0.9)
    r = orc.gate_sam(gl, lg, E=E, k=k, cap=cap, n_groups=G, weight_mode=mode)
    g = np.random.default_rng(52).standard_normal((S, k)).astype(np.float32)
    dl, dgl = orc.gate_bwd_ex(lg, r, g, kind="sam", weight_mode=mode, group_logits=gl,
                              n_groups=G)
    x, y = lg.astype(np.float64), gl.astype(np.float64)
    h = 1e-6
    for t in range(S):
        for e in range(E):
            xp, xm = x.copy(), x.copy()
            xp[t, e] += h
            xm[t, e] -= h
            fd = ((_sam_weights(y, xp, r, G, mode)[t] - _sam_weights(y, xm, r, G, mode)[t])
                  * g[t]).sum() / (2 * h)
            assert abs(dl[t, e] - fd) <= 1e-7 + 1e-6 * abs(fd), (t, e, dl[t, e], fd)
        for hh in range(G):
            yp, ym = y.copy(), y.copy()
            yp[t, hh] += h
            ym[t, hh] -= h
            fd = ((_sam_weights(yp, x, r, G, mode)[t] - _sam_weights(ym, x, r, G, mode)[t])
                  * g[t]).sum() / (2 * h)
            assert abs(dgl[t, hh] - fd) <= 1e-7 + 1e-6 * abs(fd), (t, hh, dgl[t, hh], fd)


def _d2s_weights(lg, u, r, tau, mode):
    S, E = lg.shape
    G = -np.log(-np.log(u.astype(np.float64)))
    z = (lg + G) / tau
    w = np.zeros((S, E))
    for t in range(S):
        live = r.expert_idx[t] >= 0
        sel = r.expert_idx[t, live]
        if mode == "renorm":
            w[t, :live.sum()] = softmax(z[t, sel])
        else:
            w[t, :live.sum()] = softmax(z[t])[sel]
    return w * (r.slot_idx >= 0)


@pytest.mark.parametrize("mode,tau", [("renorm", 0.7), ("softmax", 0.7), ("renorm", 2.0)])
def test_d2s_bwd_central_difference(orc, mode, tau):
    S, E = 16, 8
    lg = synthgen.logits(53, S, E)
    u = synthgen.uniforms_f32(54, S, E)
    cap = 9
    r = orc.gate_d2s(lg, cap=cap, tau=tau, eps=2e-2, uniforms=u, weight_mode=mode)
    assert (r.slot_idx < 0).any() and (r.expert_idx < 0).any()     # drops and prunes
    g = np.random.default_rng(55).standard_normal((S, E)).astype(np.float32)
    dl, dgl = orc.gate_bwd_ex(lg, r, g, kind="d2s", weight_mode=mode, uniforms=u, tau=tau)
    assert dgl is None
    x = lg.astype(np.float64)
    h = 1e-6
    for t in range(S):
        for e in range(E):
            xp, xm = x.copy(), x.copy()
            xp[t, e] += h
            xm[t, e] -= h
            fd = ((_d2s_weights(xp, u, r, tau, mode)[t] - _d2s_weights(xm, u, r, tau, mode)[t])
                  * g[t]).sum() / (2 * h)
            assert abs(dl[t, e] - fd) <= 1e-7 + 1e-6 * abs(fd), (t, e, dl[t, e], fd)
