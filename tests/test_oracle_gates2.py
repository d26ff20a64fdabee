"""Pins of the oracle's remaining logit-only gates:
hierarchical top-k / SAM (orc_gate_sam, R17) and
Dense-to-Sparse (orc_gate_d2s, R18).

Pinned against: the degenerate cases SPEC.md:159-161 and 201-203 name
(one group == top-k; k == group size == the group's softmax; tau -> inf
== uniform; tau -> 0 == argmax), a two-stage brute-force selection in numpy,
scipy.special.softmax (library) for the weights, the Gumbel-max property
(the argmax of l + G is distributed as softmax(l): a statistical pin of the
noise formula), monotone sparsification in tau, and the shared
capacity invariants.
"""
import numpy as np
import pytest
from scipy.special import softmax

import synthgen


# ------------------------------------------------------------------ SAM
def test_sam_one_group_is_topk(orc):
    """num_groups = 1 -> identical to the top-k gate."""
    S, E, k = 500, 16, 2
    gl, lg = synthgen.group_logits_and_logits(1, S, E, k, 1)
    cap = orc.capacity(S, E, k, 0.8)
    for mode in ("renorm", "softmax"):
        a = orc.gate_sam(gl, lg, E=E, k=k, cap=cap, n_groups=1, weight_mode=mode)
        b = orc.gate(lg, E=E, k=k, cap=cap, weight_mode=mode)
        assert (a.expert_idx == b.expert_idx).all() and (a.slot_idx == b.slot_idx).all()
        assert (a.weight == b.weight).all() and (a.slot_src == b.slot_src).all()


@pytest.mark.parametrize("G,k", [(2, 2), (4, 1), (4, 3), (8, 2)])
def test_sam_two_stage_brute_force(orc, G, k):
    """every selected expert lies in the argmax group, and the
    selection is the stable top-k of that group's slice."""
    S, E = 400, 32
    n = E // G
    gl, lg = synthgen.group_logits_and_logits(2 + G, S, E, k, G)
    r = orc.gate_sam(gl, lg, E=E, k=k, cap=S * k, n_groups=G)
    g = np.argmax(gl, axis=1)                      # first maximum: lowest index
    for t in range(S):
        sl = lg[t, g[t] * n:(g[t] + 1) * n]
        want = g[t] * n + np.lexsort((np.arange(n), -sl))[:k]
        assert r.expert_idx[t].tolist() == want.tolist()


def test_sam_weights_against_scipy(orc):
    S, E, G, k = 300, 32, 4, 3
    n = E // G
    gl, lg = synthgen.group_logits_and_logits(9, S, E, k, G)
    rr = orc.gate_sam(gl, lg, E=E, k=k, cap=S * k, n_groups=G, weight_mode="renorm")
    rs = orc.gate_sam(gl, lg, E=E, k=k, cap=S * k, n_groups=G, weight_mode="softmax")
    assert (rr.expert_idx == rs.expert_idx).all()
    g = np.argmax(gl, axis=1)
    for t in range(S):
        sel = rr.expert_idx[t]
        want_r = softmax(lg[t, sel].astype(np.float64))
        pg = softmax(gl[t].astype(np.float64))[g[t]]
        want_s = pg * softmax(lg[t, g[t] * n:(g[t] + 1) * n].astype(np.float64))[sel - g[t] * n]
        assert np.allclose(rr.weight[t], want_r, rtol=2.4e-7, atol=0)
        assert np.allclose(rs.weight[t], want_s, rtol=2.4e-7, atol=0)
        assert rs.weight[t].sum() <= pg * (1 + 1e-6)


def test_sam_k_equals_group_size(orc):
    """k == group size -> within-group weights are the softmax of
    the group's logits (both modes agree up to the group probability)."""
    S, E, G = 200, 24, 3
    n = E // G
    gl, lg = synthgen.group_logits_and_logits(10, S, E, n, G)
    r = orc.gate_sam(gl, lg, E=E, k=n, cap=S * n, n_groups=G)
    g = np.argmax(gl, axis=1)
    for t in range(S):
        assert sorted(r.expert_idx[t].tolist()) == list(range(g[t] * n, (g[t] + 1) * n))
        sm = softmax(lg[t, g[t] * n:(g[t] + 1) * n].astype(np.float64))
        assert np.allclose(r.weight[t], sm[r.expert_idx[t] - g[t] * n], rtol=2.4e-7, atol=0)


def test_sam_capacity_invariants_and_rejects(orc):
    S, E, G, k = 1000, 16, 2, 2
    gl, lg = synthgen.group_logits_and_logits(11, S, E, k, G)
    gl[:, 0] += 1.0  # group 0 wins more often: drops
    cap = orc.capacity(S, E, k, 0.7)
    r = orc.gate_sam(gl, lg, E=E, k=k, cap=cap, n_groups=G, priority="slot")
    adm = np.bincount(r.expert_idx[r.slot_idx >= 0], minlength=E)
    assert (adm == np.minimum(r.load, cap)).all() and (adm <= cap).all()
    assert (r.weight[r.slot_idx < 0] == 0).all()
    with pytest.raises(ValueError):
        orc.gate_sam(gl, lg, E=E, k=9, cap=cap, n_groups=G)       # k > group size
    with pytest.raises(ValueError):
        orc.gate_sam(gl[:, :1].repeat(3, 1), lg, E=E, k=1, cap=cap, n_groups=3)  # 3 does not divide 16


# ------------------------------------------------------------------ Dense-to-Sparse
def test_d2s_high_temperature_is_uniform(orc):
    """tau = 1e6, eval -> weights ~ 1/E within 1e-3, all survive."""
    S, E = 100, 16
    lg = synthgen.logits(20, S, E)
    r = orc.gate_d2s(lg, cap=S * E, tau=1e6)
    assert (r.expert_idx >= 0).all()
    assert np.abs(r.weight - 1.0 / E).max() < 1e-3


def test_d2s_low_temperature_is_argmax(orc):
    """tau = 1e-3, eval, distinct logits -> one survivor, the
    argmax, weight 1."""
    S, E = 300, 32
    lg = synthgen.logits(21, S, E, gap=1e-2)
    r = orc.gate_d2s(lg, cap=S, tau=1e-3)
    assert (r.expert_idx[:, 0] == np.argmax(lg, axis=1)).all()
    assert (r.expert_idx[:, 1:] == -1).all() and (r.weight[:, 0] == 1.0).all()


def test_d2s_sparsifies_as_tau_decreases(orc):
    """mean survivor count non-increasing over tau 10, 1, 0.1, 0.01."""
    S, E = 2000, 32
    lg = synthgen.logits(22, S, E)
    u = synthgen.uniforms_f32(23, S, E)
    counts = []
    for tau in (10.0, 1.0, 0.1, 0.01):
        r = orc.gate_d2s(lg, cap=S * E, tau=tau, uniforms=u)
        counts.append((r.expert_idx >= 0).sum(1).mean())
    assert all(a >= b for a, b in zip(counts, counts[1:])), counts
    assert counts[0] > counts[-1]


def test_d2s_against_scipy_softmax(orc):
    """Survivor set {p >= eps}, order (z desc, index asc), renormalised and
    raw weights, with p = scipy.special.softmax((l + G)/tau) in float64."""
    S, E, tau, eps = 500, 16, 0.7, 1e-2
    lg = synthgen.logits(24, S, E)
    u = synthgen.uniforms_f32(25, S, E)
    G = -np.log(-np.log(u.astype(np.float64)))
    z = (lg.astype(np.float64) + G) / tau
    p = softmax(z, axis=1)
    rr = orc.gate_d2s(lg, cap=S * E, tau=tau, eps=eps, uniforms=u)
    rs = orc.gate_d2s(lg, cap=S * E, tau=tau, eps=eps, uniforms=u, weight_mode="softmax")
    for t in range(S):
        surv = np.nonzero(p[t] >= eps)[0]
        order = surv[np.lexsort((surv, -z[t, surv]))]
        ns = len(order)
        assert rr.expert_idx[t, :ns].tolist() == order.tolist()
        assert (rr.expert_idx[t, ns:] == -1).all() and (rr.weight[t, ns:] == 0).all()
        assert np.allclose(rr.weight[t, :ns], p[t, order] / p[t, surv].sum(), rtol=2.4e-7, atol=0)
        assert np.allclose(rs.weight[t, :ns], p[t, order], rtol=2.4e-7, atol=0)
    assert np.abs(rr.weight.sum(1) - 1).max() < 1e-6


def test_d2s_gumbel_max_property(orc):
    """The Gumbel-max trick: with tau = 1 the top slot (argmax of l + G) is
    distributed as softmax(l).  20000 tokens sharing one logit row: every
    expert's frequency within 4 sigma of its probability -- pins the sign and
    nesting of -log(-log u)."""
    S, E = 20000, 6
    row = np.array([0.5, -1.0, 1.5, 0.0, -0.3, 1.0], np.float32)
    lg = np.tile(row, (S, 1))
    u = synthgen.uniforms_f32(26, S, E)
    r = orc.gate_d2s(lg, cap=S * E, tau=1.0, eps=0.0, uniforms=u)
    freq = np.bincount(r.expert_idx[:, 0], minlength=E) / S
    p = softmax(row.astype(np.float64))
    assert (np.abs(freq - p) <= 4 * np.sqrt(p * (1 - p) / S)).all(), (freq, p)


def test_d2s_capacity_and_pruned_slots(orc):
    S, E = 800, 8
    lg = synthgen.logits(27, S, E, skew=1.0)
    u = synthgen.uniforms_f32(28, S, E)
    cap = 100
    for prio in ("token", "slot"):
        r = orc.gate_d2s(lg, cap=cap, tau=0.5, uniforms=u, priority=prio)
        live = r.expert_idx >= 0
        assert (r.slot_idx[~live] == -1).all()
        assert (r.load == np.bincount(r.expert_idx[live], minlength=E)).all()
        adm = np.bincount(r.expert_idx[r.slot_idx >= 0], minlength=E)
        assert (adm == np.minimum(r.load, cap)).all()
        # survivors are a prefix of the slots
        assert (np.diff(live.astype(int), axis=1) <= 0).all()
    with pytest.raises(ValueError):
        orc.gate_d2s(lg, cap=cap, tau=0.0)
