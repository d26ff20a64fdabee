"""Pins of the oracle's gate (selection, weights, capacity) to things other
than itself: the paper's / SPEC's worked examples (tests/golden), closed forms,
brute force over all orderings, and library routines (numpy lexsort/argmax,
scipy softmax/expit).  None of these re-types the oracle's own code path.

Oracle functions pinned here: orc_capacity, orc_gate (TOPK, KTOP1, HASH;
RENORM, SOFTMAX; TOKEN, SLOT).
"""
import itertools
import math

import numpy as np
import pytest
from scipy.special import expit, softmax

from conftest import golden


# ---------------------------------------------------------------- capacity
@pytest.mark.parametrize("S,E,k,C,cap", [
    (4, 2, 1, 0.5, 1),        # SPEC.md:142 worked example
    (3, 2, 1, 1.0, 2),        # SPEC.md:255 (HW1)
    (4, 3, 2, 0.5, 2),        # HW3: ceil(4/3)
    (32768, 8, 2, 1.0, 8192),   # C2
    (32768, 64, 1, 1.0, 512),   # C3 at every P
    (65536, 32, 2, 1.0, 4096),  # C4a
    (65536, 32, 1, 1.25, 2560),  # C4b
    (1, 4, 1, 1.0, 1),        # ceil(0.25) = 1: no minimum needed
    (10, 3, 1, 1.0, 4),       # ceil(3.33)
    (9, 3, 1, 1.0, 3),        # exact division: no round-up
])
def test_capacity_closed_form(orc, S, E, k, C, cap):
    assert orc.capacity(S, E, k, C) == cap


def test_capacity_invalid(orc):
    assert orc.capacity(0, 2, 1, 1.0) == -1
    assert orc.capacity(4, 0, 1, 1.0) == -1
    assert orc.capacity(4, 2, 0, 1.0) == -1
    assert orc.capacity(4, 2, 1, 0.0) == -1


# ---------------------------------------------------------------- selection
@pytest.mark.parametrize("E", [1, 2, 3, 4, 5])
def test_topk_bruteforce_all_orderings(orc, E):
    """Every ordering of E distinct values, every k: the top-k are, by
    construction, the positions holding values E-1, E-2, ..."""
    perms = np.array(list(itertools.permutations(range(E))), np.float32)
    for k in range(1, E + 1):
        r = orc.gate(perms, E=E, k=k, cap=perms.shape[0] * k)
        want = np.stack([np.argsort(-p, kind="stable")[:k] for p in perms])
        # closed form without sorting: position of value E-1-j
        for j in range(k):
            assert (r.expert_idx[:, j] == np.argmax(perms == (E - 1 - j), axis=1)).all()
        assert (r.expert_idx == want).all()
        assert (r.slot_idx >= 0).all()  # cap large: nothing dropped


def test_topk_ties_golden(orc):
    g = golden("hw4_ties.json")
    for case in g["rows"]:
        row = np.array([case["row"]], np.float32)
        r = orc.gate(row, E=row.shape[1], k=case["k"], cap=8)
        assert r.expert_idx[0].tolist() == case["expert_idx"], case
    a = g["all_zero"]
    lg = np.zeros((a["S"], a["E"]), np.float32)
    cap = orc.capacity(a["S"], a["E"], a["k"], a["C"])
    assert cap == a["cap"]
    r = orc.gate(lg, E=a["E"], k=a["k"], cap=cap)
    assert (r.expert_idx == np.array([[0, 1]] * a["S"])).all()
    assert r.slot_idx.tolist() == a["slot_idx_token"]


@pytest.mark.parametrize("E,k", [(4, 1), (8, 2), (16, 4), (64, 2), (33, 3), (256, 8), (7, 7)])
def test_topk_vs_library_stable_sort(orc, E, k):
    """Random integer-valued logits (many ties) vs numpy's stable lexsort on
    (-value, index): SPEC.md:123 '... equals full-sort oracle with identical
    tie rule'."""
    rng = np.random.default_rng(E * 100 + k)
    lg = rng.integers(-3, 4, size=(500, E)).astype(np.float32)
    r = orc.gate(lg, E=E, k=k, cap=500 * k)
    for t in range(lg.shape[0]):
        order = np.lexsort((np.arange(E), -lg[t]))
        assert r.expert_idx[t].tolist() == order[:k].tolist()


# ---------------------------------------------------------------- weights
def test_weights_k1_renorm_exactly_one(orc):
    lg = np.random.default_rng(1).standard_normal((300, 8)).astype(np.float32)
    r = orc.gate(lg, E=8, k=1, cap=300)
    assert (r.weight == 1.0).all()   # Eq. 1 with K=1: softmax of one logit


def test_weights_k2_renorm_logistic(orc):
    """k=2 Eq. 1 weights are the logistic function of the logit gap
    (scipy.special.expit), i.e. GShard's g1/(g1+g2)."""
    lg = np.random.default_rng(2).standard_normal((400, 8)).astype(np.float32)
    r = orc.gate(lg, E=8, k=2, cap=800)
    l0 = lg[np.arange(400), r.expert_idx[:, 0]].astype(np.float64)
    l1 = lg[np.arange(400), r.expert_idx[:, 1]].astype(np.float64)
    np.testing.assert_allclose(r.weight[:, 0], expit(l0 - l1), rtol=1.2e-7, atol=0)
    np.testing.assert_allclose(r.weight[:, 1], expit(l1 - l0), rtol=1.2e-7, atol=0)
    np.testing.assert_allclose(r.weight.sum(1, dtype=np.float64), 1.0, rtol=0, atol=2.4e-7)


@pytest.mark.parametrize("mode", ["renorm", "softmax"])
def test_weights_k_equals_E_is_full_softmax(orc, mode):
    """k=E -> weights equal the full softmax (scipy)."""
    E = 6
    lg = (np.random.default_rng(3).standard_normal((200, E)) * 3).astype(np.float32)
    r = orc.gate(lg, E=E, k=E, cap=200 * E, weight_mode=mode)
    sm = softmax(lg.astype(np.float64), axis=1)
    want = np.take_along_axis(sm, r.expert_idx, axis=1)
    np.testing.assert_allclose(r.weight, want, rtol=1.2e-7, atol=0)


def test_weights_softmax_mode_is_full_row_probability(orc):
    E, k = 16, 2
    lg = np.random.default_rng(4).standard_normal((300, E)).astype(np.float32)
    r = orc.gate(lg, E=E, k=k, cap=600, weight_mode="softmax")
    sm = softmax(lg.astype(np.float64), axis=1)
    np.testing.assert_allclose(r.weight, np.take_along_axis(sm, r.expert_idx, 1),
                               rtol=1.2e-7, atol=0)
    assert (r.weight.sum(1) < 1.0).all()  # not renormalised (R1)


def test_weights_uniform_and_overflow_guard(orc):
    # uniform logits -> 1/k
    r = orc.gate(np.full((3, 8), 2.5, np.float32), E=8, k=4, cap=12)
    assert np.allclose(r.weight, 0.25, rtol=0, atol=0)
    # SPEC.md:56 overflow guard: [1000, 0] -> [1, ~0], finite
    r = orc.gate(np.array([[1000.0, 0.0]], np.float32), E=2, k=2, cap=2)
    assert r.weight[0, 0] == 1.0 and r.weight[0, 1] == 0.0
    r = orc.gate(np.array([[1000.0, 0.0]], np.float32), E=2, k=1, cap=2, weight_mode="softmax")
    assert r.weight[0, 0] == 1.0


def test_weights_shift_invariance(orc):
    """adding a constant to a row leaves the weights unchanged
    (integer-valued logits so the shift itself is exact)."""
    lg = np.random.default_rng(5).integers(-5, 6, size=(200, 8)).astype(np.float32)
    for mode in ("renorm", "softmax"):
        a = orc.gate(lg, E=8, k=3, cap=600, weight_mode=mode)
        b = orc.gate(lg + 64.0, E=8, k=3, cap=600, weight_mode=mode)
        assert (a.expert_idx == b.expert_idx).all()
        assert (a.weight == b.weight).all()


# ---------------------------------------------------------------- capacity replay
def test_hw2_golden(orc):
    g = golden("hw2_capacity.json")
    lg = np.array(g["logits"], np.float32)
    cap = orc.capacity(g["S"], g["E"], g["k"], g["C"])
    assert cap == g["cap"]
    r = orc.gate(lg, E=g["E"], k=g["k"], cap=cap)
    assert r.expert_idx.tolist() == g["expert_idx"]
    assert r.slot_idx.tolist() == g["slot_idx"]
    assert r.weight.tolist() == g["weight"]
    assert r.load.tolist() == g["load"]


@pytest.mark.parametrize("prio", ["token", "slot"])
def test_hw3_golden(orc, prio):
    g = golden("hw3_priority.json")
    lg = np.array(g["logits"], np.float32)
    cap = orc.capacity(g["S"], g["E"], g["k"], g["C"])
    assert cap == g["cap"]
    for mode, key in (("renorm", "w_renorm"), ("softmax", "w_softmax")):
        r = orc.gate(lg, E=g["E"], k=g["k"], cap=cap, weight_mode=mode, priority=prio)
        assert r.expert_idx.tolist() == g["expert_idx"]
        assert r.load.tolist() == g["load"]
        slots = g["slot_idx_token" if prio == "token" else "slot_idx_slot"]
        assert r.slot_idx.tolist() == slots
        want = np.array([g[key]] * g["S"], np.float32)
        want[np.array(slots) < 0] = 0.0
        np.testing.assert_allclose(r.weight, want, rtol=6e-8, atol=0)
        dropped_all = np.nonzero((r.slot_idx < 0).all(1))[0].tolist()
        assert dropped_all == g["fully_dropped_%s_priority" % prio]


def _slots_by_sorting(ei, S, k, E, cap, prio):
    """Independent formulation of the capacity rule: stable-sort the (expert,
    admission key) pairs with numpy lexsort; slot = rank inside the expert's
    group, dropped if >= cap (SPEC.md:256 'stable-sort oracle')."""
    t = np.repeat(np.arange(S), k)
    j = np.tile(np.arange(k), S)
    key = t * k + j if prio == "token" else j * S + t
    e = ei.reshape(-1)
    order = np.lexsort((key, e))
    rank = np.empty(S * k, np.int64)
    starts = np.searchsorted(e[order], np.arange(E))
    pos = np.arange(S * k) - starts[e[order]]
    rank[order] = pos
    slots = np.where(rank < cap, rank, -1)
    return slots.reshape(S, k)


@pytest.mark.parametrize("prio", ["token", "slot"])
@pytest.mark.parametrize("S,E,k,C,skew", [(257, 4, 1, 1.0, 0.0), (300, 8, 2, 1.0, 1.0),
                                          (129, 5, 3, 0.6, 0.5), (64, 64, 2, 1.0, 0.0),
                                          (1000, 16, 4, 0.3, 2.0)])
def test_capacity_replay_vs_sorting(orc, prio, S, E, k, C, skew):
    import synthgen
    lg = synthgen.logits(S * 7 + E, S, E, k, skew=skew)
    cap = orc.capacity(S, E, k, C)
    r = orc.gate(lg, E=E, k=k, cap=cap, priority=prio)
    assert (r.slot_idx == _slots_by_sorting(r.expert_idx, S, k, E, cap, prio)).all()
    # invariants (R6)
    load = np.bincount(r.expert_idx.reshape(-1), minlength=E)
    assert (r.load == load).all()
    admitted = np.bincount(r.expert_idx[r.slot_idx >= 0], minlength=E)
    assert (admitted == np.minimum(load, cap)).all()
    assert (admitted <= cap).all()
    big = orc.gate(lg, E=E, k=k, cap=S * k, priority=prio)   # no capacity pressure
    assert (big.expert_idx == r.expert_idx).all()             # ids never change
    keep = r.slot_idx >= 0
    assert (r.weight[keep] == big.weight[keep]).all()         # weights never grow
    assert (r.weight[~keep] == 0).all()
    # slot_src is the inverse map, -1 elsewhere
    ss = r.slot_src.reshape(E, cap)
    for e in range(E):
        filled = ss[e][ss[e] >= 0]
        assert len(filled) == admitted[e] and (ss[e][admitted[e]:] == -1).all()
        tt, jj = filled // k, filled % k
        assert (r.expert_idx[tt, jj] == e).all()
        assert (r.slot_idx[tt, jj] == np.arange(admitted[e])).all()


def test_k1_priorities_agree(orc):
    lg = np.random.default_rng(6).standard_normal((500, 8)).astype(np.float32)
    a = orc.gate(lg, E=8, k=1, cap=40, priority="token")
    b = orc.gate(lg, E=8, k=1, cap=40, priority="slot")
    assert (a.slot_idx == b.slot_idx).all()


# ---------------------------------------------------------------- k-top-1
def test_ktop1_one_prototype_is_top1(orc):
    """num_prototypes=1 -> identical to top-1."""
    lg = np.random.default_rng(7).standard_normal((300, 12)).astype(np.float32)
    a = orc.gate(lg, E=12, k=1, cap=30, kind="ktop1")
    b = orc.gate(lg, E=12, k=1, cap=30, kind="topk")
    for f in ("expert_idx", "slot_idx", "weight", "load", "slot_src"):
        assert (getattr(a, f) == getattr(b, f)).all()


def test_ktop1_E_prototypes(orc):
    """num_prototypes=E -> every prototype routes every token to
    its only expert (weight 1 under either mode)."""
    lg = np.random.default_rng(8).standard_normal((50, 6)).astype(np.float32)
    for mode in ("renorm", "softmax"):
        r = orc.gate(lg, E=6, k=6, cap=50, kind="ktop1", weight_mode=mode)
        assert (r.expert_idx == np.arange(6)).all() and (r.weight == 1.0).all()


@pytest.mark.parametrize("E,k", [(32, 2), (32, 4), (8, 2), (30, 3)])
def test_ktop1_slice_argmax_vs_numpy(orc, E, k):
    """each prototype's pick equals top-1 on its slice; numpy
    argmax returns the first (lowest-index) maximum; weights under SOFTMAX are
    the slice softmax (scipy) at the argmax."""
    rng = np.random.default_rng(E + k)
    lg = rng.integers(-4, 5, size=(400, E)).astype(np.float32)  # ties on purpose
    r = orc.gate(lg, E=E, k=k, cap=400, kind="ktop1", weight_mode="softmax")
    n = E // k
    for p in range(k):
        sl = lg[:, p * n:(p + 1) * n]
        assert (r.expert_idx[:, p] == p * n + np.argmax(sl, axis=1)).all()
        sm = softmax(sl.astype(np.float64), axis=1)
        np.testing.assert_allclose(r.weight[:, p], sm[np.arange(400), np.argmax(sl, 1)],
                                   rtol=1.2e-7, atol=0)
    r2 = orc.gate(lg, E=E, k=k, cap=400, kind="ktop1")
    assert (r2.weight == 1.0).all()   # summed prototypes, not averaged (R11)


# ---------------------------------------------------------------- hash
def test_hash_table_lookup_and_errors(orc):
    import synthgen
    ids, table = synthgen.hash_inputs(11, 4096, 1000, 8)
    r = orc.gate(None, E=8, k=1, cap=4096, kind="hash", token_ids=ids, table=table)
    assert (r.expert_idx[:, 0] == np.take(table, ids)).all() and r.bad == 0
    assert (r.weight == 1.0).all()
    # E=1 -> expert 0 regardless
    r = orc.gate(None, E=1, k=1, cap=4096, kind="hash", token_ids=ids,
                 table=np.zeros(1000, np.int32))
    assert (r.expert_idx == 0).all()
    # out-of-range ids and table entries are routed as dropped and counted (R12)
    bad_ids = ids.copy()
    bad_ids[[3, 10]] = [-1, 1000]
    bad_table = table.copy()
    bad_table[ids[20]] = 8
    r = orc.gate(None, E=8, k=1, cap=4096, kind="hash", token_ids=bad_ids, table=bad_table)
    bad_rows = np.nonzero(r.expert_idx[:, 0] < 0)[0]
    assert set([3, 10, 20]).issubset(set(bad_rows.tolist()))
    assert r.bad == len(bad_rows)
    assert (r.slot_idx[bad_rows] == -1).all() and (r.weight[bad_rows] == 0).all()
    # balanced table: each expert owns V/E ids exactly (V=1000 is not a
    # multiple of 8 -> counts differ by at most 1)
    cnt = np.bincount(table, minlength=8)
    assert cnt.max() - cnt.min() <= 1


def test_gate_rejects_bad_args(orc):
    lg = np.zeros((4, 6), np.float32)
    with pytest.raises(ValueError):
        orc.gate(lg, E=6, k=7, cap=4)           # k > E
    with pytest.raises(ValueError):
        orc.gate(lg, E=6, k=4, cap=4, kind="ktop1")  # E % k != 0
    with pytest.raises(ValueError):
        orc.gate(lg, E=6, k=1, cap=0)
