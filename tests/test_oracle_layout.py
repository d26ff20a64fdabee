"""Pins of the oracle's Layout_Transform, Reverse_Layout_Transform (weighted
combine), expert stand-in and bf16 rounding, against SPEC's worked example,
round-trip identities, multiset/linearity invariants and library routines
(torch bf16 conversion and multiply, numpy float32 multiply).

Oracle functions pinned here: orc_layout, orc_reverse_layout,
orc_expert_scale, orc_f64_to_bf16, orc_bf16_to_f64.
"""
import numpy as np
import pytest
import torch

import synthgen
from conftest import golden


def _x(S, d, dtype, seed=1):
    return synthgen.tokens(seed, S, d, dtype)


def test_hw1_layout_golden(orc):
    g = golden("hw1_layout.json")
    lg = np.array(g["logits"], np.float32)
    cap = orc.capacity(g["S"], g["E"], g["k"], g["C"])
    assert cap == g["cap"]
    r = orc.gate(lg, E=g["E"], k=g["k"], cap=cap)
    assert r.expert_idx.tolist() == g["expert_idx"]
    assert r.slot_idx.tolist() == g["slot_idx"]
    assert r.load.tolist() == g["load"]
    assert r.slot_src.tolist() == g["slot_src"]
    x = np.arange(g["S"] * 4, dtype=np.float32).reshape(g["S"], 4) + 1.0
    disp = orc.layout(x, r)
    for e in range(g["E"]):
        for s in range(cap):
            src = g["dispatch_rows"][e][s]
            want = np.zeros(4, np.float32) if src is None else x[src]
            assert (disp[e, s] == want).all()
    # SPEC's packed Permutation is the padded buffer with padding removed
    adm = np.minimum(r.load, cap)
    assert np.concatenate([[0], np.cumsum(adm)]).tolist() == g["packed_offsets"]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_round_trip_identity(orc, dtype):
    """SPEC.md:269 / acceptance #4: k=1, no drops, unit weights ->
    reverse(layout(x)) == x bitwise."""
    S, E, d = 300, 8, 40
    lg = synthgen.logits(21, S, E, 1)
    r = orc.gate(lg, E=E, k=1, cap=S)
    x = _x(S, d, dtype)
    y = orc.reverse_layout(orc.layout(x, r), r)
    assert y.dtype == x.dtype and (y.view(np.uint8) == x.view(np.uint8)).all()


def test_layout_multiset_and_padding(orc):
    """buffer rows are exactly the selected input rows
    (replicated per admitted slot); every other row is zero."""
    S, E, k, d = 200, 8, 2, 16
    lg = synthgen.logits(22, S, E, k, skew=1.0)
    cap = orc.capacity(S, E, k, 0.8)
    r = orc.gate(lg, E=E, k=k, cap=cap)
    x = _x(S, d, "f32", 3) + 100.0   # no zero rows in x
    disp = orc.layout(x, r)
    got = sorted(map(tuple, disp.reshape(-1, d)[np.abs(disp.reshape(-1, d)).sum(1) > 0]))
    tt = np.nonzero(r.slot_idx >= 0)[0]
    assert got == sorted(map(tuple, x[tt]))
    for e in range(E):
        assert (disp[e, min(r.load[e], cap):] == 0).all()


def test_dropped_tokens_give_zero_rows(orc):
    g = golden("hw2_capacity.json")
    lg = np.array(g["logits"], np.float32)
    r = orc.gate(lg, E=2, k=1, cap=g["cap"])
    x = _x(4, 8, "bf16", 4)
    y = orc.reverse_layout(orc.layout(x, r), r)
    for t in g["zero_rows"]:
        assert (y[t] == 0).all()
    for t in range(4):
        if t not in g["zero_rows"]:
            assert (y[t] == x[t]).all()


def test_combine_with_equal_rows_sums_weights(orc):
    """If every expert returns the same row v, y = (sum_j w_j) v; for RENORM
    top-k with no drops the weights sum to 1, so y == v up to
    one float rounding of the weights."""
    S, E, k, d = 128, 8, 3, 8
    lg = synthgen.logits(23, S, E, k)
    r = orc.gate(lg, E=E, k=k, cap=S * k)
    v = np.linspace(-3, 3, d).astype(np.float32)
    back = np.broadcast_to(v, (E, S * k, d)).copy()
    y = orc.reverse_layout(back, r)
    np.testing.assert_allclose(y, np.broadcast_to(v, (S, d)), rtol=3e-7, atol=1e-30)


def test_combine_linearity(orc):
    """doubling the expert outputs doubles y exactly (power of 2)."""
    S, E, k, d = 100, 4, 2, 12
    lg = synthgen.logits(24, S, E, k)
    r = orc.gate(lg, E=E, k=k, cap=50)
    back = _x(E * 50, d, "f32", 5).reshape(E, 50, d)
    y1 = orc.reverse_layout(back, r)
    y2 = orc.reverse_layout(back * np.float32(2.0), r)
    assert (y2 == 2 * y1).all()


def test_combine_single_expert_k2_matches_weighted_sum_closed_form(orc):
    """Two selected experts whose rows are constants a and b: y = w0 a + w1 b
    with w0 = expit(gap) -- evaluated in double and rounded once."""
    from scipy.special import expit
    lg = np.array([[0.5, -0.25]], np.float32)
    r = orc.gate(lg, E=2, k=2, cap=1)
    back = np.zeros((2, 1, 1), np.float32)
    back[0, 0, 0], back[1, 0, 0] = 3.0, -7.0
    y = orc.reverse_layout(back, r)
    w0 = np.float32(expit(0.75))
    w1 = np.float32(expit(-0.75))
    assert y[0, 0] == np.float32(np.float64(w0) * 3.0 + np.float64(w1) * -7.0)


# ---------------------------------------------------------------- bf16 rounding
def test_bf16_rne_vs_torch(orc):
    """For float32-representable values a single RNE to bf16 equals torch's
    float32 -> bfloat16 conversion (library routine)."""
    rng = np.random.default_rng(9)
    vals = np.concatenate([rng.standard_normal(3000) * 10.0 ** rng.integers(-40, 39, 3000),
                           np.array([0.0, -0.0, 1.0, -1.0, 3.3895e38, 1e-40, -1e-41, 2.0 ** -133])
                           ]).astype(np.float32)
    # exact halfway cases: 1 + 2^-8 * odd
    ties = (1.0 + (2 * np.arange(50) + 1) * 2.0 ** -8).astype(np.float32)
    vals = np.concatenate([vals, ties, -ties])
    want = torch.from_numpy(vals).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = np.array([orc.f64_to_bf16(float(v)) for v in vals], np.uint16)
    assert (got == want).all()
    back = np.array([orc.bf16_to_f64(int(h)) for h in want])
    assert (back == synthgen.bf16_bits_to_f32(want).astype(np.float64)).all()


def test_bf16_single_rounding_from_double(orc):
    """Straight from double, no double rounding through float:
    1 + 2^-8 + 2^-30 is above the tie, so it rounds UP to 1 + 2^-7 (0x3F81);
    going through float first would land exactly on the tie and round to even
    (0x3F80)."""
    assert orc.f64_to_bf16(1.0 + 2.0 ** -8) == 0x3F80           # tie -> even
    assert orc.f64_to_bf16(1.0 + 3 * 2.0 ** -8) == 0x3F82       # tie -> even (up)
    assert orc.f64_to_bf16(1.0 + 2.0 ** -8 + 2.0 ** -30) == 0x3F81
    assert orc.f64_to_bf16(-(1.0 + 2.0 ** -8 + 2.0 ** -30)) == 0xBF81
    assert orc.f64_to_bf16(3.5e38) == 0x7F80                      # overflow -> inf
    assert orc.f64_to_bf16(2.0 ** -134) == 0x0000                 # below half min subnormal
    assert orc.f64_to_bf16(1.5 * 2.0 ** -133) == 0x0002           # tie -> even
    assert orc.f64_to_bf16(2.0 ** -133 + 2.0 ** -140) == 0x0001


# ---------------------------------------------------------------- expert stand-in
def test_expert_scale_vs_torch(orc):
    """s_e = 1 + (e mod 8)/8 (R16).  bf16: the exact product rounded once ==
    torch bf16 multiply; f32: numpy float32 multiply (one rounding)."""
    nsrc, El, cap, d, e_base = 2, 5, 3, 16, 6
    xb = synthgen.tokens(12, nsrc * El * cap, d, "bf16").reshape(nsrc, El, cap, d)
    xf = synthgen.tokens(13, nsrc * El * cap, d, "f32").reshape(nsrc, El, cap, d)
    s = np.array([1.0 + ((e_base + le) % 8) / 8.0 for le in range(El)])
    yb = orc.expert_scale(xb, e_base)
    tb = torch.from_numpy(xb.view(np.int16)).view(torch.bfloat16)
    want = (tb * torch.tensor(s, dtype=torch.bfloat16).view(1, El, 1, 1))
    assert (yb == want.view(torch.int16).numpy().view(np.uint16)).all()
    yf = orc.expert_scale(xf, e_base)
    assert (yf == xf * s.astype(np.float32).reshape(1, El, 1, 1)).all()
