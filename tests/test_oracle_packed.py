"""Pins of the oracle's dropless packed layout and variable-size AllToAll
(SURVEY §8(f) NEXT-4): orc_expert_offsets, orc_layout_packed,
orc_reverse_layout_packed, orc_alltoallv.

Pinned against SPEC's hand trace (ids (1,0,1) -> rows token1,
token0, token2, offsets (0,1,3)), the stable-sort oracle SPEC.md:256 names
(numpy lexsort of (expert, token, slot) triples), the already pinned padded
layout / combine with the padding removed, and the flat AllToAll (uniform
counts) plus the round trip with transposed counts.
"""
import numpy as np
import pytest

import synthgen
from conftest import golden


def test_spec_hand_trace(orc):
    g = golden("hw1_layout.json")
    lg = np.array(g["logits"], np.float32)
    cap = orc.capacity(g["S"], g["E"], g["k"], g["C"])
    r = orc.gate(lg, E=g["E"], k=g["k"], cap=cap)
    off = orc.expert_offsets(r)
    assert off.tolist() == g["packed_offsets"]
    x = np.arange(g["S"] * 4, dtype=np.float32).reshape(g["S"], 4)
    packed = orc.layout_packed(x, r, off)
    assert (packed == x[[1, 0, 2]]).all()       # SPEC.md:255 row order


@pytest.mark.parametrize("S,E,k,C,prio", [(300, 8, 2, 0.7, "token"), (257, 5, 3, 0.5, "token"),
                                          (400, 16, 1, 1.0, "token"), (200, 4, 2, 0.6, "slot")])
def test_packed_is_the_stable_counting_sort(orc, S, E, k, C, prio):
    lg = synthgen.logits(31 + S, S, E, k, skew=1.0)
    cap = orc.capacity(S, E, k, C)
    r = orc.gate(lg, E=E, k=k, cap=cap, priority=prio)
    off = orc.expert_offsets(r)
    x = synthgen.tokens(32, S, 8, "f32")
    packed = orc.layout_packed(x, r, off)
    t, j = np.nonzero(r.slot_idx >= 0)
    e = r.expert_idx[t, j]
    # admission key: TOKEN = (t, j), SLOT = (j, t) -- SPEC.md:256 stable sort
    order = np.lexsort((j, t, e)) if prio == "token" else np.lexsort((t, j, e))
    assert (packed == x[t[order]]).all()
    assert off[-1] == len(t) and (np.diff(off) == np.bincount(e, minlength=E)).all()


def test_packed_equals_padded_without_padding(orc):
    S, E, k, d = 500, 8, 2, 16
    lg = synthgen.logits(33, S, E, k, skew=1.5)
    cap = orc.capacity(S, E, k, 0.8)
    r = orc.gate(lg, E=E, k=k, cap=cap)
    off = orc.expert_offsets(r)
    x = synthgen.tokens(34, S, d, "bf16")
    padded = orc.layout(x, r)
    packed = orc.layout_packed(x, r, off)
    keep = np.concatenate([padded[e, :off[e + 1] - off[e]] for e in range(E)])
    assert keep.tobytes() == packed.tobytes()
    # the packed combine on the same rows equals the padded combine, bitwise
    back = synthgen.tokens(35, E * cap, d, "bf16").reshape(E, cap, d)
    back_packed = np.concatenate([back[e, :off[e + 1] - off[e]] for e in range(E)])
    assert orc.reverse_layout_packed(back_packed, r, off).tobytes() == \
        orc.reverse_layout(back, r).tobytes()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_dropless_round_trip(orc, dtype):
    """cap >= every load (dropless): k=1 unit weights -> reverse(layout(x)) == x
    bitwise, with exactly S rows and no padding."""
    S, E = 999, 16
    lg = synthgen.logits(36, S, E, 1, skew=2.0)      # skewed: padded form would drop
    r = orc.gate(lg, E=E, k=1, cap=S)
    off = orc.expert_offsets(r)
    assert off[-1] == S
    x = synthgen.tokens(37, S, 24, dtype)
    y = orc.reverse_layout_packed(orc.layout_packed(x, r, off), r, off)
    assert y.tobytes() == x.tobytes()


def test_alltoallv_uniform_counts_is_flat(orc):
    P, n, d = 4, 5, 3
    sends = [synthgen.tokens(40 + q, P * n, d, "f32") for q in range(P)]
    counts = np.full((P, P), n)
    v = orc.alltoallv(sends, counts)
    f = orc.alltoall_flat([s.reshape(-1) for s in sends])
    assert all(a.tobytes() == b.tobytes() for a, b in zip(v, f))


def test_alltoallv_round_trip_and_conservation(orc):
    P, d = 4, 2
    rng = np.random.default_rng(41)
    counts = rng.integers(0, 6, size=(P, P))
    sends = [np.arange(counts[q].sum() * d, dtype=np.float32).reshape(-1, d) + 1000 * q
             for q in range(P)]
    recv = orc.alltoallv(sends, counts)
    assert sum(r.shape[0] for r in recv) == counts.sum()
    for r in range(P):                         # segment of q in recv[r] is q's block for r
        at = 0
        for q in range(P):
            frm = counts[q, :r].sum()
            assert (recv[r][at:at + counts[q, r]] == sends[q][frm:frm + counts[q, r]]).all()
            at += counts[q, r]
    back = orc.alltoallv(recv, counts.T)       # the combine direction
    assert all(a.tobytes() == b.tobytes() for a, b in zip(back, sends))
