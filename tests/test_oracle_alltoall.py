"""Pins of the oracle's AllToAll simulations (flat and the paper's
hierarchical five-phase scheme) and of Algorithm 1 end to end.

Pinned against: HW5 (hand-worked P=2 exchange), table routing with numpy
indexing, the paper's message-size arithmetic (PAPER.md:180, 213 -> HW6),
SPEC's data-invariance and message-count invariants, and
end-to-end degeneracies.
"""
import numpy as np
import pytest

import synthgen
from conftest import golden


def test_hw5_golden(orc):
    g = golden("hw5_alltoall.json")
    sends = [np.array(s, np.int32) for s in g["send"]]
    recvs = orc.alltoall_flat(sends)
    assert [r.tolist() for r in recvs] == g["recv"]
    back = orc.alltoall_flat(recvs)   # the layout makes AllToAll self-inverse
    assert [b.tolist() for b in back] == g["send"]
    hier, _ = orc.alltoall_hier(sends, 1)
    assert [r.tolist() for r in hier] == g["recv"]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_flat_is_table_routing(orc, P):
    """chunk addressed (src->dst) arrives at dst in ascending src
    order.  Built with numpy fancy indexing of a [src, dst, chunk] array."""
    c = 5
    rng = np.random.default_rng(P)
    sends = [rng.integers(0, 255, P * c, dtype=np.uint8) for _ in range(P)]
    cube = np.stack([s.reshape(P, c) for s in sends])     # [src, dst, c]
    want = cube.transpose(1, 0, 2)                          # [dst, src, c]
    recvs = orc.alltoall_flat(sends)
    for r in range(P):
        assert (recvs[r].reshape(P, c) == want[r]).all()


@pytest.mark.parametrize("P,G", [(1, 1), (2, 1), (2, 2), (4, 2), (4, 4), (4, 1), (6, 2), (6, 3),
                                 (8, 4), (8, 2), (8, 8), (8, 1), (16, 4)])
def test_hierarchical_equals_flat_bytewise(orc, P, G):
    """SPEC.md:342 / acceptance #1: identical chunk contents in identical
    canonical order, plus conservation of bytes."""
    rng = np.random.default_rng(P * 10 + G)
    for c in (1, 3, 64):
        sends = [rng.integers(0, 255, P * c, dtype=np.uint8) for _ in range(P)]
        flat = orc.alltoall_flat(sends)
        hier, st = orc.alltoall_hier(sends, G)
        for a, b in zip(flat, hier):
            assert a.tobytes() == b.tobytes()
        N = P // G
        assert st["inter_msgs"] == N * (N - 1)
        assert st["inter_bytes"] == N * (N - 1) * G * G * c
        fs = orc.alltoall_flat_stats(P, G, c)
        assert fs["intra_msgs"] + fs["inter_msgs"] == P * P
        assert fs["inter_msgs"] == P * (P - G)             # N*G*(N-1)*G
        assert fs["inter_bytes"] == st["inter_bytes"]      # same cross-group payload
        if N > 1:
            assert st["inter_msg_bytes"] == G * G * fs["inter_msg_bytes"]  # G^2


def test_hw6_paper_message_sizes(orc):
    """N=8, G=8, B=16MB -> 256 KB per GPU pair flat,
    16 MB per node pair hierarchical, ratio G^2 = 64; our 4+4 mimic: 16."""
    g = golden("hw6_message_sizes.json")
    N, G, B = g["N"], g["G"], g["B_bytes"]
    P = N * G
    per_pair = B // P                       # each GPU's B split into P parts
    assert per_pair == g["flat_pair_bytes"]
    fs = orc.alltoall_flat_stats(P, G, per_pair)
    assert fs["inter_msg_bytes"] == g["flat_pair_bytes"]
    assert fs["inter_msgs"] == g["flat_cross_msgs"]
    # run the five-phase simulation on 4-byte chunks (memory), scale by bytes
    sends = [np.full(P, r, np.int32) for r in range(P)]
    hier, st = orc.alltoall_hier(sends, G)
    assert st["inter_msgs"] == g["hier_cross_msgs"]
    assert st["inter_msg_bytes"] // 4 * per_pair == g["hier_pair_bytes"]
    assert st["inter_msg_bytes"] // 4 == g["ratio"]
    m = g["mimic"]
    sends = [np.full(m["P"], r, np.int32) for r in range(m["P"])]
    _, st = orc.alltoall_hier(sends, m["G"])
    assert st["inter_msg_bytes"] // 4 == m["ratio"] and st["inter_msgs"] == m["hier_cross_msgs"]


# ---------------------------------------------------------------- end to end
def test_e2e_single_expert_is_scaled_identity(orc):
    """SPEC.md:401 / acceptance #10: E=1 top-1 -> y == e_0(x) = s_0 x = x."""
    S, d = 64, 24
    x = synthgen.tokens(31, S, d, "bf16")
    lg = np.zeros((S, 1), np.float32)
    _, _, _, ys = orc.route_multi([x], [lg], E=1, k=1, cap=S)
    assert (ys[0] == x).all()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_e2e_ktop1_one_prototype_equals_top1(orc, dtype):
    """SPEC.md:402."""
    S, E, d = 128, 8, 16
    x = synthgen.tokens(32, S, d, dtype)
    lg = synthgen.logits(33, S, E, 1)
    a = orc.route_multi([x], [lg], E=E, k=1, cap=20, kind="ktop1")[3][0]
    b = orc.route_multi([x], [lg], E=E, k=1, cap=20, kind="topk")[3][0]
    assert (a == b).all()


@pytest.mark.parametrize("P,G", [(2, 1), (4, 2), (8, 4), (8, 2)])
def test_e2e_collective_independence_and_transparency(orc, P, G):
    """y identical under flat and hierarchical.  AllToAll
    transparency: with pointwise experts, y on P ranks equals each rank's
    inputs run alone (P=1) with all E experts local."""
    S, E, k, d = 96, 16, 2, 8
    xs = [synthgen.tokens(40 + r, S, d, "bf16") for r in range(P)]
    lgs = [synthgen.logits(50 + r, S, E, k, skew=0.5) for r in range(P)]
    cap = orc.capacity(S, E, k, 1.0)
    _, disp, recvs, ys = orc.route_multi(xs, lgs, E=E, k=k, cap=cap)
    _, _, recvs_h, ys_h = orc.route_multi(xs, lgs, E=E, k=k, cap=cap, algo="hier", G=G)
    for a, b in zip(ys, ys_h):
        assert (a == b).all()
    for a, b in zip(recvs, recvs_h):
        assert (a == b).all()
    for r in range(P):
        y1 = orc.route_multi([xs[r]], [lgs[r]], E=E, k=k, cap=cap)[3][0]
        assert (y1 == ys[r]).all()
    # recv_r holds, from every source q, the rows rank q dispatched to r's experts
    El = E // P
    for r in range(P):
        rv = recvs[r].reshape(P, El, cap, d)
        for q in range(P):
            assert (rv[q] == disp[q][r * El:(r + 1) * El]).all()


def test_e2e_device_count_independence_without_drops(orc):
    """SPEC.md:407 (holds when nothing is dropped, capacity being per rank):
    splitting a batch over P ranks gives the same y rows as P=1."""
    S, E, k, d, P = 64, 8, 2, 8, 4
    x = synthgen.tokens(60, S * P, d, "f32")
    lg = synthgen.logits(61, S * P, E, k)
    y1 = orc.route_multi([x], [lg], E=E, k=k, cap=S * P * k)[3][0]
    ys = orc.route_multi([x[r * S:(r + 1) * S] for r in range(P)],
                         [lg[r * S:(r + 1) * S] for r in range(P)], E=E, k=k, cap=S * k)[3]
    assert (np.concatenate(ys) == y1).all()
