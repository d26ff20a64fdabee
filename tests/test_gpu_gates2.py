"""GPU parity of the SAM (hierarchical top-k) and Dense-to-Sparse gates
 through moe_gate_ex, against orc_gate_sam /
orc_gate_d2s on the same seeded inputs: routing bit-exact, weights within 2
float ulp (both sides fp64, one rounding), then layout/reverse on the D2S
routing (pruned slots carry expert -1)."""
import numpy as np
import pytest
import torch
from scipy.special import softmax

import synthgen
from gpu_util import as_f64, assert_routing_equal, assert_y_close, combine_bound, dev, host

pytestmark = pytest.mark.gpu

import paper_2203_14685_b200 as moe  # noqa: E402

SAM_CASES = [
    dict(S=4096, E=64, G=8, k=2),
    dict(S=4096, E=64, G=1, k=2),                      # one group == top-k
    dict(S=3001, E=32, G=4, k=8),                      # k == group size
    dict(S=2049, E=256, G=32, k=4, mode="softmax"),
    dict(S=777, E=24, G=8, k=3, mode="softmax"),       # n = 3: L = 1, no vec4
    dict(S=1000, E=16, G=2, k=2, prio="slot", C=0.6, bias=1.0),
    dict(S=1, E=8, G=2, k=1),
    dict(S=5000, E=128, G=4, k=1, C=0.5, bias=2.0),
]


@pytest.mark.parametrize("c", SAM_CASES, ids=lambda c: "-".join("%s=%s" % kv for kv in c.items()))
def test_sam_parity(orc, c):
    S, E, G, k = c["S"], c["E"], c["G"], c["k"]
    mode, prio = c.get("mode", "renorm"), c.get("prio", "token")
    gl, lg = synthgen.group_logits_and_logits(S + E + G, S, E, k, G)
    if c.get("bias"):
        gl[:, 0] += np.float32(c["bias"])              # group 0 wins more: drops
    cap = orc.capacity(S, E, k, c.get("C", 1.0))
    ro = orc.gate_sam(gl, lg, E=E, k=k, cap=cap, n_groups=G, weight_mode=mode, priority=prio)
    g = moe.Gate(S, E, k, cap, "sam", mode, prio, n_groups=G)
    rg = g(dev(lg), group_logits=dev(gl))
    torch.cuda.synchronize()
    assert_routing_equal(rg, ro, str(c))


def _d2s_inputs_valid(lg, u, tau, eps):
    """The decisions both sides take in fp64 (p >= eps, the z order) must not
    sit within rounding distance of a boundary for these seeded inputs."""
    G = 0.0 if u is None else -np.log(-np.log(u.astype(np.float64)))
    z = (lg.astype(np.float64) + G) / tau
    p = softmax(z, axis=1)
    if eps > 0:
        assert (np.abs(p - eps) > 1e-9 * eps).all(), "inputs within 1e-9 of the prune threshold"
    zs = np.sort(z, axis=1)
    assert (np.diff(zs, axis=1) > 1e-12 * np.maximum(1.0, np.abs(zs[:, 1:]))).all(), "near-tie z"


D2S_CASES = [
    dict(S=4096, E=8, tau=1.0, train=True),
    dict(S=4096, E=16, tau=0.5, train=True, mode="softmax"),
    dict(S=2049, E=64, tau=2.0, train=True, eps=1e-2),
    dict(S=1024, E=256, tau=1.0, train=True),
    dict(S=3000, E=32, tau=0.1, train=False),
    dict(S=1500, E=8, tau=1e-3, train=False),          # single survivor
    dict(S=2000, E=24, tau=3.0, train=True, prio="slot", C=0.3),
    dict(S=777, E=12, tau=1e6, train=False),           # everyone survives
    dict(S=999, E=8, tau=0.7, train=True, C=0.2, bias=1.0),
]


@pytest.mark.parametrize("c", D2S_CASES, ids=lambda c: "-".join("%s=%s" % kv for kv in c.items()))
def test_d2s_parity(orc, c):
    S, E, tau, eps = c["S"], c["E"], c["tau"], c.get("eps", 1e-3)
    mode, prio = c.get("mode", "renorm"), c.get("prio", "token")
    lg = synthgen.logits(S * 5 + E, S, E, gap=1e-3, skew=c.get("bias", 0.0))
    u = synthgen.uniforms_f32(S * 7 + E, S, E) if c["train"] else None
    _d2s_inputs_valid(lg, u, tau, eps)
    cap = orc.capacity(S, E, E, c.get("C", 1.0) / E * 4)   # ~4 survivors/token at C=1
    ro = orc.gate_d2s(lg, cap=cap, tau=tau, eps=eps, uniforms=u, weight_mode=mode, priority=prio)
    g = moe.Gate(S, E, E, cap, "d2s", mode, prio, tau=tau, eps=eps)
    rg = g(dev(lg), uniforms=None if u is None else dev(u))
    torch.cuda.synchronize()
    assert_routing_equal(rg, ro, str(c))
    assert (host(rg.expert_idx)[ro.expert_idx < 0] == -1).all()


def test_d2s_layout_and_reverse(orc):
    """Layout / combine on a routing with pruned (-1) slots."""
    S, E, d, tau = 1500, 16, 256, 0.5
    lg = synthgen.logits(61, S, E, gap=1e-3)
    u = synthgen.uniforms_f32(62, S, E)
    _d2s_inputs_valid(lg, u, tau, 1e-3)
    cap = orc.capacity(S, E, E, 0.25)
    ro = orc.gate_d2s(lg, cap=cap, tau=tau, uniforms=u)
    rg = moe.Gate(S, E, E, cap, "d2s", tau=tau)(dev(lg), uniforms=dev(u))
    x = synthgen.tokens(63, S, d, "bf16")
    disp = moe.layout(dev(x), rg)
    torch.cuda.synchronize()
    assert host(disp).tobytes() == orc.layout(x, ro).tobytes()
    back = synthgen.tokens(64, E * cap, d, "bf16").reshape(E, cap, d)
    y = host(moe.reverse_layout(dev(back), rg))
    assert_y_close(y, orc.reverse_layout(back, ro), combine_bound(as_f64(back), ro), True)


def _bwd_close(got, ref, g, ro, scale=1.0):
    gs = np.abs(g.astype(np.float64) * (ro.slot_idx >= 0)).sum(1, keepdims=True)
    tol = 2.4e-7 * np.abs(ref.astype(np.float64)) + 1e-12 * scale * gs
    err = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    assert (err <= tol).all(), "%d bad, worst %.3g" % ((err > tol).sum(), (err - tol).max())


@pytest.mark.parametrize("mode", ["renorm", "softmax"])
@pytest.mark.parametrize("E,G,k", [(64, 8, 2), (24, 8, 3), (256, 32, 4)])
def test_sam_backward_parity(orc, mode, E, G, k):
    S = 2049
    gl, lg = synthgen.group_logits_and_logits(S + E + G + 1, S, E, k, G)
    cap = orc.capacity(S, E, k, 0.8)
    ro = orc.gate_sam(gl, lg, E=E, k=k, cap=cap, n_groups=G, weight_mode=mode)
    rg = moe.Gate(S, E, k, cap, "sam", mode, n_groups=G)(dev(lg), group_logits=dev(gl))
    torch.cuda.synchronize()
    assert_routing_equal(rg, ro)
    g = np.random.default_rng(S + E).standard_normal((S, k)).astype(np.float32)
    dl_o, dg_o = orc.gate_bwd_ex(lg, ro, g, kind="sam", weight_mode=mode, group_logits=gl,
                                 n_groups=G)
    dl, dg = moe.gate_backward(dev(lg), rg, dev(g), group_logits=dev(gl), n_groups=G)
    _bwd_close(host(dl), dl_o, g, ro)
    _bwd_close(host(dg), dg_o, g, ro)


@pytest.mark.parametrize("mode", ["renorm", "softmax"])
@pytest.mark.parametrize("E,tau,train", [(8, 0.7, True), (64, 2.0, True), (32, 0.5, False)])
def test_d2s_backward_parity(orc, mode, E, tau, train):
    S = 1500
    lg = synthgen.logits(S * 3 + E, S, E, gap=1e-3)
    u = synthgen.uniforms_f32(S * 5 + E, S, E) if train else None
    _d2s_inputs_valid(lg, u, tau, 1e-3)
    cap = orc.capacity(S, E, E, 0.3)
    ro = orc.gate_d2s(lg, cap=cap, tau=tau, uniforms=u, weight_mode=mode)
    rg = moe.Gate(S, E, E, cap, "d2s", mode, tau=tau)(dev(lg), uniforms=None if u is None else dev(u))
    torch.cuda.synchronize()
    assert_routing_equal(rg, ro)
    g = np.random.default_rng(S + E).standard_normal((S, E)).astype(np.float32)
    dl_o, _ = orc.gate_bwd_ex(lg, ro, g, kind="d2s", weight_mode=mode, uniforms=u, tau=tau)
    dl = moe.gate_backward(dev(lg), rg, dev(g), uniforms=None if u is None else dev(u), tau=tau)
    _bwd_close(host(dl), dl_o, g, ro, 1.0 / tau)
