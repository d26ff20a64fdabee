"""Helpers shared by the -m gpu parity tests: numpy <-> torch CUDA transfer
and the comparison rules of DESIGN.md §3 (tolerances)."""
import numpy as np
import torch

# weights: 2 float ulp (both sides evaluate in fp64 and round once)
W_RTOL = 2.4e-7


def dev(a: np.ndarray, bf16: bool = False) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a))
    if bf16 or a.dtype == np.uint16:
        t = t.view(torch.int16).view(torch.bfloat16)
    return t.cuda()


def host(t: torch.Tensor) -> np.ndarray:
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def as_f64(a: np.ndarray) -> np.ndarray:
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def assert_routing_equal(rg, ro, what=""):
    """Bit-exact routing (ids, slots, drops, load, slot_src); weights within
    W_RTOL relative and exactly 0 where dropped."""
    ei, si = host(rg.expert_idx), host(rg.slot_idx)
    assert (ei == ro.expert_idx).all(), "%s expert_idx differs at %s" % (
        what, np.argwhere(ei != ro.expert_idx)[:5].tolist())
    assert (si == ro.slot_idx).all(), "%s slot_idx differs at %s" % (
        what, np.argwhere(si != ro.slot_idx)[:5].tolist())
    assert (host(rg.load) == ro.load).all(), what + " load"
    if rg.slot_src is not None:
        assert (host(rg.slot_src) == ro.slot_src).all(), what + " slot_src"
    w = host(rg.weight)
    err = np.abs(w.astype(np.float64) - ro.weight.astype(np.float64))
    tol = W_RTOL * np.abs(ro.weight.astype(np.float64))
    bad = err > tol
    assert not bad.any(), "%s weight: %d bad, worst rel %.3g" % (
        what, bad.sum(), (err / np.maximum(np.abs(ro.weight), 1e-30)).max())
    assert (w[ro.slot_idx < 0] == 0).all()


def combine_bound(back_f64, ro):
    """sum_j |w_j * a_j| per output element (the north_star's scale)."""
    S, k = ro.expert_idx.shape
    d = back_f64.shape[-1]
    acc = np.zeros((S, d))
    for j in range(k):
        ok = ro.slot_idx[:, j] >= 0
        rows = back_f64[ro.expert_idx[ok, j], ro.slot_idx[ok, j]]
        acc[ok] += np.abs(ro.weight[ok, j].astype(np.float64)[:, None] * rows)
    return acc


def assert_y_close(y_gpu: np.ndarray, y_orc: np.ndarray, bound: np.ndarray, bf16: bool, what=""):
    """north_star: 1e-6 relative (fp32) / 1e-2 relative (bf16) of sum |w a|."""
    rel = 1e-2 if bf16 else 1e-6
    err = np.abs(as_f64(y_gpu) - as_f64(y_orc))
    tol = rel * bound + 1e-30
    bad = err > tol
    assert not bad.any(), "%s y: %d elements out of tolerance (worst %.3g vs tol %.3g)" % (
        what, bad.sum(), err[bad].max(), tol[bad][np.argmax(err[bad])])
