"""CPU oracle of the HetuMoE (arXiv 2203.14685) token-routing path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2203_14685_b200`` never imports it, and
it imports nothing from the product package.

This module is argument marshalling (numpy <-> ctypes) around ``liboracle.so``,
a plain single-threaded C11 implementation compiled with
``-O2 -ffp-contract=off`` (see ``oracle/oracle.c`` for the arithmetic and its
PAPER.md citations).  The only logic written here in Python is the composition
of the C calls into Algorithm 1's six steps for P simulated
ranks (``route_multi``), which adds no arithmetic of its own.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

TOPK, KTOP1, HASH = 0, 1, 2
RENORM, SOFTMAX = 0, 1
PRIO_TOKEN, PRIO_SLOT = 0, 1
F32, BF16 = 0, 1

KINDS = {"topk": TOPK, "ktop1": KTOP1, "hash": HASH}
MODES = {"renorm": RENORM, "softmax": SOFTMAX}
PRIOS = {"token": PRIO_TOKEN, "slot": PRIO_SLOT}
DTYPES = {"f32": F32, "bf16": BF16}


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, C11, -O2 -ffp-contract=off, no fast-math)."""
    hdr = os.path.join(_HERE, "oracle.h")
    if (not force and os.path.exists(_SO)
            and os.path.getmtime(_SO) >= max(os.path.getmtime(_SRC), os.path.getmtime(hdr))):
        return _SO
    tmp = _SO + ".tmp%d" % os.getpid()
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math",
                           "-Wall", "-Wextra", "-fPIC", "-shared", _SRC, "-o", tmp, "-lm"])
    os.replace(tmp, _SO)
    return _SO


class _Stats(ctypes.Structure):
    _fields_ = [("intra_msgs", ctypes.c_int64), ("inter_msgs", ctypes.c_int64),
                ("inter_msg_bytes", ctypes.c_int64), ("intra_bytes", ctypes.c_int64),
                ("inter_bytes", ctypes.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        L.orc_capacity.argtypes = [i32, i32, i32, ctypes.c_double]
        L.orc_capacity.restype = i32
        L.orc_gate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, i32, i32, i32, i32,
                               P, P, P, i32, P, P, P, P, P]
        L.orc_gate.restype = i64
        L.orc_layout.argtypes = [i32, i32, i32, i32, i64, P, P, P, P]
        L.orc_layout.restype = None
        L.orc_reverse_layout.argtypes = [ctypes.c_int, i32, i32, i32, i32, i32, P, P, P, P, P]
        L.orc_reverse_layout.restype = None
        L.orc_expert_scale.argtypes = [ctypes.c_int, i32, i32, i32, i32, i32, P, P]
        L.orc_expert_scale.restype = None
        L.orc_alltoall_flat.argtypes = [i32, i64, ctypes.POINTER(P), ctypes.POINTER(P)]
        L.orc_alltoall_flat.restype = None
        L.orc_alltoall_hier.argtypes = [i32, i32, i64, ctypes.POINTER(P), ctypes.POINTER(P),
                                        ctypes.POINTER(_Stats)]
        L.orc_alltoall_hier.restype = ctypes.c_int
        L.orc_alltoall_flat_stats.argtypes = [i32, i32, i64, ctypes.POINTER(_Stats)]
        L.orc_alltoall_flat_stats.restype = None
        L.orc_gate_sam.argtypes = [ctypes.c_int, ctypes.c_int, i32, i32, i32, i32, i32, P, P,
                                   P, P, P, P, P]
        L.orc_gate_sam.restype = i64
        L.orc_gate_d2s.argtypes = [ctypes.c_int, ctypes.c_int, i32, i32, i32, ctypes.c_double,
                                   ctypes.c_double, P, P, P, P, P, P, P]
        L.orc_gate_d2s.restype = i64
        L.orc_expert_offsets.argtypes = [i32, i32, P, P]
        L.orc_expert_offsets.restype = None
        L.orc_layout_packed.argtypes = [i32, i32, i32, i64, P, P, P, P, P]
        L.orc_layout_packed.restype = None
        L.orc_reverse_layout_packed.argtypes = [ctypes.c_int, i32, i32, i32, i32, P, P, P, P, P,
                                                P]
        L.orc_reverse_layout_packed.restype = None
        L.orc_alltoallv.argtypes = [i32, i64, P, ctypes.POINTER(P), ctypes.POINTER(P)]
        L.orc_alltoallv.restype = None
        L.orc_reverse_layout_bwd.argtypes = [ctypes.c_int, i32, i32, i32, i32, i32, P, P, P,
                                             P, P, P, P]
        L.orc_reverse_layout_bwd.restype = None
        L.orc_layout_bwd.argtypes = [ctypes.c_int, i32, i32, i32, i32, i32, P, P, P, P]
        L.orc_layout_bwd.restype = None
        L.orc_gate_bwd.argtypes = [ctypes.c_int, ctypes.c_int, i32, i32, i32, P, P, P, P, P]
        L.orc_gate_bwd.restype = ctypes.c_int
        L.orc_gate_bwd_ex.argtypes = [ctypes.c_int, ctypes.c_int, i32, i32, i32, P, P, i32, P,
                                      ctypes.c_double, P, P, P, P, P]
        L.orc_gate_bwd_ex.restype = ctypes.c_int
        L.orc_bf16_to_f64.argtypes = [ctypes.c_uint16]
        L.orc_bf16_to_f64.restype = ctypes.c_double
        L.orc_f64_to_bf16.argtypes = [ctypes.c_double]
        L.orc_f64_to_bf16.restype = ctypes.c_uint16
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


def capacity(S, E, k, C) -> int:
    return int(lib().orc_capacity(S, E, k, float(C)))


@dataclass
class Routing:
    expert_idx: np.ndarray  # [S, k] int32
    slot_idx: np.ndarray    # [S, k] int32
    weight: np.ndarray      # [S, k] float32
    load: np.ndarray        # [E]    int32
    slot_src: np.ndarray    # [E*cap] int32
    S: int
    E: int
    k: int
    cap: int
    bad: int


def gate(logits=None, *, S=None, E, k, cap, kind="topk", weight_mode="renorm",
         priority="token", token_ids=None, table=None) -> Routing:
    kind_i = KINDS[kind]
    logits = _c(logits, np.float32)
    if logits is not None:
        S = logits.shape[0]
        assert logits.shape == (S, E)
    else:
        token_ids = _c(token_ids, np.int32)
        S = token_ids.shape[0]
    token_ids = _c(token_ids, np.int32)
    table = _c(table, np.int32)
    vocab = 0 if table is None else int(table.shape[0])
    ei = np.empty((S, k), np.int32)
    si = np.empty((S, k), np.int32)
    w = np.empty((S, k), np.float32)
    load = np.empty((E,), np.int32)
    ss = np.empty((E * cap,), np.int32)
    bad = lib().orc_gate(kind_i, MODES[weight_mode], PRIOS[priority], S, E, k, cap,
                         _ptr(logits), _ptr(token_ids), _ptr(table), vocab,
                         _ptr(ei), _ptr(si), _ptr(w), _ptr(load), _ptr(ss))
    if bad < 0:
        raise ValueError("orc_gate rejected its arguments")
    return Routing(ei, si, w, load, ss, S, E, k, cap, int(bad))


def gate_sam(group_logits, logits, *, E, k, cap, n_groups, weight_mode="renorm",
             priority="token") -> Routing:
    """Hierarchical top-k (SAM; R17)."""
    gl = _c(group_logits, np.float32)
    lg = _c(logits, np.float32)
    S = lg.shape[0]
    assert lg.shape == (S, E) and gl.shape == (S, n_groups)
    ei, si = np.empty((S, k), np.int32), np.empty((S, k), np.int32)
    w, load, ss = np.empty((S, k), np.float32), np.empty((E,), np.int32), np.empty((E * cap,), np.int32)
    rc = lib().orc_gate_sam(MODES[weight_mode], PRIOS[priority], S, E, k, cap, n_groups, _ptr(gl),
                            _ptr(lg), _ptr(ei), _ptr(si), _ptr(w), _ptr(load), _ptr(ss))
    if rc < 0:
        raise ValueError("orc_gate_sam rejected its arguments")
    return Routing(ei, si, w, load, ss, S, E, k, cap, 0)


def gate_d2s(logits, *, cap, tau, eps=1e-3, uniforms=None, weight_mode="renorm",
             priority="token") -> Routing:
    """Dense-to-Sparse (R18): k = E slots, pruned slots -1."""
    lg = _c(logits, np.float32)
    S, E = lg.shape
    u = _c(uniforms, np.float32)
    assert u is None or u.shape == (S, E)
    ei, si = np.empty((S, E), np.int32), np.empty((S, E), np.int32)
    w, load, ss = np.empty((S, E), np.float32), np.empty((E,), np.int32), np.empty((E * cap,), np.int32)
    rc = lib().orc_gate_d2s(MODES[weight_mode], PRIOS[priority], S, E, cap, float(tau), float(eps),
                            _ptr(lg), _ptr(u), _ptr(ei), _ptr(si), _ptr(w), _ptr(load), _ptr(ss))
    if rc < 0:
        raise ValueError("orc_gate_d2s rejected its arguments")
    return Routing(ei, si, w, load, ss, S, E, E, cap, 0)


def layout(x: np.ndarray, r: Routing) -> np.ndarray:
    """x: [S, d] of any element type -> dispatch [E, cap, d] of the same type."""
    x = np.ascontiguousarray(x)
    S, d = x.shape
    out = np.empty((r.E, r.cap, d), x.dtype)
    lib().orc_layout(S, r.E, r.k, r.cap, d * x.itemsize, _ptr(r.expert_idx), _ptr(r.slot_idx),
                     _ptr(x), _ptr(out))
    return out


def _dt(a):
    if a.dtype == np.float32:
        return F32
    if a.dtype == np.uint16:  # raw bf16 bits
        return BF16
    raise TypeError("oracle data must be float32 or uint16 (bf16 bits)")


def reverse_layout(back: np.ndarray, r: Routing) -> np.ndarray:
    back = np.ascontiguousarray(back)
    E, cap, d = back.shape
    assert E == r.E and cap == r.cap
    y = np.empty((r.S, d), back.dtype)
    lib().orc_reverse_layout(_dt(back), r.S, r.E, r.k, r.cap, d, _ptr(r.expert_idx),
                             _ptr(r.slot_idx), _ptr(r.weight), _ptr(back), _ptr(y))
    return y


def expert_scale(buf: np.ndarray, e_base: int) -> np.ndarray:
    """buf: [nsrc, E_local, cap, d] -> s_e * buf."""
    buf = np.ascontiguousarray(buf)
    nsrc, El, cap, d = buf.shape
    out = np.empty_like(buf)
    lib().orc_expert_scale(_dt(buf), nsrc, El, e_base, cap, d, _ptr(buf), _ptr(out))
    return out


def expert_offsets(r: Routing) -> np.ndarray:
    """SPEC's Permutation.expert_offsets [E+1] of the admitted slots."""
    out = np.empty((r.E + 1,), np.int32)
    lib().orc_expert_offsets(r.E, r.cap, _ptr(np.ascontiguousarray(r.load, np.int32)), _ptr(out))
    return out


def layout_packed(x: np.ndarray, r: Routing, offsets: np.ndarray) -> np.ndarray:
    """Dropless packed layout: [offsets[E], d] rows, expert-major."""
    x = np.ascontiguousarray(x)
    S, d = x.shape
    offsets = np.ascontiguousarray(offsets, np.int32)
    out = np.empty((int(offsets[-1]), d), x.dtype)
    lib().orc_layout_packed(S, r.E, r.k, d * x.itemsize, _ptr(r.expert_idx), _ptr(r.slot_idx),
                            _ptr(offsets), _ptr(x), _ptr(out))
    return out


def reverse_layout_packed(back: np.ndarray, r: Routing, offsets: np.ndarray) -> np.ndarray:
    back = np.ascontiguousarray(back)
    d = back.shape[-1]
    offsets = np.ascontiguousarray(offsets, np.int32)
    y = np.empty((r.S, d), back.dtype)
    lib().orc_reverse_layout_packed(_dt(back), r.S, r.E, r.k, d, _ptr(r.expert_idx),
                                    _ptr(r.slot_idx), _ptr(r.weight), _ptr(offsets), _ptr(back),
                                    _ptr(y))
    return y


def alltoallv(sends, counts):
    """sends[q]: [rows_q, ...] arrays of one row size; counts [P, P]: rows q
    sends to r.  Returns recv[r] (segments in ascending source rank)."""
    P = len(sends)
    sends = [np.ascontiguousarray(s) for s in sends]
    counts = np.ascontiguousarray(counts, np.int64)
    row_shape = sends[0].shape[1:]
    row_bytes = int(np.prod(row_shape, dtype=np.int64)) * sends[0].itemsize
    recvs = [np.empty((int(counts[:, r].sum()),) + row_shape, sends[0].dtype) for r in range(P)]
    lib().orc_alltoallv(P, row_bytes, _ptr(counts), _ptrs(sends), _ptrs(recvs))
    return recvs


def reverse_layout_bwd(dy: np.ndarray, back: np.ndarray, r: Routing):
    """Adjoint of the combine: (d_back [E,cap,d], d_weight [S,k] float32)."""
    dy = np.ascontiguousarray(dy)
    back = np.ascontiguousarray(back)
    E, cap, d = back.shape
    assert E == r.E and cap == r.cap and dy.shape == (r.S, d) and dy.dtype == back.dtype
    d_back = np.empty_like(back)
    d_w = np.empty((r.S, r.k), np.float32)
    lib().orc_reverse_layout_bwd(_dt(back), r.S, r.E, r.k, r.cap, d, _ptr(r.expert_idx),
                                 _ptr(r.slot_idx), _ptr(r.weight), _ptr(dy), _ptr(back),
                                 _ptr(d_back), _ptr(d_w))
    return d_back, d_w


def layout_bwd(d_dispatch: np.ndarray, r: Routing) -> np.ndarray:
    """Adjoint of Layout_Transform: [E,cap,d] -> dx [S,d]."""
    g = np.ascontiguousarray(d_dispatch)
    E, cap, d = g.shape
    assert E == r.E and cap == r.cap
    dx = np.empty((r.S, d), g.dtype)
    lib().orc_layout_bwd(_dt(g), r.S, r.E, r.k, r.cap, d, _ptr(r.expert_idx), _ptr(r.slot_idx),
                         _ptr(g), _ptr(dx))
    return dx


def gate_bwd(logits: np.ndarray, r: Routing, d_weight: np.ndarray, *, kind="topk",
             weight_mode="renorm") -> np.ndarray:
    """Adjoint of Eq. 1's weights w.r.t. the logits (selection fixed)."""
    logits = _c(logits, np.float32)
    d_weight = _c(d_weight, np.float32)
    S, E = logits.shape
    assert d_weight.shape == (S, r.k)
    out = np.empty((S, E), np.float32)
    rc = lib().orc_gate_bwd(KINDS[kind], MODES[weight_mode], S, E, r.k, _ptr(logits),
                            _ptr(r.expert_idx), _ptr(r.slot_idx), _ptr(d_weight), _ptr(out))
    if rc != 0:
        raise ValueError("orc_gate_bwd rejected its arguments")
    return out


def gate_bwd_ex(logits, r: Routing, d_weight, *, kind, weight_mode="renorm", group_logits=None,
                n_groups=1, uniforms=None, tau=1.0):
    """Adjoint of the SAM / Dense-to-Sparse weights (selection fixed).
    Returns (d_logits [S,E], d_group_logits [S,n_groups] or None)."""
    K = {"topk": TOPK, "ktop1": KTOP1, "hash": HASH, "sam": 3, "d2s": 4}[kind]
    lg = _c(logits, np.float32)
    S, E = lg.shape
    gl = _c(group_logits, np.float32)
    u = _c(uniforms, np.float32)
    dw = _c(d_weight, np.float32)
    out = np.empty((S, E), np.float32)
    dg = np.empty((S, n_groups), np.float32) if kind == "sam" else None
    rc = lib().orc_gate_bwd_ex(K, MODES[weight_mode], S, E, r.k, _ptr(lg), _ptr(gl), n_groups,
                               _ptr(u), float(tau), _ptr(r.expert_idx), _ptr(r.slot_idx),
                               _ptr(dw), _ptr(out), _ptr(dg))
    if rc != 0:
        raise ValueError("orc_gate_bwd_ex rejected its arguments")
    return out, dg


def _ptrs(bufs):
    arr = (ctypes.c_void_p * len(bufs))()
    for i, b in enumerate(bufs):
        arr[i] = b.ctypes.data
    return arr


def alltoall_flat(sends):
    P = len(sends)
    sends = [np.ascontiguousarray(s) for s in sends]
    nbytes = sends[0].nbytes
    assert all(s.nbytes == nbytes for s in sends) and nbytes % P == 0
    recvs = [np.empty_like(s) for s in sends]
    lib().orc_alltoall_flat(P, nbytes // P, _ptrs(sends), _ptrs(recvs))
    return recvs


def alltoall_hier(sends, G):
    P = len(sends)
    sends = [np.ascontiguousarray(s) for s in sends]
    nbytes = sends[0].nbytes
    assert all(s.nbytes == nbytes for s in sends) and nbytes % P == 0
    recvs = [np.empty_like(s) for s in sends]
    st = _Stats()
    rc = lib().orc_alltoall_hier(P, G, nbytes // P, _ptrs(sends), _ptrs(recvs), ctypes.byref(st))
    if rc != 0:
        raise ValueError("P % G != 0")
    return recvs, {f: getattr(st, f) for f, _ in _Stats._fields_}


def alltoall_flat_stats(P, G, bytes_per_peer):
    st = _Stats()
    lib().orc_alltoall_flat_stats(P, G, bytes_per_peer, ctypes.byref(st))
    return {f: getattr(st, f) for f, _ in _Stats._fields_}


def bf16_to_f64(h: int) -> float:
    return float(lib().orc_bf16_to_f64(h))


def f64_to_bf16(v: float) -> int:
    return int(lib().orc_f64_to_bf16(float(v)))


def route_multi(xs, logits_list, *, E, k, cap, kind="topk", weight_mode="renorm",
                priority="token", token_ids_list=None, table=None, algo="flat", G=None,
                scale=True):
    """Algorithm 1 for P simulated ranks, experts in contiguous
    blocks of E/P per rank (R10).  Returns (routings, dispatches, recvs, ys).

    Step 1 Gate -> 2 Layout_Transform -> 3 AllToAll -> 4 expert (fixed scale,
    R16; identity if scale=False) -> 5 AllToAll -> 6 Reverse_Layout_Transform.
    """
    P = len(xs)
    assert E % P == 0
    El = E // P
    routings, disp, ys = [], [], []
    for r in range(P):
        rt = gate(None if logits_list is None else logits_list[r], E=E, k=k, cap=cap, kind=kind,
                  weight_mode=weight_mode, priority=priority,
                  token_ids=None if token_ids_list is None else token_ids_list[r], table=table)
        routings.append(rt)
        disp.append(layout(xs[r], rt))
    a2a = alltoall_flat if algo == "flat" else (lambda s: alltoall_hier(s, G)[0])
    recvs = a2a(disp)  # recv_r: [P_src][El][cap][d] viewed as [E, cap, d]
    outs = []
    for r in range(P):
        rv = recvs[r].reshape(P, El, cap, -1)
        outs.append(expert_scale(rv, r * El).reshape(recvs[r].shape) if scale else recvs[r])
    backs = a2a(outs)
    for r in range(P):
        ys.append(reverse_layout(backs[r], routings[r]))
    return routings, disp, recvs, ys
