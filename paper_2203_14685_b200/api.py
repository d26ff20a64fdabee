"""Python face of libmoe_b200: the four calls of Algorithm 1's routing path on
torch CUDA tensors and the current torch stream.

PyTorch is used for device memory, streams and torch.distributed bootstrap
only; these functions check dtype/contiguity/device/alignment, pass
``data_ptr()`` and the stream handle to the C ABI, and return tensors.  Every
byte of routing work is done by the library's kernels (or NCCL).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

import contextlib

from ._lib import A2AOp, GateDesc, GateInputs, RoutingC, Tuning, TUNING_FIELDS, check, lib

KINDS = {"topk": 0, "ktop1": 1, "hash": 2, "sam": 3, "d2s": 4}
MODES = {"renorm": 0, "softmax": 1}
PRIOS = {"token": 0, "slot": 1}
ALGOS = {"flat": 0, "hier": 1, "p2p": 2, "hier2d": 3}
_DT = {torch.float32: 0, torch.bfloat16: 1}


def _stream(device=None) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _p(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _need_cuda(t: torch.Tensor, name: str, dtype=None):
    if not t.is_cuda:
        raise ValueError("%s must be a CUDA tensor (no CPU fallback)" % name)
    if not t.is_contiguous():
        raise ValueError("%s must be contiguous" % name)
    if dtype is not None and t.dtype != dtype:
        raise TypeError("%s must be %s, got %s" % (name, dtype, t.dtype))


def capacity(S: int, E: int, k: int, C: float) -> int:
    """cap = ceil(C*S*k/E) (R4)."""
    c = lib().moe_capacity(S, E, k, float(C))
    if c < 0:
        raise ValueError("invalid capacity arguments S=%d E=%d k=%d C=%r" % (S, E, k, C))
    return c


@dataclass
class Routing:
    """W_(S,E), id_S of Algorithm 1, sparse: index t*k+j."""
    expert_idx: torch.Tensor   # [S, k] int32
    slot_idx: torch.Tensor     # [S, k] int32, -1 = dropped
    weight: torch.Tensor       # [S, k] float32
    load: torch.Tensor         # [E] int32
    slot_src: Optional[torch.Tensor]  # [E*cap] int32 or None
    S: int
    E: int
    k: int
    cap: int
    kind: int = 0
    weight_mode: int = 0
    priority: int = 0

    def desc(self) -> GateDesc:
        return GateDesc(self.S, self.E, self.k, self.cap, self.kind, self.weight_mode,
                        self.priority)

    def c(self) -> RoutingC:
        return RoutingC(self.expert_idx.data_ptr(), self.slot_idx.data_ptr(),
                        self.weight.data_ptr(), self.load.data_ptr(),
                        None if self.slot_src is None else self.slot_src.data_ptr())

    @staticmethod
    def empty(S, E, k, cap, device, kind=0, weight_mode=0, priority=0, slot_src=True):
        i32 = dict(dtype=torch.int32, device=device)
        return Routing(torch.empty((S, k), **i32), torch.empty((S, k), **i32),
                       torch.empty((S, k), dtype=torch.float32, device=device),
                       torch.empty((E,), **i32),
                       torch.empty((E * cap,), **i32) if slot_src else None,
                       S, E, k, cap, kind, weight_mode, priority)


class Gate:
    """moe_gate with its persistent (self-resetting) workspace."""

    def __init__(self, S: int, E: int, k: int, capacity: int, kind: str = "topk",
                 weight_mode: str = "renorm", priority: str = "token", device=None,
                 n_groups: int = 1, tau: float = 1.0, eps: float = 1e-3):
        """kind: topk | ktop1 | hash | sam (n_groups: the Switch Router's
        groups) | d2s (k must equal E; tau, eps: temperature and prune
        threshold -- the caller owns the schedule)."""
        self.S, self.E, self.k, self.cap = S, E, k, capacity
        self.n_groups, self.tau, self.eps = n_groups, tau, eps
        self.kind, self.mode, self.prio = KINDS[kind], MODES[weight_mode], PRIOS[priority]
        self.device = torch.device("cuda") if device is None else torch.device(device)
        d = GateDesc(S, E, k, capacity, self.kind, self.mode, self.prio)
        nb = lib().moe_gate_workspace_bytes(ctypes.byref(d))
        if nb == 0:
            # let moe_gate produce the precise error message
            check(lib().moe_gate(ctypes.byref(d), None, None, None, 0, None, None, 0, None),
                  "moe_gate")
        self.ws = torch.zeros(nb, dtype=torch.uint8, device=self.device)

    def __call__(self, logits: Optional[torch.Tensor] = None, token_ids=None, table=None,
                 out: Optional[Routing] = None, slot_src: bool = True,
                 group_logits: Optional[torch.Tensor] = None,
                 uniforms: Optional[torch.Tensor] = None) -> Routing:
        """uniforms (d2s, train mode): [S,E] float32 draws in (0,1) for the
        Gumbel noise; None = eval (no noise)."""
        if out is None:
            out = Routing.empty(self.S, self.E, self.k, self.cap, self.device, self.kind,
                                self.mode, self.prio, slot_src)
        vocab = 0
        if self.kind == KINDS["hash"]:
            _need_cuda(token_ids, "token_ids", torch.int32)
            _need_cuda(table, "table", torch.int32)
            vocab = table.numel()
        else:
            _need_cuda(logits, "logits", torch.float32)
            if tuple(logits.shape) != (self.S, self.E):
                raise ValueError("logits shape %s != (S=%d, E=%d)" % (tuple(logits.shape),
                                                                     self.S, self.E))
        if self.kind == KINDS["sam"]:
            _need_cuda(group_logits, "group_logits", torch.float32)
            if tuple(group_logits.shape) != (self.S, self.n_groups):
                raise ValueError("group_logits must be [S=%d, n_groups=%d]" % (self.S, self.n_groups))
        if uniforms is not None:
            _need_cuda(uniforms, "uniforms", torch.float32)
            if tuple(uniforms.shape) != (self.S, self.E):
                raise ValueError("uniforms must be [S=%d, E=%d]" % (self.S, self.E))
        out.kind, out.weight_mode, out.priority = self.kind, self.mode, self.prio
        d = GateDesc(self.S, self.E, self.k, self.cap, self.kind, self.mode, self.prio)
        inp = GateInputs(_p(logits), _p(token_ids), _p(table), vocab, _p(group_logits),
                         self.n_groups, _p(uniforms), float(self.tau), float(self.eps))
        rc = out.c()
        check(lib().moe_gate_ex(ctypes.byref(d), ctypes.byref(inp), ctypes.byref(rc), _p(self.ws),
                                self.ws.numel(), _stream(self.device)), "moe_gate")
        return out

    def _inputs(self, logits, token_ids, table, group_logits, uniforms):
        vocab = table.numel() if table is not None else 0
        return GateInputs(_p(logits), _p(token_ids), _p(table), vocab, _p(group_logits),
                          self.n_groups, _p(uniforms), float(self.tau), float(self.eps))

    def with_layout(self, x: torch.Tensor, dispatch: torch.Tensor, logits=None, token_ids=None,
                    table=None, out: Optional[Routing] = None, group_logits=None,
                    uniforms=None) -> Routing:
        """moe_gate_layout: the gate and Layout_Transform in one call, the
        gate's capacity pass fused into the layout kernel.  Same routing and
        dispatch as gate() then layout()."""
        if out is None:
            out = Routing.empty(self.S, self.E, self.k, self.cap, self.device, self.kind,
                                self.mode, self.prio)
        _need_cuda(x, "x")
        _need_cuda(dispatch, "dispatch", x.dtype)
        out.kind, out.weight_mode, out.priority = self.kind, self.mode, self.prio
        d = GateDesc(self.S, self.E, self.k, self.cap, self.kind, self.mode, self.prio)
        inp = self._inputs(logits, token_ids, table, group_logits, uniforms)
        rc = out.c()
        check(lib().moe_gate_layout(ctypes.byref(d), ctypes.byref(inp), ctypes.byref(rc),
                                    _p(self.ws), self.ws.numel(), _p(x), x.shape[-1],
                                    _DT[x.dtype], _p(dispatch), _stream(self.device)),
              "moe_gate_layout")
        return out

    def with_dispatch_p2p(self, comm: "Comm", x: torch.Tensor, recv: torch.Tensor, logits=None,
                          token_ids=None, table=None, out: Optional[Routing] = None,
                          group_logits=None, uniforms=None, flags: int = 0) -> Routing:
        """moe_gate_dispatch_p2p: gate + Layout_Transform + the NVLink dispatch
        in one call (capacity pass fused into the dispatch kernel)."""
        if out is None:
            out = Routing.empty(self.S, self.E, self.k, self.cap, self.device, self.kind,
                                self.mode, self.prio)
        out.kind, out.weight_mode, out.priority = self.kind, self.mode, self.prio
        d = GateDesc(self.S, self.E, self.k, self.cap, self.kind, self.mode, self.prio)
        inp = self._inputs(logits, token_ids, table, group_logits, uniforms)
        rc = out.c()
        check(lib().moe_gate_dispatch_p2p(comm._h, ctypes.byref(d), ctypes.byref(inp),
                                          ctypes.byref(rc), _p(self.ws), self.ws.numel(), _p(x),
                                          x.shape[-1], _DT[x.dtype], _p(recv), flags,
                                          _stream(self.device)), "moe_gate_dispatch_p2p")
        return out

    def check(self) -> int:
        """Invalid hash ids since the last check (synchronises the stream)."""
        n = ctypes.c_int32(0)
        check(lib().moe_gate_check(_p(self.ws), _stream(self.device), ctypes.byref(n)),
              "moe_gate_check")
        return n.value


def gate(logits: Optional[torch.Tensor] = None, *, E: Optional[int] = None, k: int = 1,
         capacity_factor: float = 1.0, capacity_: Optional[int] = None, kind: str = "topk",
         weight_mode: str = "renorm", priority: str = "token", token_ids=None, table=None,
         slot_src: bool = True) -> Routing:
    """One-shot convenience wrapper around Gate (allocates a workspace)."""
    if logits is not None:
        S, E = logits.shape
        dev = logits.device
    else:
        S = token_ids.numel()
        dev = token_ids.device
    cap = capacity_ if capacity_ is not None else capacity(S, E, k, capacity_factor)
    g = Gate(S, E, k, cap, kind, weight_mode, priority, dev)
    return g(logits, token_ids, table, slot_src=slot_src)


def layout(x: torch.Tensor, r: Routing, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Layout_Transform (Alg. 1 step 2): [S,d] -> padded [E,cap,d]."""
    _need_cuda(x, "x")
    if x.dtype not in _DT:
        raise TypeError("x must be float32 or bfloat16")
    S, d = x.shape
    if S != r.S:
        raise ValueError("x has %d rows, routing has S=%d" % (S, r.S))
    if out is None:
        out = torch.empty((r.E, r.cap, d), dtype=x.dtype, device=x.device)
    _need_cuda(out, "dispatch", x.dtype)
    desc, rc = r.desc(), r.c()
    check(lib().moe_layout(ctypes.byref(desc), ctypes.byref(rc), _p(x), d, _DT[x.dtype], _p(out),
                           _stream(x.device)), "moe_layout")
    return out


def reverse_layout(back: torch.Tensor, r: Routing,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Reverse_Layout_Transform + weighted combine (Alg. 1 steps 4/6)."""
    _need_cuda(back, "back")
    if back.dtype not in _DT:
        raise TypeError("back must be float32 or bfloat16")
    d = back.shape[-1]
    if back.numel() != r.E * r.cap * d:
        raise ValueError("back must hold [E=%d, cap=%d, d] rows" % (r.E, r.cap))
    if out is None:
        out = torch.empty((r.S, d), dtype=back.dtype, device=back.device)
    _need_cuda(out, "y", back.dtype)
    desc, rc = r.desc(), r.c()
    check(lib().moe_reverse_layout(ctypes.byref(desc), ctypes.byref(rc), _p(back), d,
                                   _DT[back.dtype], _p(out), _stream(back.device)),
          "moe_reverse_layout")
    return out


def expert_offsets(r: Routing, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """[E+1] int32: offsets[e] = sum_{e'<e} min(load[e'], cap) (NEXT-4,
    SPEC's Permutation.expert_offsets), computed on the device."""
    if out is None:
        out = torch.empty((r.E + 1,), dtype=torch.int32, device=r.load.device)
    _need_cuda(out, "offsets", torch.int32)
    desc, rc = r.desc(), r.c()
    check(lib().moe_expert_offsets(ctypes.byref(desc), ctypes.byref(rc), _p(out),
                                   _stream(out.device)), "moe_expert_offsets")
    return out


def layout_packed(x: torch.Tensor, r: Routing, offsets: torch.Tensor,
                  out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Dropless Layout_Transform: admitted rows expert-major, no padding.
    `out` defaults to the worst case [S*k, d] (rows >= offsets[E] unused)."""
    _need_cuda(x, "x")
    _need_cuda(offsets, "offsets", torch.int32)
    S, d = x.shape
    if out is None:
        out = torch.empty((r.S * r.k, d), dtype=x.dtype, device=x.device)
    desc, rc = r.desc(), r.c()
    check(lib().moe_layout_packed(ctypes.byref(desc), ctypes.byref(rc), _p(offsets), _p(x), d,
                                  _DT[x.dtype], _p(out), _stream(x.device)), "moe_layout_packed")
    return out


def reverse_layout_packed(back: torch.Tensor, r: Routing, offsets: torch.Tensor,
                          out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Dropless weighted Reverse_Layout_Transform from the packed rows."""
    _need_cuda(back, "back")
    _need_cuda(offsets, "offsets", torch.int32)
    d = back.shape[-1]
    if out is None:
        out = torch.empty((r.S, d), dtype=back.dtype, device=back.device)
    desc, rc = r.desc(), r.c()
    check(lib().moe_reverse_layout_packed(ctypes.byref(desc), ctypes.byref(rc), _p(offsets),
                                          _p(back), d, _DT[back.dtype], _p(out),
                                          _stream(back.device)), "moe_reverse_layout_packed")
    return out


def reverse_layout_packed_backward(dy: torch.Tensor, back: torch.Tensor, r: Routing,
                                   offsets: torch.Tensor, d_back: Optional[torch.Tensor] = None,
                                   d_weight: Optional[torch.Tensor] = None):
    """Adjoint of the packed combine: d_back rows at offsets[e] + s."""
    _need_cuda(dy, "dy")
    _need_cuda(offsets, "offsets", torch.int32)
    d = dy.shape[-1]
    if d_back is None:
        d_back = torch.empty((r.S * r.k, d), dtype=dy.dtype, device=dy.device)
    if d_weight is None:
        d_weight = torch.empty((r.S, r.k), dtype=torch.float32, device=dy.device)
    desc, rc = r.desc(), r.c()
    check(lib().moe_reverse_layout_packed_backward(ctypes.byref(desc), ctypes.byref(rc),
                                                   _p(offsets), _p(dy), _p(back), d,
                                                   _DT[dy.dtype], _p(d_back), _p(d_weight),
                                                   _stream(dy.device)),
          "moe_reverse_layout_packed_backward")
    return d_back, d_weight


def layout_packed_backward(d_packed: torch.Tensor, r: Routing, offsets: torch.Tensor,
                           out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Adjoint of the packed Layout_Transform: dx[t] = sum_j d_packed[offsets[e_j] + s_j]."""
    _need_cuda(d_packed, "d_packed")
    _need_cuda(offsets, "offsets", torch.int32)
    d = d_packed.shape[-1]
    if out is None:
        out = torch.empty((r.S, d), dtype=d_packed.dtype, device=d_packed.device)
    desc, rc = r.desc(), r.c()
    check(lib().moe_layout_packed_backward(ctypes.byref(desc), ctypes.byref(rc), _p(offsets),
                                           _p(d_packed), d, _DT[d_packed.dtype], _p(out),
                                           _stream(d_packed.device)), "moe_layout_packed_backward")
    return out


def alltoallv_plan(offsets, recv_counts, nranks: int):
    """Host plan of the NCCL dropless exchange (NEXT-4, moe_alltoallv_plan):
    from this rank's expert offsets [E+1] (moe_expert_offsets) and the
    per-expert counts it receives, recv_counts[src*E/P + le] (an AllToAll of
    the count table), return (send_rows[P], recv_rows[P], recv_offsets[E+1])
    for moe_alltoallv (R10, R20)."""
    off = [int(v) for v in offsets]
    rc = [int(v) for v in recv_counts]
    E = len(off) - 1
    if len(rc) != E:
        raise ValueError("need E recv counts (E=%d, got %d)" % (E, len(rc)))
    i32a, i64a = ctypes.c_int32 * (E + 1), ctypes.c_int64 * max(1, nranks)
    o, c = i32a(*off), (ctypes.c_int32 * max(1, E))(*rc)
    sr, rr, ro = i64a(), i64a(), i32a()
    check(lib().moe_alltoallv_plan(nranks, E, o, c, sr, rr, ro), "moe_alltoallv_plan")
    return list(sr)[:nranks], list(rr)[:nranks], list(ro)


def reverse_layout_backward(dy: torch.Tensor, back: torch.Tensor, r: Routing,
                            d_back: Optional[torch.Tensor] = None,
                            d_weight: Optional[torch.Tensor] = None):
    """Adjoint of the combine (NEXT-1): d_back [E,cap,d] = w * dy scattered to
    the slots (padding rows 0), d_weight [S,k] = <dy[t], back[e][s]>."""
    _need_cuda(dy, "dy")
    _need_cuda(back, "back", dy.dtype)
    if dy.dtype not in _DT:
        raise TypeError("dy must be float32 or bfloat16")
    S, d = dy.shape
    if S != r.S or back.numel() != r.E * r.cap * d:
        raise ValueError("dy must be [S=%d, d], back [E=%d, cap=%d, d]" % (r.S, r.E, r.cap))
    if d_back is None:
        d_back = torch.empty((r.E, r.cap, d), dtype=dy.dtype, device=dy.device)
    if d_weight is None:
        d_weight = torch.empty((r.S, r.k), dtype=torch.float32, device=dy.device)
    _need_cuda(d_back, "d_back", dy.dtype)
    _need_cuda(d_weight, "d_weight", torch.float32)
    desc, rc = r.desc(), r.c()
    check(lib().moe_reverse_layout_backward(ctypes.byref(desc), ctypes.byref(rc), _p(dy), _p(back),
                                            d, _DT[dy.dtype], _p(d_back), _p(d_weight),
                                            _stream(dy.device)), "moe_reverse_layout_backward")
    return d_back, d_weight


def layout_backward(d_dispatch: torch.Tensor, r: Routing,
                    out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Adjoint of Layout_Transform (NEXT-1): dx[t] = sum_j d_dispatch[e_j][s_j]."""
    _need_cuda(d_dispatch, "d_dispatch")
    if d_dispatch.dtype not in _DT:
        raise TypeError("d_dispatch must be float32 or bfloat16")
    d = d_dispatch.shape[-1]
    if d_dispatch.numel() != r.E * r.cap * d:
        raise ValueError("d_dispatch must hold [E=%d, cap=%d, d] rows" % (r.E, r.cap))
    if out is None:
        out = torch.empty((r.S, d), dtype=d_dispatch.dtype, device=d_dispatch.device)
    _need_cuda(out, "dx", d_dispatch.dtype)
    desc, rc = r.desc(), r.c()
    check(lib().moe_layout_backward(ctypes.byref(desc), ctypes.byref(rc), _p(d_dispatch), d,
                                    _DT[d_dispatch.dtype], _p(out), _stream(d_dispatch.device)),
          "moe_layout_backward")
    return out


def gate_backward(logits: torch.Tensor, r: Routing, d_weight: torch.Tensor,
                  out: Optional[torch.Tensor] = None, *, group_logits=None, n_groups: int = 1,
                  d_group_logits=None, uniforms=None, tau: float = 1.0):
    """Adjoint of the gate weights w.r.t. the logits (NEXT-1), selection
    fixed.  SAM: also returns d_group_logits (pass group_logits, n_groups);
    D2S: pass the same uniforms and tau as the forward."""
    _need_cuda(logits, "logits", torch.float32)
    _need_cuda(d_weight, "d_weight", torch.float32)
    if tuple(logits.shape) != (r.S, r.E) or d_weight.numel() != r.S * r.k:
        raise ValueError("logits must be [S=%d, E=%d], d_weight [S, k=%d]" % (r.S, r.E, r.k))
    if out is None:
        out = torch.empty_like(logits)
    _need_cuda(out, "d_logits", torch.float32)
    sam = r.kind == KINDS["sam"]
    if sam and d_group_logits is None:
        d_group_logits = torch.empty((r.S, n_groups), dtype=torch.float32, device=logits.device)
    desc, rc = r.desc(), r.c()
    inp = GateInputs(_p(logits), None, None, 0, _p(group_logits), n_groups, _p(uniforms),
                     float(tau), 0.0)
    check(lib().moe_gate_backward_ex(ctypes.byref(desc), ctypes.byref(inp), ctypes.byref(rc),
                                     _p(d_weight), _p(out), _p(d_group_logits),
                                     _stream(logits.device)), "moe_gate_backward")
    return (out, d_group_logits) if sam else out


def expert_scale(buf: torch.Tensor, nsrc: int, E_local: int, e_base: int,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Bench stand-in expert (R16): s_e * buf over [nsrc][E_local][cap][d]."""
    _need_cuda(buf, "buf")
    d = buf.shape[-1]
    cap = buf.numel() // (nsrc * E_local * d)
    if out is None:
        out = buf
    check(lib().moe_expert_scale(_p(buf), _p(out), nsrc, E_local, e_base, cap, d,
                                 _DT[buf.dtype], _stream(buf.device)), "moe_expert_scale")
    return out


def alltoall_plan(nranks: int, rank: int, algo: str = "flat", group_size: int = 1):
    """The schedule moe_alltoall executes on `rank` (host only)."""
    n = ctypes.c_int32(0)
    L = lib()
    L.moe_alltoall_plan(nranks, rank, ALGOS[algo], group_size, None, 0, ctypes.byref(n))
    ops = (A2AOp * max(1, n.value))()
    check(L.moe_alltoall_plan(nranks, rank, ALGOS[algo], group_size, ops, n.value,
                              ctypes.byref(n)), "moe_alltoall_plan")
    return [{f: getattr(o, f) for f, _ in A2AOp._fields_} for o in ops[:n.value]]


class Comm:
    """The library-owned NCCL communicator (moe_comm_t)."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int, _handle=None):
        self.nranks, self.rank = nranks, rank
        self._owned = _handle is None
        if _handle is not None:        # a simulated rank (SimWorld.comm): owned by its world
            self._h = _handle
            return
        h = ctypes.c_void_p()
        check(lib().moe_comm_init(unique_id, nranks, rank, ctypes.byref(h)), "moe_comm_init")
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(lib().moe_comm_unique_id(buf), "moe_comm_unique_id")
        return buf.raw

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        """Bootstrap over torch.distributed: rank 0 makes the NCCL id and
        broadcasts it (object broadcast over the default group's backend)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(obj[0], world, rank)

    def workspace_bytes(self, algo: str, group_size: int, bytes_per_peer: int) -> int:
        return lib().moe_alltoall_workspace_bytes(self.nranks, ALGOS[algo], group_size,
                                                  bytes_per_peer)

    def alltoall(self, send: torch.Tensor, recv: torch.Tensor, algo: str = "flat",
                 group_size: int = 1, ws: Optional[torch.Tensor] = None) -> torch.Tensor:
        """AllToAll (Alg. 1 steps 3/5): recv[q] on rank r = send[r] on rank q."""
        _need_cuda(send, "send")
        _need_cuda(recv, "recv")
        nb = send.numel() * send.element_size()
        if nb != recv.numel() * recv.element_size() or nb % self.nranks:
            raise ValueError("send/recv must be equal and divisible into nranks chunks")
        check(lib().moe_alltoall(self._h, ALGOS[algo], group_size, _p(send), _p(recv),
                                 nb // self.nranks, _p(ws),
                                 0 if ws is None else ws.numel() * ws.element_size(),
                                 _stream(send.device)), "moe_alltoall")
        return recv

    def symm_empty(self, shape, dtype) -> torch.Tensor:
        """A tensor over a library-owned symmetric buffer (mapped into every
        peer; collective).  Freed by symm_free or destroy."""
        nb = int(torch.Size(shape).numel()) * torch.empty((), dtype=dtype).element_size()
        p = ctypes.c_void_p()
        check(lib().moe_comm_symm_alloc(self._h, nb, ctypes.byref(p)), "moe_comm_symm_alloc")
        return _tensor_from_ptr(p.value, shape, dtype, torch.cuda.current_device())

    def mem_empty(self, shape, dtype) -> torch.Tensor:
        """A tensor over NCCL-registered memory (ncclMemAlloc +
        ncclCommRegister): zero-copy send/recv buffers for alltoall."""
        nb = int(torch.Size(shape).numel()) * torch.empty((), dtype=dtype).element_size()
        p = ctypes.c_void_p()
        check(lib().moe_comm_mem_alloc(self._h, nb, ctypes.byref(p)), "moe_comm_mem_alloc")
        return _tensor_from_ptr(p.value, shape, dtype, torch.cuda.current_device())

    def mem_free(self, t: torch.Tensor):
        check(lib().moe_comm_mem_free(self._h, _p(t)), "moe_comm_mem_free")

    def symm_free(self, t: torch.Tensor):
        check(lib().moe_comm_symm_free(self._h, _p(t)), "moe_comm_symm_free")

    def barrier(self):
        """Device-side barrier of all ranks on the current stream."""
        check(lib().moe_comm_barrier(self._h, _stream()), "moe_comm_barrier")

    NO_ENTRY_BARRIER, NO_EXIT_BARRIER, RECV_UNMODIFIED = 1, 2, 4

    def dispatch_p2p(self, x: torch.Tensor, r: "Routing", recv: torch.Tensor,
                     flags: int = 0) -> torch.Tensor:
        """Layout_Transform fused with the dispatch AllToAll over NVLink:
        rows land directly in the owner rank's symmetric `recv`."""
        _need_cuda(x, "x")
        d = x.shape[-1]
        desc, rc = r.desc(), r.c()
        check(lib().moe_dispatch_p2p(self._h, ctypes.byref(desc), ctypes.byref(rc), _p(x), d,
                                     _DT[x.dtype], _p(recv), flags, _stream(x.device)),
              "moe_dispatch_p2p")
        return recv

    def combine_p2p(self, expert_out: torch.Tensor, r: "Routing",
                    y: Optional[torch.Tensor] = None, flags: int = 0) -> torch.Tensor:
        """AllToAll combine fused with Reverse_Layout_Transform over NVLink:
        every admitted row is read from its owner's symmetric `expert_out`."""
        d = expert_out.shape[-1]
        if y is None:
            y = torch.empty((r.S, d), dtype=expert_out.dtype, device=expert_out.device)
        desc, rc = r.desc(), r.c()
        check(lib().moe_combine_p2p(self._h, ctypes.byref(desc), ctypes.byref(rc), _p(expert_out),
                                    d, _DT[expert_out.dtype], _p(y), flags, _stream(y.device)),
              "moe_combine_p2p")
        return y

    def alltoallv(self, send: torch.Tensor, send_rows, recv: torch.Tensor, recv_rows) -> torch.Tensor:
        """Variable-size AllToAll (NCCL): send_rows / recv_rows are host
        sequences [nranks] of rows of send's row size."""
        _need_cuda(send, "send")
        _need_cuda(recv, "recv", send.dtype)
        row_bytes = send[0].numel() * send.element_size() if send.dim() > 1 else send.element_size()
        sr = (ctypes.c_int64 * self.nranks)(*[int(v) for v in send_rows])
        rr = (ctypes.c_int64 * self.nranks)(*[int(v) for v in recv_rows])
        check(lib().moe_alltoallv(self._h, _p(send), sr, _p(recv), rr, row_bytes,
                                  _stream(send.device)), "moe_alltoallv")
        return recv

    def dispatch_packed_p2p(self, x: torch.Tensor, r: "Routing", offsets: torch.Tensor,
                            counts: torch.Tensor, recv: torch.Tensor, peer_base=None,
                            recv_offsets=None, flags: int = 0):
        """Dropless dispatch over NVLink with the count exchange on the
        device.  counts: symmetric int32 [E]; recv: symmetric [rows, d] with
        rows >= nranks*S*k.  Returns (peer_base [P], recv_offsets [E+1])."""
        _need_cuda(x, "x")
        d = x.shape[-1]
        if peer_base is None:
            peer_base = torch.empty((self.nranks,), dtype=torch.int32, device=x.device)
        if recv_offsets is None:
            recv_offsets = torch.empty((r.E + 1,), dtype=torch.int32, device=x.device)
        desc, rc = r.desc(), r.c()
        check(lib().moe_dispatch_packed_p2p(self._h, ctypes.byref(desc), ctypes.byref(rc),
                                            _p(offsets), _p(counts), _p(peer_base),
                                            _p(recv_offsets), _p(x), d, _DT[x.dtype], _p(recv),
                                            recv.shape[0], flags, _stream(x.device)),
              "moe_dispatch_packed_p2p")
        return peer_base, recv_offsets

    def combine_packed_p2p(self, expert_out: torch.Tensor, r: "Routing", offsets: torch.Tensor,
                           peer_base: torch.Tensor, y: Optional[torch.Tensor] = None,
                           flags: int = 0) -> torch.Tensor:
        """Dropless combine over NVLink from the owners' symmetric expert_out
        (recv layout of dispatch_packed_p2p)."""
        d = expert_out.shape[-1]
        if y is None:
            y = torch.empty((r.S, d), dtype=expert_out.dtype, device=expert_out.device)
        desc, rc = r.desc(), r.c()
        check(lib().moe_combine_packed_p2p(self._h, ctypes.byref(desc), ctypes.byref(rc),
                                           _p(offsets), _p(peer_base), _p(expert_out), d,
                                           _DT[expert_out.dtype], expert_out.shape[0], _p(y),
                                           flags, _stream(y.device)), "moe_combine_packed_p2p")
        return y

    def combine_backward_p2p(self, dy: torch.Tensor, expert_out: torch.Tensor, r: "Routing",
                             d_expert_out: torch.Tensor, d_weight: Optional[torch.Tensor] = None,
                             flags: int = 0):
        """Adjoint of combine_p2p: w*dy stored into the owners' symmetric
        d_expert_out over NVLink, d_weight from the owners' expert_out."""
        _need_cuda(dy, "dy")
        d = dy.shape[-1]
        if d_weight is None:
            d_weight = torch.empty((r.S, r.k), dtype=torch.float32, device=dy.device)
        desc, rc = r.desc(), r.c()
        check(lib().moe_combine_backward_p2p(self._h, ctypes.byref(desc), ctypes.byref(rc), _p(dy),
                                             _p(expert_out), d, _DT[dy.dtype], _p(d_expert_out),
                                             _p(d_weight), flags, _stream(dy.device)),
              "moe_combine_backward_p2p")
        return d_expert_out, d_weight

    def combine_backward_push_p2p(self, dy: torch.Tensor, expert_out: torch.Tensor, r: "Routing",
                                  d_expert_out: torch.Tensor, wtab: torch.Tensor,
                                  dwtab: torch.Tensor, d_weight: Optional[torch.Tensor] = None,
                                  flags: int = 0):
        """Adjoint of combine_p2p, push form: dy rows and weights go to the
        experts' owners, which scale in place and dot with their local
        expert_out (half the NVLink bytes of combine_backward_p2p).
        wtab, dwtab: symmetric float32 [E*cap] scratch."""
        _need_cuda(dy, "dy")
        d = dy.shape[-1]
        if d_weight is None:
            d_weight = torch.empty((r.S, r.k), dtype=torch.float32, device=dy.device)
        desc, rc = r.desc(), r.c()
        check(lib().moe_combine_backward_push_p2p(self._h, ctypes.byref(desc), ctypes.byref(rc),
                                                  _p(dy), _p(expert_out), d, _DT[dy.dtype],
                                                  _p(d_expert_out), _p(wtab), _p(dwtab),
                                                  _p(d_weight), flags, _stream(dy.device)),
              "moe_combine_backward_push_p2p")
        return d_expert_out, d_weight

    def combine_packed_backward_p2p(self, dy: torch.Tensor, expert_out: torch.Tensor,
                                    r: "Routing", offsets: torch.Tensor, peer_base: torch.Tensor,
                                    d_expert_out: torch.Tensor,
                                    d_weight: Optional[torch.Tensor] = None, flags: int = 0):
        """Adjoint of combine_packed_p2p (dropless, NVLink)."""
        d = dy.shape[-1]
        if d_weight is None:
            d_weight = torch.empty((r.S, r.k), dtype=torch.float32, device=dy.device)
        desc, rc = r.desc(), r.c()
        check(lib().moe_combine_packed_backward_p2p(self._h, ctypes.byref(desc), ctypes.byref(rc),
                                                    _p(offsets), _p(peer_base), _p(dy),
                                                    _p(expert_out), d, _DT[dy.dtype],
                                                    expert_out.shape[0], _p(d_expert_out),
                                                    _p(d_weight), flags, _stream(dy.device)),
              "moe_combine_packed_backward_p2p")
        return d_expert_out, d_weight

    def dispatch_packed_backward_p2p(self, d_recv: torch.Tensor, r: "Routing",
                                     offsets: torch.Tensor, peer_base: torch.Tensor,
                                     dx: Optional[torch.Tensor] = None, flags: int = 0):
        """Adjoint of dispatch_packed_p2p (dropless, NVLink)."""
        d = d_recv.shape[-1]
        if dx is None:
            dx = torch.empty((r.S, d), dtype=d_recv.dtype, device=d_recv.device)
        desc, rc = r.desc(), r.c()
        check(lib().moe_dispatch_packed_backward_p2p(self._h, ctypes.byref(desc), ctypes.byref(rc),
                                                     _p(offsets), _p(peer_base), _p(d_recv), d,
                                                     _DT[d_recv.dtype], d_recv.shape[0], _p(dx),
                                                     flags, _stream(dx.device)),
              "moe_dispatch_packed_backward_p2p")
        return dx

    def dispatch_backward_p2p(self, d_recv: torch.Tensor, r: "Routing",
                              dx: Optional[torch.Tensor] = None, flags: int = 0) -> torch.Tensor:
        """Adjoint of dispatch_p2p: dx[t] = sum_j of the owners' d_recv rows."""
        d = d_recv.shape[-1]
        if dx is None:
            dx = torch.empty((r.S, d), dtype=d_recv.dtype, device=d_recv.device)
        desc, rc = r.desc(), r.c()
        check(lib().moe_dispatch_backward_p2p(self._h, ctypes.byref(desc), ctypes.byref(rc),
                                              _p(d_recv), d, _DT[d_recv.dtype], _p(dx), flags,
                                              _stream(dx.device)), "moe_dispatch_backward_p2p")
        return dx

    def check(self):
        """Failure detection (moe_comm_check; synchronises the current
        stream): raises MoeError with status MOE_ERR_TIMEOUT if a device
        barrier gave up waiting for a peer, MOE_ERR_NCCL on an asynchronous
        NCCL error."""
        check(lib().moe_comm_check(self._h, _stream()), "moe_comm_check")

    def abort(self):
        """ncclCommAbort + release, without waiting for the peers."""
        if getattr(self, "_h", None) and self._owned:
            check(lib().moe_comm_abort(self._h), "moe_comm_abort")
        self._h = None

    def destroy(self):
        if getattr(self, "_h", None) and self._owned:
            check(lib().moe_comm_destroy(self._h), "moe_comm_destroy")
        self._h = None


class SimWorld:
    """TEST INFRASTRUCTURE (moe_sim_world): P ranks of the multi-GPU path
    simulated on the current GPU.  comm(r) is a Comm usable with every
    method; its calls are queued, and run() executes all ranks' queued steps
    phase by phase (barriers as step boundaries, NCCL groups matched across
    ranks) on the current stream, with the real kernels."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        h = ctypes.c_void_p()
        check(lib().moe_sim_world_create(nranks, ctypes.byref(h)), "moe_sim_world_create")
        self._h = h
        self.comms = []
        for r in range(nranks):
            c = ctypes.c_void_p()
            check(lib().moe_sim_world_comm(self._h, r, ctypes.byref(c)), "moe_sim_world_comm")
            self.comms.append(Comm(b"", nranks, r, _handle=c))

    def comm(self, rank: int) -> Comm:
        return self.comms[rank]

    def run(self):
        check(lib().moe_sim_world_run(self._h, _stream()), "moe_sim_world_run")

    def live_barrier(self, rank: int):
        """One rank's real (bounded) barrier kernel: tests the timeout."""
        check(lib().moe_sim_live_barrier(self._h, rank, _stream()), "moe_sim_live_barrier")

    def destroy(self):
        if getattr(self, "_h", None):
            for c in self.comms:
                c._h = None
            check(lib().moe_sim_world_destroy(self._h), "moe_sim_world_destroy")
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()


def _tensor_from_ptr(ptr: int, shape, dtype, device_index: int) -> torch.Tensor:
    """Wrap library-owned device memory as a torch tensor (no copy, no free)."""
    n = int(torch.Size(shape).numel())
    typestr = {torch.bfloat16: "<i2", torch.float32: "<f4", torch.int32: "<i4",
               torch.uint8: "|u1"}[dtype]

    class _Holder:
        __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                    "version": 3, "strides": None}
    t = torch.as_tensor(_Holder(), device=torch.device("cuda", device_index))
    if dtype == torch.bfloat16:
        t = t.view(torch.bfloat16)
    return t.view(shape)


def get_tuning() -> dict:
    """The library's process-wide tuning table (moe_tuning_t) as a dict."""
    t = Tuning()
    check(lib().moe_get_tuning(ctypes.byref(t)), "moe_get_tuning")
    return {f: getattr(t, f) for f in TUNING_FIELDS}


def set_tuning(**fields) -> dict:
    """Change fields of the tuning table; returns the previous table."""
    old = get_tuning()
    bad = set(fields) - set(TUNING_FIELDS)
    if bad:
        raise KeyError("unknown tuning fields: %s" % sorted(bad))
    new = dict(old, **fields)
    t = Tuning(*[int(new[f]) for f in TUNING_FIELDS])
    check(lib().moe_set_tuning(ctypes.byref(t)), "moe_set_tuning")
    return old


@contextlib.contextmanager
def tuned(**fields):
    """Run a block with some tuning fields changed (kernel-variant selection;
    every variant computes the same bits), restoring the table after."""
    old = set_tuning(**fields)
    try:
        yield
    finally:
        set_tuning(**old)


def version() -> str:
    return lib().moe_version().decode()
