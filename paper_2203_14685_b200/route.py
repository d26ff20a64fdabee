"""Algorithm 1's routing path on one rank, with every buffer
resident in HBM and sized once: gate -> Layout_Transform -> AllToAll ->
(expert stand-in) -> AllToAll -> Reverse_Layout_Transform.

Orchestration only: each step is one call into libmoe_b200 (kernels) or its
NCCL communicator, all enqueued on the current torch stream with no host
synchronisation (the padded layout makes every size static, R9).
"""
from __future__ import annotations

from typing import Optional

import torch

from .api import (Comm, Gate, Routing, expert_offsets, expert_scale, gate_backward, layout,
                  layout_backward, layout_packed, layout_packed_backward, reverse_layout,
                  reverse_layout_backward, reverse_layout_packed, reverse_layout_packed_backward)


class RoutePipeline:
    def __init__(self, S: int, d: int, E: int, k: int, cap: int, dtype=torch.bfloat16,
                 kind: str = "topk", weight_mode: str = "renorm", priority: str = "token",
                 comm: Optional[Comm] = None, algo: str = "flat", group_size: int = 1,
                 device=None, slot_src: bool = True, dropless: bool = False,
                 fuse_gate_layout: Optional[bool] = None, identity_alias: bool = False,
                 nvtx: bool = False, double_buffer: bool = True, bwd_push: bool = True):
        """dropless=True (NEXT-4): capacity is ignored (cap = S*k, nothing is
        dropped) and the packed layout is used -- locally moe_layout_packed /
        moe_reverse_layout_packed, across ranks the device-side NVLink
        exchange (algo "p2p" only).  The expert stand-in is the identity.
        fuse_gate_layout: steps 1 + 2 as one persistent kernel
        (moe_gate_layout / moe_gate_dispatch_p2p; the library runs the two
        steps separately for shapes it has no fused kernel for).  None =
        off: the separate gate -> layout pair under PDL measured as fast or
        faster (P=1: C2 71.4 vs 77.0 us per step, C3 91.6 vs 100.0; P=2
        one-sided: C2 251.3 vs 251.7, C3 257.0 vs 258.6, C4b 263.6 vs 263.3;
        profiles/r02_gate_layout).
        identity_alias=True (p2p only): a step with expert=False tells the
        combine that recv is unmodified (MOE_P2P_RECV_UNMODIFIED): no entry
        barrier and one read of a row sent once for two slots.  A measurement
        of the routing alone; a real expert always takes the default path.
        nvtx=True: every stage of step() is an NVTX range ("moe/gate",
        "moe/layout", ...) for Nsight timelines.
        double_buffer (padded one-sided path, P > 1): steps alternate two
        symmetric receive buffers, so the combine needs no exit barrier (the
        next dispatch into the same buffer is two steps later, behind another
        dispatch's exit barrier; include/moe.h MOE_P2P_*).  `recv` is the
        buffer of the latest step.
        bwd_push (p2p backward): the push-form combine adjoint (dy rows cross
        once, dots at the owners) instead of reading expert outputs across."""
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self.dropless = dropless
        self.fuse = bool(fuse_gate_layout) and not dropless
        self.identity_alias = identity_alias
        self.nvtx = nvtx
        self.bwd_push = bwd_push
        if dropless:
            cap = S * k
            slot_src = False
        self.comm = comm
        self.P = comm.nranks if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        if E % self.P:
            raise ValueError("E=%d experts do not shard over %d ranks (R10)" % (E, self.P))
        self.S, self.d, self.E, self.k, self.cap = S, d, E, k, cap
        self.E_local = E // self.P
        self.algo, self.group_size = algo, group_size
        self.gate = Gate(S, E, k, cap, kind, weight_mode, priority, self.device)
        self.routing = Routing.empty(S, E, k, cap, self.device, self.gate.kind, self.gate.mode,
                                     self.gate.prio, slot_src)
        mk = lambda *shape: torch.empty(shape, dtype=dtype, device=self.device)
        if dropless:
            if self.P > 1 and algo != "p2p":
                raise ValueError("dropless across ranks uses the device-side NVLink exchange "
                                 "(algo='p2p'); see moe_alltoallv for the NCCL form")
            self.offsets = torch.empty((E + 1,), dtype=torch.int32, device=self.device)
            if self.P > 1:
                rows = self.P * S * k   # worst case: every row to one rank
                self.counts = comm.symm_empty((E,), torch.int32)
                self.recv = comm.symm_empty((rows, d), dtype)
                self.peer_base = torch.empty((self.P,), dtype=torch.int32, device=self.device)
                self.recv_offsets = torch.empty((E + 1,), dtype=torch.int32, device=self.device)
            else:
                self.recv = mk(S * k, d)
            self.dispatch = self.back = self.recv
        elif self.P > 1 and algo == "p2p":
            # one-sided NVLink path: layout fused into the dispatch (rows are
            # stored into the owner's symmetric recv), combine fused into the
            # reverse (rows are read from the owner's recv); no staging
            # buffers; two receive buffers used in turn (double_buffer)
            self._recvs = [comm.symm_empty((E, cap, d), dtype)
                           for _ in range(2 if double_buffer else 1)]
            self._parity = 0
            self.recv = self._recvs[0]
            self.dispatch = self.back = self.recv
        elif self.P > 1:
            # NCCL's send/recv buffers in NCCL-registered memory (ncclMemAlloc
            # + ncclCommRegister): zero-copy over NVLink, measured 491 vs 280
            # GB/s busBW at 128 MiB per rank, P=2 (profiles/r02_multi)
            reg = lambda *shape: comm.mem_empty(shape, dtype)
            self.dispatch = reg(E, cap, d)
            self.recv = reg(E, cap, d)
            self.back = reg(E, cap, d)
        else:
            self.dispatch = mk(E, cap, d)
            self.recv = self.back = self.dispatch
        self.y = mk(S, d)
        self.ws = None
        if self.P > 1 and algo in ("hier", "hier2d"):
            nb = comm.workspace_bytes(algo, group_size, self.dispatch.nbytes // self.P)
            self.ws = comm.mem_empty((max(1, nb),), torch.uint8)

    def _first_flags(self):
        # The first dispatch into a receive buffer needs its entry barrier
        # (peers may not have reached it yet); later ones follow a combine's
        # exit barrier, or (two buffers) the exit barrier of the dispatch into
        # the other buffer, which no rank passes before its combine of this
        # one has finished reading.
        used = getattr(self, "_used", None)
        if used is None:
            used = self._used = set()
        key = self.recv.data_ptr()
        if key not in used:
            used.add(key)
            return 0
        return self.comm.NO_ENTRY_BARRIER

    @property
    def double_buffered(self) -> bool:
        return len(getattr(self, "_recvs", ())) == 2

    def _p2p_begin(self):
        """The padded one-sided path: this step's receive buffer."""
        if hasattr(self, "_recvs"):
            self.recv = self.dispatch = self.back = self._recvs[self._parity]

    def _p2p_end(self):
        if hasattr(self, "_recvs"):
            self._parity = (self._parity + 1) % len(self._recvs)

    def alltoall(self, send, recv):
        if self.P > 1:
            self.comm.alltoall(send, recv, self.algo, self.group_size, self.ws)

    def step(self, logits=None, x=None, token_ids=None, table=None, expert: bool = False,
             mark=None, y=None):
        """One pass of Algorithm 1 on device-resident inputs; returns y.
        `mark(name)` (optional) is called after each stage is enqueued (the
        bench records a CUDA event there)."""
        mark = mark or (lambda name: None)
        if y is not None and y is not self.y:   # write this step's y elsewhere
            saved, self.y = self.y, y
            try:
                return self.step(logits, x, token_ids, table, expert, mark)
            finally:
                self.y = saved
        if self.nvtx:   # NVTX ranges between the stage marks; the last mark is "reverse"
            inner = mark
            torch.cuda.nvtx.range_push("moe/gate")

            def mark(name, _inner=inner):
                _inner(name)
                torch.cuda.nvtx.range_pop()
                if name != "reverse":
                    torch.cuda.nvtx.range_push("moe/after_" + name)
        if self.fuse:
            if self.P > 1 and self.algo == "p2p":
                self._p2p_begin()
                try:
                    return self._step_fused(logits, x, token_ids, table, expert, mark)
                finally:
                    self._p2p_end()
            return self._step_fused(logits, x, token_ids, table, expert, mark)
        if self.P > 1 and self.algo == "p2p" and not self.dropless:
            self._p2p_begin()
            try:
                return self._step_p2p(logits, x, token_ids, table, expert, mark)
            finally:
                self._p2p_end()
        r = self.gate(logits, token_ids, table, out=self.routing)          # step 1
        if self.dropless:
            return self._step_dropless(r, x, mark)
        mark("gate")
        layout(x, r, out=self.dispatch)                                    # step 2
        mark("layout")
        self.alltoall(self.dispatch, self.recv)                            # step 3
        mark("a2a_dispatch")
        if expert:                                                         # step 4 (stand-in)
            expert_scale(self.recv, self.P, self.E_local, self.rank * self.E_local, out=self.recv)
            mark("expert")
        self.alltoall(self.recv, self.back)                                # step 5
        mark("a2a_combine")
        reverse_layout(self.back, r, out=self.y)                           # step 6
        mark("reverse")
        return self.y

    def _step_p2p(self, logits, x, token_ids, table, expert, mark):
        """The padded step on the one-sided NVLink path."""
        r = self.gate(logits, token_ids, table, out=self.routing)          # step 1
        mark("gate")
        self.comm.dispatch_p2p(x, r, self.recv, flags=self._first_flags())  # steps 2+3
        mark("layout")
        mark("a2a_dispatch")
        if expert:                                                         # step 4 (stand-in)
            expert_scale(self.recv, self.P, self.E_local, self.rank * self.E_local, out=self.recv)
            mark("expert")
        # steps 5+6: the entry barrier orders every rank's expert (and the
        # owners' duplicate-row copies) before the reads
        self.comm.combine_p2p(self.recv, r, self.y, flags=self._combine_flags(expert))
        mark("a2a_combine")
        mark("reverse")
        return self.y

    def _combine_flags(self, expert: bool) -> int:
        f = self.comm.NO_EXIT_BARRIER if self.double_buffered else 0
        if self.identity_alias and not expert:
            f |= self.comm.NO_ENTRY_BARRIER | self.comm.RECV_UNMODIFIED
        return f

    def _step_fused(self, logits, x, token_ids, table, expert, mark):
        """The step with the gate and the layout as one kernel (P=1, NCCL
        AllToAlls) or the gate and the one-sided dispatch (p2p).  Its time
        is the "layout" stage (the "gate" stage is empty)."""
        mark("gate")
        if self.P > 1 and self.algo == "p2p":                              # steps 1+2+3
            r = self.gate.with_dispatch_p2p(self.comm, x, self.recv, logits, token_ids, table,
                                            out=self.routing, flags=self._first_flags())
            mark("layout")
            mark("a2a_dispatch")
        else:                                                              # steps 1+2
            r = self.gate.with_layout(x, self.dispatch, logits, token_ids, table,
                                      out=self.routing)
            mark("layout")
            self.alltoall(self.dispatch, self.recv)                        # step 3
            mark("a2a_dispatch")
        if expert:                                                         # step 4 (stand-in)
            expert_scale(self.recv, self.P, self.E_local, self.rank * self.E_local, out=self.recv)
            mark("expert")
        if self.P > 1 and self.algo == "p2p":                              # steps 5+6 fused
            self.comm.combine_p2p(self.recv, r, self.y, flags=self._combine_flags(expert))
            mark("a2a_combine")
            mark("reverse")
            return self.y
        self.alltoall(self.recv, self.back)                                # step 5
        mark("a2a_combine")
        reverse_layout(self.back, r, out=self.y)                           # step 6
        mark("reverse")
        return self.y

    def _step_dropless(self, r, x, mark):
        expert_offsets(r, out=self.offsets)
        mark("gate")
        if self.P > 1:
            self.comm.dispatch_packed_p2p(x, r, self.offsets, self.counts, self.recv,
                                          self.peer_base, self.recv_offsets,
                                          flags=self._first_flags())
            mark("layout")
            mark("a2a_dispatch")
            self.comm.combine_packed_p2p(self.recv, r, self.offsets, self.peer_base, self.y,
                                         flags=self.comm.NO_ENTRY_BARRIER)
            mark("a2a_combine")
            mark("reverse")
            return self.y
        layout_packed(x, r, self.offsets, out=self.recv)
        mark("layout")
        mark("a2a_dispatch")
        mark("a2a_combine")
        reverse_layout_packed(self.recv, r, self.offsets, out=self.y)
        mark("reverse")
        return self.y

    def backward(self, dy: torch.Tensor, logits: Optional[torch.Tensor] = None):
        """Backward of the last step (NEXT-1) with the routing held fixed and
        an identity expert: the adjoints in reverse order -- combine
        (d_back, d_weight) -> AllToAll -> AllToAll -> layout (dx), plus the
        gate (d_logits, when the gate has logits).  Returns (dx, d_logits)."""
        r = self.routing
        if self.dropless and self.P > 1:
            if not hasattr(self, "d_weight"):
                self.d_weight = torch.empty((self.S, self.k), dtype=torch.float32,
                                            device=self.device)
                self.d_recv = self.comm.symm_empty(tuple(self.recv.shape), self.y.dtype)
                self.dx = torch.empty_like(self.y)
                self.d_logits = torch.empty((self.S, self.E), dtype=torch.float32,
                                            device=self.device)
            self.comm.combine_packed_backward_p2p(dy, self.recv, r, self.offsets, self.peer_base,
                                                  self.d_recv, self.d_weight)
            self.comm.dispatch_packed_backward_p2p(self.d_recv, r, self.offsets, self.peer_base,
                                                   self.dx, flags=self.comm.NO_ENTRY_BARRIER)
            dl = None
            if logits is not None and self.gate.kind not in (2, 3, 4):
                dl = gate_backward(logits, r, self.d_weight, out=self.d_logits)
            return self.dx, dl
        if self.dropless:
            if not hasattr(self, "d_weight"):
                self.d_weight = torch.empty((self.S, self.k), dtype=torch.float32,
                                            device=self.device)
                self.d_back = torch.empty_like(self.recv)
                self.dx = torch.empty_like(self.y)
                self.d_logits = torch.empty((self.S, self.E), dtype=torch.float32,
                                            device=self.device)
            reverse_layout_packed_backward(dy, self.recv, r, self.offsets, self.d_back,
                                           self.d_weight)
            layout_packed_backward(self.d_back, r, self.offsets, out=self.dx)
            dl = None
            if logits is not None and self.gate.kind not in (2, 3, 4):
                dl = gate_backward(logits, r, self.d_weight, out=self.d_logits)
            return self.dx, dl
        if not hasattr(self, "d_weight"):
            mk = lambda *shape: torch.empty(shape, dtype=self.y.dtype, device=self.device)
            self.d_weight = torch.empty((self.S, self.k), dtype=torch.float32, device=self.device)
            self.dx = mk(self.S, self.d)
            self.d_logits = torch.empty((self.S, self.E), dtype=torch.float32, device=self.device)
            if self.P > 1 and self.algo == "p2p":
                self.d_recv = self.comm.symm_empty((self.E, self.cap, self.d), self.y.dtype)
                self.wtab = self.comm.symm_empty((self.E * self.cap,), torch.float32)
                self.dwtab = self.comm.symm_empty((self.E * self.cap,), torch.float32)
            elif self.P > 1:   # NCCL send/recv buffers: registered (see __init__)
                self.d_back, self.d_recv, self.d_disp = (
                    self.comm.mem_empty((self.E, self.cap, self.d), self.y.dtype) for _ in range(3))
            else:
                self.d_back = self.d_recv = self.d_disp = mk(self.E, self.cap, self.d)
        if self.P > 1 and self.algo == "p2p":
            # d_back rows are stored straight into the owners' d_recv, then
            # every dx row gathers its gradient rows back over NVLink
            if self.bwd_push:
                # push form: dy rows travel once, dots are taken at the owners
                self.comm.combine_backward_push_p2p(dy, self.recv, r, self.d_recv, self.wtab,
                                                    self.dwtab, self.d_weight)
            else:
                self.comm.combine_backward_p2p(dy, self.recv, r, self.d_recv, self.d_weight)
            self.comm.dispatch_backward_p2p(self.d_recv, r, self.dx,
                                            flags=self.comm.NO_ENTRY_BARRIER)
        else:
            reverse_layout_backward(dy, self.back, r, self.d_back, self.d_weight)
            self.alltoall(self.d_back, self.d_recv)        # adjoint of step 5
            self.alltoall(self.d_recv, self.d_disp)        # adjoint of step 3 (identity expert)
            layout_backward(self.d_disp, r, out=self.dx)
        dl = None
        if logits is not None and self.gate.kind != 2:
            dl = gate_backward(logits, r, self.d_weight, out=self.d_logits)
        return self.dx, dl

    STAGES = ("gate", "layout", "a2a_dispatch", "a2a_combine", "reverse")

    def capture(self, logits=None, x=None, token_ids=None, table=None, expert: bool = False,
                stages: bool = False, events=None):
        """Capture the step into CUDA graph(s) bound to these input tensors
        (refill them in place between replays).  stages=False: one graph for
        the whole step; with `events` (len(STAGES)+1 torch.cuda.Event(
        enable_timing=True, external=True)) event-record nodes bracket every
        stage inside that graph.  stages=True: {stage: graph}.  Run one eager
        step first (NCCL's lazy setup must not happen inside a capture).
        Double-buffered one-sided path (stages=False): one graph per receive
        buffer (an eager step first initialises a buffer not used yet),
        returned as one object whose replay() runs the graph of the buffer
        whose turn it is -- graphs and eager steps may be mixed freely."""
        if self.double_buffered and not stages:
            graphs = {}
            while not all(b.data_ptr() in getattr(self, "_used", ()) for b in self._recvs):
                self.step(logits, x, token_ids, table, expert)
            for _ in range(2):
                p = self._parity
                graphs[p] = self._capture_one(logits, x, token_ids, table, expert, False, events)
            return _AlternatingGraph(self, graphs)
        return self._capture_one(logits, x, token_ids, table, expert, stages, events)

    def _capture_one(self, logits, x, token_ids, table, expert, stages, events):
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        graphs = {}
        with torch.cuda.stream(s):
            if not stages:
                g = torch.cuda.CUDAGraph()
                mark = None
                if events is not None:
                    order = {n: i + 1 for i, n in enumerate(self.STAGES)}
                    mark = lambda name: events[order[name]].record() if name in order else None
                with torch.cuda.graph(g, stream=s):
                    if events is not None:
                        events[0].record()
                    self.step(logits, x, token_ids, table, expert, mark=mark)
                graphs = g
            else:
                if self.dropless or self.fuse:
                    raise NotImplementedError("per-stage graphs cover the padded, unfused step; "
                                              "use stages=False with events= instead")
                r = self.routing
                p2p = self.P > 1 and self.algo == "p2p"
                fns = {
                    "gate": lambda: self.gate(logits, token_ids, table, out=r),
                    "layout": (lambda: self.comm.dispatch_p2p(x, r, self.recv, flags=1)) if p2p else
                              (lambda: layout(x, r, out=self.dispatch)),
                    "a2a_dispatch": lambda: self.alltoall(self.dispatch, self.recv),
                    "a2a_combine": (lambda: self.comm.combine_p2p(self.recv, r, self.y, flags=1))
                                   if p2p else
                                   (lambda: self.alltoall(self.recv, self.back)),
                    "reverse": lambda: reverse_layout(self.back, r, out=self.y),
                }
                for name in self.STAGES:
                    if (self.P == 1 or p2p) and name == "a2a_dispatch":
                        continue   # P=1: recv aliases dispatch; p2p: fused into "layout"
                    if self.P == 1 and name == "a2a_combine":
                        continue
                    if p2p and name == "reverse":
                        continue   # fused into "a2a_combine"
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=s):
                        fns[name]()
                    graphs[name] = g
        torch.cuda.current_stream(self.device).wait_stream(s)
        return graphs

    def run_host(self, batches, outs, expert: bool = False):
        """End-to-end over HOST batches with the copies overlapped: batch i's
        inputs go host->device on a copy-in stream while batch i-1 computes,
        and batch i-1's y goes device->host on a copy-out stream (PCIe is
        full duplex), with double-buffered device staging.  `batches`: dicts
        of pinned host tensors (logits, x, token_ids, table); `outs`: pinned
        host y tensors, one per batch.  Enqueues everything; the caller
        synchronises (or records events) as it likes."""
        dev = self.device
        cur = torch.cuda.current_stream(dev)
        if not hasattr(self, "_pipe_streams"):
            self._pipe_streams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
            self._pipe_stage = [{}, {}]
            self._pipe_y = [torch.empty_like(self.y), torch.empty_like(self.y)]
        s_in, s_out = self._pipe_streams
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_comp = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        used = [False, False]
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        for i, (b, y_h) in enumerate(zip(batches, outs)):
            j = i % 2
            stage = self._pipe_stage[j]
            with torch.cuda.stream(s_in):
                if used[j]:
                    s_in.wait_event(ev_comp[j])       # step i-2 is done reading stage j
                for name in ("logits", "x", "token_ids", "table"):
                    h = b.get(name)
                    if h is None:
                        continue
                    t = stage.get(name)
                    if t is None:
                        t = stage[name] = torch.empty(h.shape, dtype=h.dtype, device=dev)
                    t.copy_(h, non_blocking=True)
                ev_in[j].record(s_in)
            cur.wait_event(ev_in[j])
            if used[j]:
                cur.wait_event(ev_out[j])             # y buffer j has been read out
            self.step(stage.get("logits"), stage.get("x"), stage.get("token_ids"),
                      stage.get("table"), expert, y=self._pipe_y[j])
            ev_comp[j].record(cur)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_comp[j])
                y_h.copy_(self._pipe_y[j], non_blocking=True)
                ev_out[j].record(s_out)
            used[j] = True
        cur.wait_stream(s_in)
        cur.wait_stream(s_out)
        return outs

    def step_host(self, logits_h=None, x_h=None, y_h=None, token_ids_h=None, table_h=None,
                  expert: bool = False, inputs=None):
        """The same pass from HOST buffers (pinned for async copies): copy the
        step's inputs host->device, run it, copy y device->host into y_h.
        `inputs` (optional) are device staging tensors to reuse."""
        dev_in = inputs or {}
        def up(name, h):
            if h is None:
                return None
            t = dev_in.get(name)
            if t is None:
                t = dev_in[name] = torch.empty(h.shape, dtype=h.dtype, device=self.device)
            t.copy_(h, non_blocking=True)
            return t
        y = self.step(up("logits", logits_h), up("x", x_h), up("token_ids", token_ids_h),
                      up("table", table_h), expert)
        if y_h is None:
            y_h = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
        y_h.copy_(y, non_blocking=True)
        return y_h


class _AlternatingGraph:
    """The step graphs of a double-buffered pipeline, one per receive buffer:
    replay() runs the one whose turn it is and advances the turn (shared with
    eager steps)."""

    def __init__(self, pipe: RoutePipeline, graphs: dict):
        self.pipe, self.graphs = pipe, graphs

    def replay(self):
        p = self.pipe._parity
        self.pipe.recv = self.pipe.dispatch = self.pipe.back = self.pipe._recvs[p]
        self.graphs[p].replay()
        self.pipe._parity = (p + 1) % len(self.pipe._recvs)
