#!/usr/bin/env python
"""bench.py -- MoE dispatch+combine tokens/s of the HetuMoE routing path on
B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2]
                    [--algo p2p|flat|hier|hier2d] [--group-size G] [--impl ours|reference]
    # N > 1 is launched either way:
    #   python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...
    #   python bench.py --gpus N ...   (re-executes itself under torch.distributed.run)

A step is one pass of the whole routing path on one batch of S tokens per
rank (Algorithm 1): gate (select + weights + capacity) ->
Layout_Transform -> AllToAll dispatch -> AllToAll combine ->
Reverse_Layout_Transform.  The expert is the identity inside the timed step
(routing isolated, north_star); the s_e stand-in is timed separately
(`expert_ms`).  Inputs are synthetic (synthgen, seeded) and resident in HBM;
the L2 is flushed (a 2x-L2 memset, then a 2x-L2 read so no dirty line is left) between
timed steps, outside the events.
Each step is timed with CUDA events on the launching stream; the reported
time is the max over ranks.  `value` = tokens of all ranks / time.

--impl reference runs the CPU oracle (oracle/, plain single-threaded C) on a
bounded sample of the same workload -- the reference arm of this tier.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "MoE dispatch+combine tokens/s"
UNIT = "tokens/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
NVLINK_GBS = 770.0         # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--tokens", type=int, default=0,
                    help="tokens per rank instead of the workload's S (e.g. C5's end-to-end "
                         "points: S = 4096 / 32768 / 262144 for B = 16 / 128 / 1024 MiB)")
    ap.add_argument("--algo", default="p2p", choices=["p2p", "flat", "hier", "hier2d"],
                    help="AllToAll at N>1: p2p = fused one-sided NVLink path (falls back to "
                         "flat if the GPUs cannot map each other's memory); flat / hier (the "
                         "paper's leader scheme) / hier2d (two-level) = NCCL")
    ap.add_argument("--group-size", type=int, default=0, help="hier group size (default N/2)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-backward", action="store_true")
    ap.add_argument("--fuse", default="auto", choices=["auto", "on", "off"],
                    help="gate + layout (+ NVLink dispatch) as one kernel: auto = the "
                         "RoutePipeline default (off: the separate pair measured as fast)")
    ap.add_argument("--single-buffer", action="store_true",
                    help="one-sided path: one receive buffer (combine keeps its exit barrier) "
                         "instead of the default two used in turn")
    ap.add_argument("--dropless", action="store_true",
                    help="NEXT-4: packed dropless layout (capacity = S*k), device-side exchange")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--verbose", action="store_true", help="progress on stderr")
    return ap.parse_args()


# ---------------------------------------------------------------- helpers
def relaunch_if_needed():
    """`bench.py --gpus N` without torchrun: re-execute under
    torch.distributed.run with N ranks (one per GPU) and return its exit
    code; None when this process is already one rank of the right world.
    A WORLD_SIZE that disagrees with --gpus is an error."""
    a = parse()
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != a.gpus:
            sys.stderr.write("bench.py: --gpus %d but WORLD_SIZE=%s\n" % (a.gpus, world))
            return 2
        return None
    if a.gpus <= 1:
        return None
    import socket
    with socket.socket() as s:          # a free rendezvous port on 127.0.0.1
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(a.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the
    timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                 "-i", ",".join(map(str, self.gpus)), "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def rejected(clocks):
    if not clocks:
        return False
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if bad & set(clocks["reasons"]):
        return True
    return clocks["sm_mhz"] < 0.5 * clocks["sm_max_mhz"] and not clocks["reasons"]


def algorithmic_bytes(w, S, cap, P, row):
    """Per-launch algorithmic bytes."""
    return {
        "gate": S * (4 * w.E if w.kind != "hash" else 8) + 12 * S * w.k + 4 * w.E + 4 * w.E * cap,
        "layout": S * row + w.E * cap * row + 8 * S * w.k,
        "reverse": None,   # needs the admitted count: filled in at run time
        "a2a": (P - 1) * (w.E * cap * row // P),
    }


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------- reference arm
def oracle_step(orc, w, inputs, cap, P):
    xs = [i[3] for i in inputs]
    lgs = None if w.kind == "hash" else [i[0] for i in inputs]
    ids = None if w.kind != "hash" else [i[1] for i in inputs]
    table = None if w.kind != "hash" else inputs[0][2]
    return orc.route_multi(xs, lgs, E=w.E, k=w.k, cap=cap, kind=w.kind, token_ids_list=ids,
                           table=table, scale=False)


def cpu_sample(w, P, target_s):
    """A bounded sample of the workload for the oracle: S_s tokens per rank
    (the full S if one P-rank step costs <= ~1.5 s on one core)."""
    per_tok = 14e-6 * w.d / 1024 * max(1, w.k)   # measured ~0.45 s for C2 (32768 tok) per rank
    S_s = w.S
    while S_s > 256 and P * S_s * per_tok > 1.5:
        S_s //= 2
    return S_s


def run_reference(a, w, world, rank):
    import oracle
    import synthgen
    if rank != 0:
        return
    P = world
    S_s = cpu_sample(w, P, a.cpu_seconds)
    cap = oracle.capacity(S_s, w.E, w.k, w.C)
    inputs = [synthgen.workload_inputs(w, r, S=S_s) for r in range(P)]
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass
    for _ in range(max(0, a.warmup)):
        oracle_step(oracle, w, inputs, cap, P)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        oracle_step(oracle, w, inputs, cap, P)
    dt = (time.perf_counter() - t0) / max(1, a.steps)
    value = P * S_s / dt
    sample = ("oracle route (gate+layout+AllToAll sim+AllToAll sim+reverse) on %d simulated "
              "rank(s) x %d tokens per rank of %s (full S=%d), 1 thread" % (P, S_s, w.name, w.S))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 (oracle)", "data": "synthetic",
        "config": {"workload": w.name, "S_per_rank": S_s, "d": w.d, "E": w.E, "k": w.k,
                   "gate": w.kind, "capacity_factor": w.C, "parallelism": "ep%d" % P},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- our arm
def main():
    a = parse()
    import synthgen
    w = synthgen.WORKLOADS[a.workload]
    if a.tokens:
        import dataclasses
        w = dataclasses.replace(w, S=a.tokens)
    world, rank, local = dist_env()
    if a.impl == "reference":
        run_reference(a, w, world, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2203_14685_b200 as moe

    t_start = time.time()

    def log(msg):
        if a.verbose:
            sys.stderr.write("[bench r%d %.1fs] %s\n" % (rank, time.time() - t_start, msg))
            sys.stderr.flush()

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("cpu:gloo,cuda:nccl", device_id=dev)
    P = world
    G = a.group_size or max(1, P // 2)
    log("process group up")
    comm = moe.Comm.from_process_group() if P > 1 else None
    log("moe comm up")
    S = w.S
    cap = moe.capacity(S, w.E, w.k, w.C)
    dt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    row = w.d * (2 if w.dtype == "bf16" else 4)
    algo = a.algo if P > 1 else "flat"
    if a.dropless:
        cap = S * w.k     # nothing is dropped; the packed form has no padding (NEXT-4)
        if P > 1:
            algo = "p2p"
    try:
        pipe = moe.RoutePipeline(S, w.d, w.E, w.k, cap, dt, w.kind, comm=comm, algo=algo,
                                 group_size=G, device=dev, dropless=a.dropless,
                                 fuse_gate_layout={"auto": None, "on": True, "off": False}[a.fuse],
                                 double_buffer=not a.single_buffer)
    except moe.MoeError as err:
        if algo != "p2p":
            raise
        log("p2p unavailable (%s): NCCL flat AllToAll instead" % err)
        algo = "flat"
        pipe = moe.RoutePipeline(S, w.d, w.E, w.k, cap, dt, w.kind, comm=comm, algo=algo,
                                 group_size=G, device=dev,
                                 fuse_gate_layout={"auto": None, "on": True, "off": False}[a.fuse],
                                 double_buffer=not a.single_buffer)

    lg, ids, table, x = synthgen.workload_inputs(w, rank)

    def pinned(arr):
        if arr is None:
            return None
        t = torch.from_numpy(np.ascontiguousarray(arr))
        if arr.dtype == np.uint16:
            t = t.view(torch.int16).view(torch.bfloat16)
        return t.pin_memory()

    host = {"logits": pinned(lg), "x": pinned(x), "token_ids": pinned(ids), "table": pinned(table)}
    d_in = {k: (None if v is None else v.to(dev)) for k, v in host.items()}
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20), dtype=torch.uint8, device=dev)
    flush_rd = torch.zeros_like(flush)
    flush_sink = torch.empty((), dtype=torch.int64, device=dev)

    def flush_l2():
        # write 2x L2 (evicts every line of the previous step), then read
        # another 2x L2 so the write-back of those dirty lines happens HERE,
        # outside the events, not inside the next timed step: L2 is left cold
        # (no line of the step's data) and clean.
        flush.zero_()
        torch.sum(flush_rd.view(torch.int64), dim=0, out=flush_sink)

    def barrier():
        if P > 1:
            dist.barrier()

    # Per-step alignment of the ranks' streams, OUTSIDE the events: without
    # it, host-side launch skew between ranks shows up as device time inside
    # the step (the first exchange waits for the latest rank).  A device-side
    # barrier (moe_comm_barrier over NVLink) when peer memory is available.
    can_align = P > 1 and comm is not None
    def align():
        nonlocal can_align
        if can_align:
            try:
                comm.barrier()
            except moe.MoeError:
                can_align = False

    def step(mark=None):
        return pipe.step(d_in["logits"], d_in["x"], d_in["token_ids"], d_in["table"],
                         expert=False, mark=mark)

    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize()
    log("eager warm-up done")

    stages = list(pipe.STAGES)
    # The timed step is ONE CUDA graph replay (gate, layout, AllToAll x2,
    # reverse: no host launch gaps); the per-stage breakdown comes from a
    # second capture with timing events recorded inside the graph.
    g_step = pipe.capture(d_in["logits"], d_in["x"], d_in["token_ids"], d_in["table"])
    ev_in = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(stages) + 1)]
    g_timed = pipe.capture(d_in["logits"], d_in["x"], d_in["token_ids"], d_in["table"],
                           events=ev_in)
    log("graphs captured")
    for _ in range(2):
        g_step.replay()
        g_timed.replay()
    torch.cuda.synchronize()
    log("graph warm-up done")

    def timed(K):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)]
        barrier()
        torch.cuda.synchronize()
        for i in range(K):
            flush_l2()                          # L2 flush, outside the events
            align()
            ev[i][0].record()
            g_step.replay()
            ev[i][1].record()
        torch.cuda.synchronize()
        barrier()
        return [s.elapsed_time(e) for s, e in ev]

    def timed_stages(K):
        """Per-stage device times from event-record nodes INSIDE the step
        graph (no extra launch latency in the breakdown)."""
        out = [[] for _ in stages]
        barrier()
        torch.cuda.synchronize()
        for i in range(K):
            flush_l2()
            align()
            g_timed.replay()
            torch.cuda.synchronize()
            for j in range(len(stages)):
                out[j].append(ev_in[j].elapsed_time(ev_in[j + 1]))
        barrier()
        return out

    def timed_eager(K):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)]
        barrier()
        torch.cuda.synchronize()
        for i in range(K):
            flush_l2()
            align()
            ev[i][0].record()
            step()
            ev[i][1].record()
        torch.cuda.synchronize()
        barrier()
        return [s.elapsed_time(e) for s, e in ev]

    gpus = list(range(torch.cuda.device_count())) if P > 1 else [local]
    clocks = None
    for attempt in range(2):
        sampler = ClockSampler(gpus) if (rank == 0 and not a.no_clocks) else None
        if sampler:
            sampler.start()
            time.sleep(0.3)
        tot = timed(a.steps)
        if sampler:
            time.sleep(0.25)
            clocks = sampler.stop()
        bad = torch.tensor([1.0 if rejected(clocks) else 0.0])
        if P > 1:
            dist.broadcast(bad, 0)
        if bad.item() == 0:
            break
    log("timed steps done")
    st = timed_stages(a.steps)
    log("stage timing done")
    eager = timed_eager(max(3, a.steps // 2))
    log("eager timing done")
    # N > 1 one-sided path: the row kernels' own spans (moe_set_trace stamps
    # per CTA, one traced graph replay after the timed steps, max over ranks):
    # the dispatch kernel (k_layout in peer mode) and the combine kernel
    # (k_reverse_k in peer mode), without the barriers and owner-side copies
    # that the stage times include
    kernel_spans = None
    if P > 1 and algo == "p2p" and not a.dropless:
        from paper_2203_14685_b200._lib import lib as _tlib
        tbuf = torch.zeros(1 << 20, dtype=torch.int64, device=dev)
        _tlib().moe_set_trace(tbuf.data_ptr(), tbuf.numel() * 8)
        g_tr = pipe.capture(d_in["logits"], d_in["x"], d_in["token_ids"], d_in["table"])
        _tlib().moe_set_trace(None, 0)
        spans = []
        for _ in range(3):
            flush_l2()
            tbuf.zero_()
            torch.cuda.synchronize()
            barrier()
            align()
            g_tr.replay()
            torch.cuda.synchronize()
            raw = tbuf.cpu().numpy()
            n = raw.size
            sp = []
            for lo in (n // 2, 3 * n // 4):
                c = raw[lo:lo + n // 4].reshape(-1, 4)[:, :3]
                c = c[c[:, 0] > 0]
                sp.append(float(c[:, 2].max() - c[:, 1].min()) / 1e3 if c.size else 0.0)
            spans.append(sp)
        del g_tr
        sp_t = torch.tensor([statistics.median(x[0] for x in spans),
                             statistics.median(x[1] for x in spans)], dtype=torch.float64, device=dev)
        dist.all_reduce(sp_t, op=dist.ReduceOp.MAX)
        kernel_spans = {"dispatch_us": float(sp_t[0]), "combine_us": float(sp_t[1])}
        log("row-kernel spans done")
    # N > 1 one-sided path: the identity-expert alias form, an extra (the
    # headline above keeps the combine's entry barrier and reads every slot)
    alias_ms = None
    if P > 1 and algo == "p2p" and not a.dropless:
        pipe.identity_alias = True
        step()
        torch.cuda.synchronize()
        g_alias = pipe.capture(d_in["logits"], d_in["x"], d_in["token_ids"], d_in["table"])
        g_alias.replay()
        torch.cuda.synchronize()
        ev_a = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(max(3, a.steps // 2))]
        barrier()
        torch.cuda.synchronize()
        for s_, e_ in ev_a:
            flush_l2()
            align()
            s_.record()
            g_alias.replay()
            e_.record()
        torch.cuda.synchronize()
        barrier()
        t_a = torch.tensor([statistics.mean(s_.elapsed_time(e_) for s_, e_ in ev_a)],
                           dtype=torch.float64, device=dev)
        dist.all_reduce(t_a, op=dist.ReduceOp.MAX)
        alias_ms = float(t_a.item())
        pipe.identity_alias = False
        del g_alias
        log("identity-alias timing done")
    # max over ranks (per step mean, per stage mean)
    vals = torch.tensor([statistics.mean(tot)] + [statistics.mean(s) for s in st] +
                        [min(tot), statistics.mean(eager)], dtype=torch.float64)
    if P > 1:
        vals_d = vals.to(dev)
        dist.all_reduce(vals_d, op=dist.ReduceOp.MAX)
        vals = vals_d.cpu()
    ms = float(vals[0])
    stage_ms = {s: float(vals[1 + j]) for j, s in enumerate(stages)}
    value = P * S / (ms / 1e3)

    # expert stand-in, timed on its own (not part of the step)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush_l2()
    e0.record()
    if not a.dropless:
        moe.expert_scale(pipe.recv, P, w.E // P, rank * (w.E // P), out=pipe.recv)
    e1.record()
    torch.cuda.synchronize()
    expert_ms = None if a.dropless else e0.elapsed_time(e1)

    # ---- backward of the routing path (NEXT-1), informational: the adjoint
    # kernels of the same step (combine -> AllToAll x2 -> layout, + gate),
    # one CUDA graph, L2 flushed between replays, max over ranks
    bwd = None
    if not a.no_backward:
        dy = torch.from_numpy(synthgen.tokens(synthgen.seed_for(w.index, rank, 9), S, w.d,
                                              w.dtype))
        if w.dtype == "bf16":
            dy = dy.view(torch.int16).view(torch.bfloat16)
        dy = dy.to(dev)
        step()
        for _ in range(2):
            pipe.backward(dy, d_in["logits"])
        torch.cuda.synchronize()
        sb = torch.cuda.Stream(dev)
        sb.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(sb):
            g_bwd = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_bwd, stream=sb):
                pipe.backward(dy, d_in["logits"])
        torch.cuda.current_stream(dev).wait_stream(sb)
        g_bwd.replay()
        torch.cuda.synchronize()
        Kb = max(3, a.steps // 2)
        evb = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(Kb)]
        barrier()
        torch.cuda.synchronize()
        for i in range(Kb):
            flush_l2()
            align()
            evb[i][0].record()
            g_bwd.replay()
            evb[i][1].record()
        torch.cuda.synchronize()
        barrier()
        tb = torch.tensor([statistics.mean(s_.elapsed_time(e_) for s_, e_ in evb)],
                          dtype=torch.float64)
        if P > 1:
            tbd = tb.to(dev)
            dist.all_reduce(tbd, op=dist.ReduceOp.MAX)
            tb = tbd.cpu()
        bms = float(tb[0])
        bwd = {"ms_per_step": bms, "train_value": P * S / ((ms + bms) / 1e3), "unit": UNIT,
               "what": "adjoints of the routing step with an identity expert: "
                       "reverse_layout_backward (d_back scatter + d_weight) -> AllToAll x2 -> "
                       "layout_backward (dx) + gate_backward (d_logits); train_value = tokens / "
                       "(forward + backward)"}
        del g_bwd
        log("backward timing done")

    # ---- end to end through the public API from pinned host buffers:
    # RoutePipeline.run_host over K2 batches, the H2D of batch i+1 and the D2H
    # of batch i-1 overlapping batch i's compute (PCIe is full duplex); every
    # batch's input copy and output read is inside the timed region
    e2e = None
    if not a.no_e2e:
        y_hs = [torch.empty((S, w.d), dtype=dt, pin_memory=True) for _ in range(2)]
        batch = {"logits": host["logits"], "x": host["x"], "token_ids": host["token_ids"],
                 "table": host["table"]}
        K2 = max(4, a.steps // 2)
        pipe.run_host([batch] * 2, y_hs)                      # warm-up (allocations)
        torch.cuda.synchronize()
        staging = {}
        pipe.step_host(host["logits"], host["x"], y_hs[0], host["token_ids"], host["table"],
                       inputs=staging)
        torch.cuda.synchronize()
        barrier()
        flush_l2()
        align()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.run_host([batch] * K2, [y_hs[i % 2] for i in range(K2)])
        e1.record()
        torch.cuda.synchronize()
        barrier()
        # the serial form (one batch at a time) for comparison
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(3)]
        for i in range(3):
            flush_l2()
            align()
            evs[i][0].record()
            pipe.step_host(host["logits"], host["x"], y_hs[0], host["token_ids"], host["table"],
                           inputs=staging)
            evs[i][1].record()
        torch.cuda.synchronize()
        barrier()
        t_e2e = torch.tensor([e0.elapsed_time(e1) / K2,
                              statistics.mean(s_.elapsed_time(e_) for s_, e_ in evs)],
                             dtype=torch.float64)
        if P > 1:
            t_d = t_e2e.to(dev)
            dist.all_reduce(t_d, op=dist.ReduceOp.MAX)
            t_e2e = t_d.cpu()
        h2d = sum(v.numel() * v.element_size() for k, v in host.items()
                  if v is not None and k != "table") + (
            host["table"].numel() * 4 if host["table"] is not None else 0)
        e2e = {"value": P * S / (float(t_e2e[0]) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(S * row),
               "ms_per_step": float(t_e2e[0]), "batches": K2,
               "how": "RoutePipeline.run_host: pinned host batches, H2D / compute / D2H on "
                      "separate streams, double-buffered (max over ranks)",
               "serial_ms_per_step": float(t_e2e[1])}

    # ---- roofline of the dominant kernel
    admitted = int((pipe.routing.slot_idx >= 0).sum().item())
    ab = algorithmic_bytes(w, S, cap, P, row)
    ab["reverse"] = admitted * row + S * row + 12 * S * w.k
    tun = moe.get_tuning()
    p2p_flags = {"dedupe": False, "local_pad": False, "precombine": False}
    if a.dropless:
        # packed: no padding rows; the rows leaving this rank are the admitted
        # rows of other ranks' experts
        ab["layout"] = S * row + admitted * row + 8 * S * w.k
        ab["gate"] = S * (4 * w.E if w.kind != "hash" else 8) + 12 * S * w.k + 8 * w.E
    if P > 1 and algo == "p2p":
        # bytes that actually cross NVLink per rank and direction (DESIGN.md
        # §6): admitted rows of other ranks' experts -- a token's row once per
        # remote owner when the dispatch dedupes (k >= 2, E/P >= 2) -- plus,
        # in the padded form, the padding rows of the remote chunks unless the
        # owners write them (local padding).  The timed combine reads every
        # admitted remote slot (an expert may have written recv); the
        # identity-expert alias form reads a deduped row once.
        El = w.E // P
        ex, sl = pipe.routing.expert_idx.view(S, w.k), pipe.routing.slot_idx.view(S, w.k)
        adm = (ex >= 0) & (sl >= 0)
        own = torch.where(adm, ex // El, torch.full_like(ex, -1))
        remote_slots = int((adm & (own != rank)).sum().item())
        owners = torch.zeros((S, P), dtype=torch.bool, device=own.device)
        for j in range(w.k):
            m = own[:, j] >= 0
            owners[torch.nonzero(m).squeeze(1), own[m, j].long()] = True
        owners[:, rank] = False
        pairs = int(owners.sum().item())
        dedupe = (not a.dropless) and tun["p2p_dedupe"] and w.k >= 2 and El >= 2
        heavy = w.E * cap > 1.05 * S * w.k
        local_pad = a.dropless or (heavy if tun["p2p_local_pad"] < 0 else bool(tun["p2p_local_pad"]))
        pads = 0
        if not local_pad:
            load = pipe.routing.load.view(P, El)
            padrows = cap - load.clamp(max=cap)
            pads = int(padrows.sum().item() - padrows[rank].sum().item())
        precombine = bool(dedupe and w.k == 2 and tun["p2p_precombine"] and tun["reverse_kspec"]
                          and row % 32 == 0)
        p2p_flags = {"dedupe": bool(dedupe), "local_pad": bool(local_pad),
                     "double_buffer": pipe.double_buffered, "precombine": precombine}
        ab["a2a_buffer"] = ab["a2a"]
        ab["a2a_dispatch"] = ((pairs if dedupe else remote_slots) + pads) * row
        # the combine reads every admitted remote slot, except that a
        # pre-combined pair (both slots on one remote owner) is one row
        ab["a2a_combine"] = (pairs if precombine else remote_slots) * row
        ab["a2a_combine_alias"] = (pairs if dedupe else remote_slots) * row
        ab["a2a"] = ab["a2a_dispatch"]
    elif P > 1:
        ab["a2a_dispatch"] = ab["a2a_combine"] = ab["a2a"]
    # gate + layout as one kernel (moe_gate_layout / moe_gate_dispatch_p2p):
    # its time is the "layout" stage and its bytes are both steps' bytes
    fused_gl = pipe.fuse and w.kind in ("topk", "ktop1", "hash") and w.k <= 8 and row % 32 == 0
    if fused_gl:
        ab["layout"] += ab["gate"]
    peak, peak_src = measured_peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f)
    except Exception:
        tr = {}
    fused = P > 1 and algo == "p2p"
    if not fused:
        # N=1 (or NCCL AllToAll): layout / reverse are HBM-bound row movers
        dom = "layout" if stage_ms["layout"] >= stage_ms["reverse"] else "reverse"
        achieved = ab[dom] / (stage_ms[dom] / 1e3) / 1e9
        kname = "k_gate_layout" if (dom == "layout" and fused_gl) else "k_" + dom
        roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak,
                "traffic": tr.get("%s/%s" % (w.name, dom + ("_k" if dom == "reverse" and w.k <= 2 else "")),
                                  tr.get("%s/%s" % (w.name, dom))),
                "algorithmic_bytes": ab[dom], "peak_source": peak_src}
    else:
        # fused one-sided path: the dispatch (k_layout in peer mode) and the
        # combine (k_reverse in peer mode) are bound by the bytes that must
        # cross NVLink (ab["a2a_dispatch"], ab["a2a_combine"])
        t_d, t_c = stage_ms["layout"] / 1e3, stage_ms["a2a_combine"] / 1e3
        dom = "layout" if t_d >= t_c else "a2a_combine"
        nb = ab["a2a_dispatch"] if dom == "layout" else ab["a2a_combine"]
        achieved = nb / (t_d if dom == "layout" else t_c) / 1e9
        roof = {"bound": "nvlink", "kernel": ("k_gate_layout" if fused_gl else "k_layout") +
                " (peer dispatch)" if dom == "layout"
                else "k_reverse_k (peer combine)", "achieved": achieved, "peak": NVLINK_GBS,
                "unit": "GB/s", "frac": achieved / NVLINK_GBS, "traffic": None,
                "algorithmic_bytes": nb,
                "peak_source": "measured peer copy per direction (B200_PROFILING.md), 900 nominal",
                "note": "stage time from CUDA-event nodes in the step graph: it includes the "
                        "device barriers and owner-side copies enqueued with the row kernel; "
                        "the row kernels' own spans are alltoall.row_kernels"}
    if fused:
        # the layout / reverse stages ARE the NVLink dispatch / combine (the
        # "reverse" and "a2a_dispatch" marks are empty stages: event resolution)
        roof["per_kernel_gbs"] = {
            "gate": None if fused_gl else ab["gate"] / (stage_ms["gate"] / 1e3) / 1e9,
            "k_layout (peer dispatch), NVLink per direction":
                ab["a2a_dispatch"] / (stage_ms["layout"] / 1e3) / 1e9,
            "k_reverse_k (peer combine), NVLink per direction":
                ab["a2a_combine"] / (stage_ms["a2a_combine"] / 1e3) / 1e9}
    else:
        roof["per_kernel_gbs"] = {
            "gate": None if fused_gl else ab["gate"] / (stage_ms["gate"] / 1e3) / 1e9,
            "layout": ab["layout"] / (stage_ms["layout"] / 1e3) / 1e9,
            "reverse": ab["reverse"] / (stage_ms["reverse"] / 1e3) / 1e9}
    a2a = None
    if P > 1:
        if fused:
            bw = {"dispatch (fused with layout)": ab["a2a_dispatch"] / (stage_ms["layout"] / 1e3) / 1e9,
                  "combine (fused with reverse)":
                      ab["a2a_combine"] / (stage_ms["a2a_combine"] / 1e3) / 1e9}
        else:
            bw = {s_: ab["a2a"] / (stage_ms[s_] / 1e3) / 1e9 for s_ in ("a2a_dispatch", "a2a_combine")}
        a2a = {"bytes_out_per_rank": ab["a2a"], "busbw_gbs": bw, "peak_gbs": NVLINK_GBS,
               "p2p": p2p_flags if algo == "p2p" else None,
               "algo": algo, "group_size": G if algo in ("hier", "hier2d") else None}
        if "a2a_buffer" in ab:
            a2a["buffer_bytes_per_rank"] = ab["a2a_buffer"]
            a2a["dispatch_bytes_per_rank"] = ab["a2a_dispatch"]
            a2a["combine_bytes_per_rank"] = ab["a2a_combine"]
            a2a["note"] = ("bytes that cross NVLink per rank and direction: the dispatch sends a "
                           "token's row once per remote owner (dedupe) plus the padding rows the "
                           "owners do not write themselves; the combine reads every admitted "
                           "remote slot, a token's two slots on one remote owner as the one row "
                           "that owner pre-combined after its expert (entry barrier kept, as "
                           "with a real expert)")
        a2a["frac"] = min(bw.values()) / NVLINK_GBS
        if kernel_spans and "a2a_buffer" in ab and min(kernel_spans.values()) > 0:
            # (the fused gate + dispatch kernel keeps its own trace format: no
            # per-CTA dispatch span there, so no row-kernel figure)
            # the same bytes over the row kernels' own spans (max over ranks)
            kg = {"dispatch": ab["a2a_dispatch"] / (kernel_spans["dispatch_us"] / 1e6) / 1e9,
                  "combine": ab["a2a_combine"] / (kernel_spans["combine_us"] / 1e6) / 1e9}
            a2a["row_kernels"] = {
                "span_us": kernel_spans, "gbs": kg, "frac": min(kg.values()) / NVLINK_GBS,
                "what": "bytes that cross over the dispatch / combine kernel's own span (first "
                        "CTA released -> last CTA end, moe_set_trace, one traced replay, max "
                        "over ranks): the link rate of the row kernels; the stage figures above "
                        "add the device barriers and the owners' duplicate-row copies"}
        if alias_ms is not None:
            a2a["identity_alias"] = {
                "ms_per_step": alias_ms, "value": P * S / (alias_ms / 1e3),
                "combine_bytes_per_rank": ab["a2a_combine_alias"],
                "what": "extra, not the headline: the same step with an identity expert "
                        "declared to the combine (MOE_P2P_RECV_UNMODIFIED: no entry barrier, a "
                        "row sent once for two slots read once)"}

    # ---- CPU baseline: the oracle, rank 0, N=1 only, bounded sample
    cpu = None
    if rank == 0 and P == 1 and not a.no_cpu_baseline:
        import oracle
        S_s = cpu_sample(w, 1, a.cpu_seconds)
        capo = oracle.capacity(S_s, w.E, w.k, w.C)
        inputs = [synthgen.workload_inputs(w, 0, S=S_s)]
        try:
            aff = os.sched_getaffinity(0)
            os.sched_setaffinity(0, {sorted(aff)[0]})
        except Exception:
            aff = None
        oracle_step(oracle, w, inputs, capo, 1)
        n, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < a.cpu_seconds or n < 2:
            oracle_step(oracle, w, inputs, capo, 1)
            n += 1
        dtc = (time.perf_counter() - t0) / n
        if aff:
            os.sched_setaffinity(0, aff)
        cpu = {"value": S_s / dtc, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": "%d oracle steps (gate+layout+reverse, AllToAll identity at P=1) on "
                         "%d of %d tokens of %s, single thread pinned to one core; %d host cores "
                         "present" % (n, S_s, w.S, w.name, os.cpu_count()),
               "cpu_model": cpu_model()}

    # our kernels per step: gate (k_gate_select, k_gate_scan, k_gate_slots),
    # layout, reverse; on hierarchical leaders one chunk permute per AllToAll,
    # with the two-level form two transposes per AllToAll on every rank; on
    # the one-sided path the barriers (dispatch exit, combine entry, and the
    # combine's exit unless the pipeline alternates two receive buffers), the
    # owners' duplicate-row copies (dedupe) and padding fill
    import ctypes
    from paper_2203_14685_b200._lib import lib as _moelib
    gate_k = _moelib().moe_gate_kernel_count(ctypes.byref(pipe.routing.desc()), 1)
    if a.dropless:
        # gate + expert offsets + (P=1: packed layout, packed reverse;
        # P>1: counts, barrier, plan, layout, exit barrier, reverse, exit barrier)
        launches_per_step = gate_k + 1 + (7 if P > 1 else 2)
    else:
        launches_per_step = (1 if fused_gl else gate_k + 1) + 1
        if P > 1 and algo == "hier" and rank % G == 0:
            launches_per_step += 2
        elif P > 1 and algo == "hier2d":
            launches_per_step += 4
        elif P > 1 and algo == "p2p":
            launches_per_step += (2 + (0 if pipe.double_buffered else 1) +
                                  int(p2p_flags["dedupe"]) + int(p2p_flags["local_pad"]) +
                                  int(p2p_flags["precombine"]))
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": P, "steps": a.steps,
            "warmup": max(3, a.warmup), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": w.dtype,
            "data": "synthetic (synthgen: seeded N(0,1) logits/tokens, no near ties)",
            "config": {"workload": w.name, "desc": w.note, "S_per_rank": S, "d": w.d, "E": w.E,
                       "k": w.k, "gate": w.kind, "capacity_factor": w.C, "capacity": cap,
                       "a2a": algo if P > 1 else None,
                       "layout_form": "packed dropless (NEXT-4)" if a.dropless else "padded [E,cap,d]",
                       "parallelism": "ep%d (experts sharded, tokens data-parallel)" % P,
                       "l2": "flushed between timed steps (2x L2 memset + 2x L2 read, outside events)",
                       "expert": "identity in the timed step; s_e stand-in timed separately",
                       "gate_layout": "one fused kernel" if fused_gl else "separate kernels"},
            "stages_ms": stage_ms, "expert_ms": expert_ms, "min_ms_per_step": float(vals[-2]),
            "eager_ms_per_step": float(vals[-1]),
            "timing": "CUDA-graph replay of the whole step (events outside the graph); stages_ms "
                      "from event-record nodes inside the step graph",
            "admitted_slots": admitted, "roofline": roof, "alltoall": a2a, "clocks": clocks,
            "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches_per_step * a.steps,
            "backward": bwd,
            "library": moe.version(), "gpu": torch.cuda.get_device_name(dev),
        }
        print(json.dumps(out), flush=True)
    # CUDA graphs that captured NCCL work must go before the communicator
    del g_step, g_timed
    torch.cuda.synchronize()
    barrier()
    if comm is not None:
        comm.destroy()
    if P > 1:
        dist.destroy_process_group()


def _json_stdout():
    """Keep stdout for the ONE JSON line: native libraries (NCCL's version
    banner, ...) print to fd 1, so fd 1 is pointed at stderr and the JSON is
    written to a saved duplicate of the original stdout."""
    sys.stdout.flush()
    real = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(real, "w")


if __name__ == "__main__":
    rc = relaunch_if_needed()
    if rc is not None:
        sys.exit(rc)
    _json_stdout()
    main()
