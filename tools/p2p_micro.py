#!/usr/bin/env python
"""Where the one-sided NVLink step's time goes (run under
torch.distributed.run, one rank per GPU): each piece of the C2-shaped step
captured alone in a CUDA graph and timed with CUDA events (ranks aligned by
a device barrier outside the events, L2 flushed, median of 20, max over
ranks): a device barrier, the dispatch rows alone (no barriers), the dispatch
with its exit barrier and duplicate copies, the combine reads alone, the
combine with its barriers, a contiguous one-sided AllToAll of the same bytes,
and the whole step.

    python -m torch.distributed.run --nproc-per-node 2 tools/p2p_micro.py [--workload C2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2203_14685_b200 as moe  # noqa: E402
import synthgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--barrier-pdl", action="store_true",
                    help="also time the barrier-heavy pieces with PDL-launched barriers")
    ap.add_argument("--variants", action="store_true",
                    help="also time the row kernels under other tuning values")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    P, rank = dist.get_world_size(), dist.get_rank()
    comm = moe.Comm.from_process_group()
    w = synthgen.WORKLOADS[a.workload]
    S, cap = w.S, moe.capacity(w.S, w.E, w.k, w.C)
    pipe = moe.RoutePipeline(S, w.d, w.E, w.k, cap, torch.bfloat16, w.kind, comm=comm, algo="p2p")
    lg, ids, table, x = synthgen.workload_inputs(w, rank)

    def dev(v):
        if v is None:
            return None
        t = torch.from_numpy(np.ascontiguousarray(v))
        if v.dtype == np.uint16:
            t = t.view(torch.int16).view(torch.bfloat16)
        return t.cuda()

    lg_d, x_d, ids_d, tb_d = dev(lg), dev(x), dev(ids), dev(table)
    for _ in range(3):
        pipe.step(lg_d, x_d, ids_d, tb_d)
    torch.cuda.synchronize()
    r = pipe.routing
    y = pipe.y
    NE, NX = comm.NO_ENTRY_BARRIER, comm.NO_EXIT_BARRIER
    send = torch.empty_like(pipe.recv)
    a2a_recv = comm.symm_empty(tuple(pipe.recv.shape), pipe.recv.dtype)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    pieces = {
        "barrier": lambda: comm.barrier(),
        "dispatch_rows_only": lambda: comm.dispatch_p2p(x_d, r, pipe.recv, flags=NE | NX),
        "dispatch_with_exit": lambda: comm.dispatch_p2p(x_d, r, pipe.recv, flags=NE),
        "combine_reads_only": lambda: comm.combine_p2p(pipe.recv, r, y, flags=NE | NX),
        "combine_with_barriers": lambda: comm.combine_p2p(pipe.recv, r, y, flags=0),
        "a2a_p2p_contiguous": lambda: comm.alltoall(send, a2a_recv, "p2p"),
        "gate": lambda: pipe.gate(lg_d, ids_d, tb_d, out=r),
        "step": lambda: pipe.step(lg_d, x_d, ids_d, tb_d),
    }
    out = {"P": P, "workload": w.name, "recv_bytes": pipe.recv.numel() * 2}
    runs = [("", {}, pieces)]
    if a.barrier_pdl:   # the step and the barrier-heavy pieces with PDL-launched barriers
        bar = {k: pieces[k] for k in ("barrier", "dispatch_with_exit", "combine_with_barriers",
                                      "step")}
        runs.append(("@bpdl", {"barrier_pdl": 1}, bar))
    if a.variants:
        rows = {k: pieces[k] for k in ("dispatch_rows_only", "dispatch_with_exit",
                                       "combine_reads_only")}
        for tag, tu in (("u4", {"layout_u": 4}), ("u1", {"layout_u": 1}),
                        ("cta8", {"row_ctas_per_sm": 8}), ("cta3", {"row_ctas_per_sm": 3}),
                        ("ccta6", {"combine_ctas_per_sm": 6}), ("ccta8", {"combine_ctas_per_sm": 8}),
                        ("ccta12", {"combine_ctas_per_sm": 12}), ("ccta16", {"combine_ctas_per_sm": 16}),
                        ("ku2", {"reverse_ku": 2}), ("nodedupe", {"p2p_dedupe": 0}),
                        ("rev", {"reverse_backwards": 1})):
            runs.append(("@" + tag, tu, rows))
    for tag, tu, group in runs:
        old_t = moe.set_tuning(**tu)
        _time_pieces(group, tag, out, comm, flush, a.reps)
        moe.set_tuning(**old_t)
    if rank == 0:
        print(json.dumps(out), flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


def _time_pieces(pieces, tag, out, comm, flush, reps):
    for name, fn in pieces.items():
        fn()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            comm.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        t = torch.tensor([float(np.median(ts))], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[name + tag + "_us"] = round(float(t[0]), 2)
        del g


if __name__ == "__main__":
    main()
