#!/usr/bin/env python
"""Run the N=1 routing step of a workload a few times (eager, no timing):
the target of `ncu -k regex:...` captures (B200_PROFILING.md).

    python tools/prof_step.py [--workload C2] [--iters 4] [--no-fuse]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_14685_b200 as moe  # noqa: E402
import synthgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--fuse", action="store_true")
    ap.add_argument("--tile", type=int, default=0, help="tuning gate_max_tile")
    a = ap.parse_args()
    if a.tile:
        moe.set_tuning(gate_max_tile=a.tile)
    w = synthgen.WORKLOADS[a.workload]
    S = w.S
    cap = moe.capacity(S, w.E, w.k, w.C)
    dt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    pipe = moe.RoutePipeline(S, w.d, w.E, w.k, cap, dt, w.kind, fuse_gate_layout=True if a.fuse else (False if a.no_fuse else None))
    lg, ids, table, x = synthgen.workload_inputs(w, 0)

    def dev(v):
        if v is None:
            return None
        t = torch.from_numpy(np.ascontiguousarray(v))
        if v.dtype == np.uint16:
            t = t.view(torch.int16).view(torch.bfloat16)
        return t.cuda()

    d = [dev(v) for v in (lg, x, ids, table)]
    for _ in range(a.iters):
        pipe.step(d[0], d[1], d[2], d[3])
    torch.cuda.synchronize()
    print("ok", a.workload, "fused" if pipe.fuse else "separate")


if __name__ == "__main__":
    main()
