#!/usr/bin/env python
"""Per-phase timeline of k_gate (MOE_LIB_VARIANT=trace build): every CTA
stamps %globaltimer at 0 start, 1 logits staged, 2 selection done,
3 aggregates published, 4 look-back done, 5 end.  Prints, per phase, the
min / median / max over tiles of (stamp - earliest start), in microseconds.

    MOE_LIB_VARIANT=trace python tools/trace_gate.py [--workload C3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
assert os.environ.get("MOE_LIB_VARIANT") == "trace", "run with MOE_LIB_VARIANT=trace"

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_14685_b200 as moe  # noqa: E402
import synthgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C3")
a = ap.parse_args()
w = synthgen.WORKLOADS[a.workload]
lg, ids, table, _ = synthgen.workload_inputs(w, 0)
cap = moe.capacity(w.S, w.E, w.k, w.C)
g = moe.Gate(w.S, w.E, w.k, cap, w.kind)
dev = lambda v: None if v is None else torch.from_numpy(v).cuda()
args = (dev(lg), dev(ids), dev(table))
out = moe.Routing.empty(w.S, w.E, w.k, cap, "cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(4):
    flush.zero_()
    g(*args, out=out)
torch.cuda.synchronize()
ws = g.ws.cpu().numpy()
# tile plan of gate.cu (gate_plan): >= 256 tiles of 32..256 tokens, <= 2048
# items and <= 64 KiB of staged logits per tile
tt = 256
while tt > 32 and (w.S + tt - 1) // tt < 256:
    tt //= 2
while tt > 1 and tt * w.k > 2048:
    tt //= 2
if w.kind != "hash":
    while tt > 1 and tt * w.E * 4 > 65536:
        tt //= 2
n_tiles = (w.S + tt - 1) // tt
tr = ws.view(np.uint64)[-n_tiles * 8:].reshape(n_tiles, 8).astype(np.int64)
tr = tr[:, :6]
t0 = tr[:, 0].min()
rel = (tr - t0) / 1e3
names = ["start", "staged", "selected", "agg published", "look-back done", "end"]
print("workload", w.name, "tiles", n_tiles, "kernel span %.1f us" % (rel[:, 5].max()))
for k, nm in enumerate(names):
    print("%-16s min %7.2f  med %7.2f  max %7.2f us" % (nm, rel[:, k].min(), np.median(rel[:, k]),
                                                       rel[:, k].max()))
d = np.diff(rel, axis=1)
for k in range(5):
    print("  %-14s -> %-16s med %6.2f max %6.2f us" % (names[k], names[k + 1], np.median(d[:, k]),
                                                      d[:, k].max()))
