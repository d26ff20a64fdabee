#!/usr/bin/env python
"""Timeline of the N=1 routing step: the separate gate (k_gate_select ->
k_gate_slots2), the layout and the reverse (moe_set_trace): per tile, when the select CTA starts, passes
its grid-dependency wait, has its logits staged, finishes selection, the
in-tile ranks and the tile aggregate, and ends; when the slots2 CTA starts,
passes its wait, has reduced the prefixes and ends -- all from %globaltimer,
relative to the first select CTA's start.  The step runs as a CUDA graph
replay after an L2 flush, as bench.py times it.  Needs a GPU.

    python tools/trace_gate.py [--workload C2] [--out FILE.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_14685_b200 as moe  # noqa: E402
from paper_2203_14685_b200._lib import lib  # noqa: E402
import synthgen  # noqa: E402

SELECT = ["entry", "waited", "staged", "selected", "ranked", "aggregate", "end"]
SLOTS = ["entry", "waited", "reduced", "end"]  # slots2 (slots: no "reduced")


def pct(v):
    v = np.asarray(v, dtype=np.float64)
    if v.size == 0:
        return None
    return {q: round(float(np.percentile(v, q)), 2) for q in (0, 10, 50, 90, 100)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--out", default="")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    w = synthgen.WORKLOADS[a.workload]
    S = w.S
    cap = moe.capacity(S, w.E, w.k, w.C)
    dt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    pipe = moe.RoutePipeline(S, w.d, w.E, w.k, cap, dt, w.kind, fuse_gate_layout=False)
    lg, ids, table, x = synthgen.workload_inputs(w, 0)

    def dev(v):
        if v is None:
            return None
        t = torch.from_numpy(np.ascontiguousarray(v))
        if v.dtype == np.uint16:
            t = t.view(torch.int16).view(torch.bfloat16)
        return t.cuda()

    d = [dev(v) for v in (lg, x, ids, table)]
    for _ in range(3):
        pipe.step(d[0], d[1], d[2], d[3])
    torch.cuda.synchronize()
    buf = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")
    lib().moe_set_trace(buf.data_ptr(), buf.numel() * 8)
    g = pipe.capture(d[0], d[1], d[2], d[3])  # the graph keeps the trace buffer
    lib().moe_set_trace(None, 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    runs = []
    for _ in range(a.reps):
        flush.zero_()
        buf.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        runs.append(buf.cpu().numpy().copy())
    out = {"workload": w.name, "runs": []}
    for raw in runs:
        n_tiles, per, kind = int(raw[0]), int(raw[1]), int(raw[3])
        assert per == 16 and kind == 2, (per, kind)
        t = raw[4:4 + 16 * n_tiles].reshape(n_tiles, 16).astype(np.float64)
        t0 = t[:, 0].min()
        us = lambda v: (v - t0) / 1e3
        r = {"n_tiles": n_tiles}
        for i, name in enumerate(SELECT):
            r["select_" + name + "_us"] = pct(us(t[:, i]))
        for i, name in enumerate(SLOTS):
            if np.all(t[:, 8 + i] > 0):
                r["slots_" + name + "_us"] = pct(us(t[:, 8 + i]))
        r["select_phase_us"] = {f"{SELECT[i]}->{SELECT[i + 1]}": pct((t[:, i + 1] - t[:, i]) / 1e3)
                                for i in range(len(SELECT) - 1)}
        if np.all(t[:, 10] > 0):  # select -> slots2
            r["slots2_phase_us"] = {f"{SLOTS[i]}->{SLOTS[i + 1]}": pct((t[:, 9 + i] - t[:, 8 + i]) / 1e3)
                                    for i in range(len(SLOTS) - 1)}
        else:  # select -> scan -> slots
            sc = t[t[:, 12] > 0]
            r["scan_entry_us"] = pct(us(sc[:, 12]))
            r["scan_waited_us"] = pct(us(sc[:, 13]))
            r["scan_end_us"] = pct(us(sc[:, 14]))
        r["select_end_to_slots_waited_us"] = round(float((t[:, 9].min() - t[:, 6].max()) / 1e3), 2)
        r["gate_us"] = round(float(us(t[:, 11].max())), 2)
        n = raw.size
        for name, lo in (("layout", n // 2), ("reverse", 3 * n // 4)):
            c = raw[lo:lo + n // 4].reshape(-1, 4)[:, :3].astype(np.float64)
            c = c[c[:, 0] > 0]
            if c.size:
                r[name] = {"ctas": int(c.shape[0]), "first_entry_us": round(float(us(c[:, 0].min())), 2),
                           "first_waited_us": round(float(us(c[:, 1].min())), 2),
                           "last_waited_us": round(float(us(c[:, 1].max())), 2),
                           "end_us": pct(us(c[:, 2]))}
        if "layout" in r and "reverse" in r:
            lay, rev = r["layout"], r["reverse"]
            r["timeline_us"] = {
                "gate (first select entry -> last slots end)": r["gate_us"],
                "layout (first wait released -> last CTA end)":
                    round(lay["end_us"][100] - lay["first_waited_us"], 2),
                "reverse (first wait released -> last CTA end)":
                    round(rev["end_us"][100] - rev["first_waited_us"], 2),
                "step (first select entry -> last reverse end)": rev["end_us"][100],
            }
        out["runs"].append(r)
    print(json.dumps(out["runs"][-1], indent=1))
    print("timeline per run:", [r.get("timeline_us") or r["gate_us"] for r in out["runs"]])
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
