"""Backward-only driver for profiling (ncu) and timing the adjoint kernels
of one workload on one GPU: one forward step, then --iters backward passes
(combine adjoint, layout adjoint, gate adjoint), each timed with CUDA events
after an L2 flush.  Prints one JSON line with per-kernel-call device times.

    python tools/bench_bwd.py --workload C2 --iters 10
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2203_14685_b200 as moe  # noqa: E402
import synthgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    w = synthgen.WORKLOADS[a.workload]
    dt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    cap = moe.capacity(w.S, w.E, w.k, w.C)
    pipe = moe.RoutePipeline(w.S, w.d, w.E, w.k, cap, dt, w.kind)
    lg, ids, table, x = synthgen.workload_inputs(w, 0)

    def d(a_):
        if a_ is None:
            return None
        t = torch.from_numpy(a_)
        if a_.dtype.name == "uint16":
            t = t.view(torch.int16).view(torch.bfloat16)
        return t.cuda()
    lg_d, x_d = d(lg), d(x)
    pipe.step(lg_d, x_d, d(ids), d(table))
    dy = d(synthgen.tokens(7, w.S, w.d, w.dtype))
    nb = 2 * torch.cuda.get_device_properties(0).L2_cache_size
    flush = torch.empty(nb, dtype=torch.uint8, device="cuda")
    flush_rd = torch.zeros(nb // 8, dtype=torch.int64, device="cuda")
    sink = torch.empty((), dtype=torch.int64, device="cuda")
    r = pipe.routing
    pipe.backward(dy, lg_d)
    torch.cuda.synchronize()
    parts = {"combine_bwd": lambda: moe.reverse_layout_backward(dy, pipe.back, r, pipe.d_back,
                                                                pipe.d_weight),
             "layout_bwd": lambda: moe.layout_backward(pipe.d_disp, r, out=pipe.dx)}
    if lg_d is not None:
        parts["gate_bwd"] = lambda: moe.gate_backward(lg_d, r, pipe.d_weight, out=pipe.d_logits)
    out = {}
    for name, fn in parts.items():
        ts = []
        for _ in range(a.iters):
            flush.zero_()                              # evict, then read so L2 is clean
            torch.sum(flush_rd, dim=0, out=sink)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        out[name + "_us"] = statistics.median(ts)
    row = w.d * (2 if w.dtype == "bf16" else 4)
    adm = int((r.slot_idx >= 0).sum().item())
    out["algorithmic_bytes"] = {
        "combine_bwd": w.S * row + adm * row + w.E * cap * row + 16 * w.S * w.k,
        "layout_bwd": adm * row + w.S * row + 8 * w.S * w.k,
        "gate_bwd": 8 * w.S * w.E + 12 * w.S * w.k}
    out["gbs"] = {k: out["algorithmic_bytes"][k] / out[k + "_us"] / 1e3
                  for k in parts}
    out["workload"] = w.name
    print(json.dumps(out))


if __name__ == "__main__":
    main()
