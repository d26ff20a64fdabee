#!/usr/bin/env python
"""E3 micro-bench (PAPER.md:108-121, 170-171 -- Fig. 3 "Topk kernel
performance comparison with PyTorch", swept over #experts and #tokens):
moe_gate (selection + fp64 weights + capacity slots, 2-3 PDL-chained kernels) against
torch.topk + softmax of the selected logits (selection and weights only, no
capacity), both replayed from CUDA graphs, L2 flushed between replays.

    python tools/bench_gate.py [--k 2] [--out profiles/gate_vs_torch.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2203_14685_b200 as moe  # noqa: E402
import synthgen  # noqa: E402


def graph_time(fn, flush, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "gate_vs_torch.json"))
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for E in (2, 4, 8, 16, 32, 64, 128):
        for S in (1024, 4096, 16384, 65536):
            k = min(a.k, E)
            lg = torch.from_numpy(synthgen.logits(E * 1000 + S, S, E, k)).cuda()
            cap = moe.capacity(S, E, k, 1.0)
            g = moe.Gate(S, E, k, cap)
            out = moe.Routing.empty(S, E, k, cap, "cuda")
            t_ours = graph_time(lambda: g(lg, out=out), flush)

            def torch_gate():
                v, i = torch.topk(lg, k, dim=1)
                return torch.softmax(v, dim=1), i
            t_torch = graph_time(torch_gate, flush)
            rows.append({"E": E, "S": S, "k": k, "moe_gate_us": t_ours, "torch_topk_softmax_us": t_torch,
                         "speedup": t_torch / t_ours})
            print(json.dumps(rows[-1]), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
