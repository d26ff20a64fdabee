#!/usr/bin/env python
"""Timeline of the fused gate + layout kernel (moe_set_trace): when each
gate tile is claimed / publishes its aggregate / resolves its prefix / is
ready, when each 32-token scatter chunk is claimed and how long it waits for
its tile, and each CTA's start and end -- all from %globaltimer, relative to
the first CTA's start.  Needs a GPU.

    python tools/trace_gate_layout.py [--workload C2] [--out FILE.json]
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


def pct(v):
    v = np.asarray(v, dtype=np.float64)
    if v.size == 0:
        return None
    return {q: round(float(np.percentile(v, q)), 2) for q in (0, 10, 50, 90, 100)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    w = synthgen.WORKLOADS[a.workload]
    S = w.S
    cap = moe.capacity(S, w.E, w.k, w.C)
    dt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    pipe = moe.RoutePipeline(S, w.d, w.E, w.k, cap, dt, w.kind, fuse_gate_layout=True)
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
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush.zero_()
    pipe.step(d[0], d[1], d[2], d[3])
    torch.cuda.synchronize()
    lib().moe_set_trace(None, 0)
    raw = buf.cpu().numpy()
    n_tiles, n_chunks, n_ctas = int(raw[0]), int(raw[1]), int(raw[2])
    t = raw[4:].astype(np.float64)
    tiles = t[:4 * n_tiles].reshape(n_tiles, 4)
    chunks = t[4 * n_tiles:4 * n_tiles + 2 * n_chunks].reshape(n_chunks, 2)
    ctas = t[4 * n_tiles + 2 * n_chunks:4 * n_tiles + 2 * n_chunks + 2 * n_ctas].reshape(n_ctas, 2)
    t0 = ctas[:, 0].min()
    us = lambda v: (v - t0) / 1e3
    out = {
        "workload": w.name, "n_tiles": n_tiles, "n_chunks": n_chunks, "ctas": int(ctas.shape[0]),
        "kernel_us": float(us(ctas[:, 1].max())),
        "cta_start_us": pct(us(ctas[:, 0])), "cta_end_us": pct(us(ctas[:, 1])),
        "tile_claim_us": pct(us(tiles[:, 0])), "tile_aggregate_us": pct(us(tiles[tiles[:, 1] > 0, 1])),
        "tile_prefix_us": pct(us(tiles[:, 2])), "tile_ready_us": pct(us(tiles[:, 3])),
        "tile_gate_us (claim->aggregate)": pct((tiles[tiles[:, 1] > 0, 1] - tiles[tiles[:, 1] > 0, 0]) / 1e3),
        "tile_lookback_us (aggregate->prefix)": pct((tiles[tiles[:, 1] > 0, 2] - tiles[tiles[:, 1] > 0, 1]) / 1e3),
        "tile_finalize_us (prefix->ready)": pct((tiles[:, 3] - tiles[:, 2]) / 1e3),
        "chunk_claim_us": pct(us(chunks[chunks[:, 0] > 0, 0])),
        "chunk_wait_us": pct((chunks[chunks[:, 0] > 0, 1] - chunks[chunks[:, 0] > 0, 0]) / 1e3),
        "ready_by_tile_decile_us": [round(float(us(tiles[int(i), 3])), 2)
                                    for i in np.linspace(0, n_tiles - 1, 11)],
    }
    print(json.dumps(out, indent=1))
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
