#!/usr/bin/env python
"""Timeline of the one-sided NVLink step's row kernels on every rank (run
under torch.distributed.run, one rank per GPU): moe_set_trace stamps per CTA
of the dispatch (k_layout in peer mode) and of the combine (k_reverse_k in
peer mode) inside a CUDA-graph replay of RoutePipeline.step, ranks aligned
by a device barrier and the L2 flushed before each replay.  Reports each
kernel's span (first wait released -> last CTA end) and the spread of its
CTAs' ends, per rank, and the bytes each rank sends / reads over NVLink.

    python -m torch.distributed.run --nproc-per-node 2 tools/trace_p2p.py [--workload C2]
    (MOE_P2P_DEDUPE=0 to send every row)
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
from paper_2203_14685_b200._lib import lib  # noqa: E402
import synthgen  # noqa: E402


def pct(v):
    v = np.asarray(v, dtype=np.float64)
    return {q: round(float(np.percentile(v, q)), 2) for q in (0, 10, 50, 90, 100)} if v.size else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="")
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

    d = [dev(v) for v in (lg, x, ids, table)]
    for _ in range(3):
        pipe.step(*d)
    torch.cuda.synchronize()
    buf = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")
    lib().moe_set_trace(buf.data_ptr(), buf.numel() * 8)
    g = pipe.capture(*d)
    lib().moe_set_trace(None, 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    runs = []
    for _ in range(a.reps):
        flush.zero_()
        buf.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        comm.barrier()
        g.replay()
        torch.cuda.synchronize()
        raw = buf.cpu().numpy().copy()
        n = raw.size
        r = {}
        for name, lo in (("dispatch", n // 2), ("combine", 3 * n // 4)):
            c = raw[lo:lo + n // 4].reshape(-1, 4)[:, :3].astype(np.float64)
            c = c[c[:, 0] > 0]
            r[name] = c
        t0 = min(r["dispatch"][:, 0].min(), r["combine"][:, 0].min())
        out = {}
        for name, c in r.items():
            out[name] = {"ctas": int(c.shape[0]),
                         "span_us": round(float((c[:, 2].max() - c[:, 1].min()) / 1e3), 2),
                         "wait_released_us": round(float((c[:, 1].min() - t0) / 1e3), 2),
                         "cta_end_us": pct((c[:, 2] - t0) / 1e3)}
        runs.append(out)
    # NVLink bytes of this rank (as bench.py counts them)
    El = w.E // P
    rt = pipe.routing
    ex, sl = rt.expert_idx.view(S, w.k), rt.slot_idx.view(S, w.k)
    adm = (ex >= 0) & (sl >= 0)
    own = torch.where(adm, ex // El, torch.full_like(ex, -1))
    remote_slots = int((adm & (own != rank)).sum().item())
    owners = torch.zeros((S, P), dtype=torch.bool, device=own.device)
    for j in range(w.k):
        m = own[:, j] >= 0
        owners[torch.nonzero(m).squeeze(1), own[m, j].long()] = True
    owners[:, rank] = False
    row = w.d * 2
    res = {"rank": rank, "workload": w.name, "P": P, "dedupe": moe.get_tuning()["p2p_dedupe"],
           "remote_rows_sent": int(owners.sum().item()) if moe.get_tuning()["p2p_dedupe"] and w.k >= 2
           else remote_slots, "remote_slots_read": remote_slots, "row_bytes": row,
           "dispatch_span_us": [o["dispatch"]["span_us"] for o in runs],
           "combine_span_us": [o["combine"]["span_us"] for o in runs], "last": runs[-1]}
    allres = [None] * P
    dist.all_gather_object(allres, res)
    if rank == 0:
        print(json.dumps(allres, indent=1))
        if a.out:
            json.dump(allres, open(a.out, "w"), indent=1)
    del g
    torch.cuda.synchronize()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
