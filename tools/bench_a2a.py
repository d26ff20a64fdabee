#!/usr/bin/env python
"""C5 sweep (BASELINE.json configs[4]; Figs. 5-7):
flat vs hierarchical (group aggregate-then-exchange) AllToAll through
moe_alltoall, per-rank payload B = 1 MiB .. 1 GiB, on N GPUs of one box.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/bench_a2a.py [--group-size G] [--max-mib 1024] [--out FILE]

Every rank fills its send buffer with the closed-form pattern
w = (src << 20) ^ (dst << 12) ^ (i & 0xfff) (int32 words, chunk dst of rank
src); after each collective the receiver checks recv chunk q == pattern(q, r)
on the device (no oracle needed).  Times are CUDA events around
a CUDA-graph replay of one collective, max over ranks; busBW = B (P-1)/P / t.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2203_14685_b200 as moe  # noqa: E402


def pattern(src, dst, n_words, device):
    i = torch.arange(n_words, dtype=torch.int32, device=device)
    return ((src << 20) ^ (dst << 12)) ^ (i & 0xFFF)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--group-size", type=int, default=0)
    ap.add_argument("--max-mib", type=int, default=1024)
    ap.add_argument("--min-mib", type=int, default=1)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="")
    ap.add_argument("--p2p", action="store_true", help="also time the one-sided NVLink AllToAll")
    ap.add_argument("--algos", default="flat,hier",
                    help="comma list of flat, flat_reg (NCCL-registered ncclMemAlloc buffers), "
                         "a2a (ncclAlltoAll), a2a_reg, hier (leader), hier2d (two-level), p2p")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("cpu:gloo,cuda:nccl", device_id=dev)
    P, r = dist.get_world_size(), dist.get_rank()
    G = a.group_size or max(1, P // 2)
    comm = moe.Comm.from_process_group()
    rows = []
    mib = a.min_mib
    while mib <= a.max_mib:
        B = mib << 20
        chunk_words = B // 4 // P
        send = torch.cat([pattern(r, q, chunk_words, dev) for q in range(P)])
        recv = torch.empty_like(send)
        recv_sym = comm.symm_empty(send.shape, send.dtype) if (a.p2p or "p2p" in a.algos) else None
        ws = torch.empty(comm.workspace_bytes("hier", G, B // P) if r % G == 0 else 0,
                         dtype=torch.uint8, device=dev)
        res = {"B_mib": mib, "P": P, "G": G, "per_peer_bytes": B // P}
        algos = [x for x in a.algos.split(",") if x] + (["p2p"] if a.p2p and "p2p" not in a.algos else [])
        reg = None
        if any(x.endswith("_reg") for x in algos):
            reg = (comm.mem_empty(send.shape, send.dtype), comm.mem_empty(send.shape, send.dtype))
            reg[0].copy_(send)
        if "hier2d" in algos:
            ws2 = torch.empty(comm.workspace_bytes("hier2d", G, B // P), dtype=torch.uint8, device=dev)
        for name in algos:
            algo = {"flat_reg": "flat", "a2a": "flat", "a2a_reg": "flat"}.get(name, name)
            moe.set_tuning(nccl_alltoall=1 if name.startswith("a2a") else 0)
            sd = reg[0] if name.endswith("_reg") else send
            rv = recv_sym if algo == "p2p" else (reg[1] if name.endswith("_reg") else recv)
            w_ = ws2 if algo == "hier2d" else ws
            rv.fill_(-1)
            comm.alltoall(sd, rv, algo, G, w_)        # eager warm-up + check
            torch.cuda.synchronize()
            want = torch.cat([pattern(q, r, chunk_words, dev) for q in range(P)])
            ok = torch.tensor([1 if torch.equal(rv, want) else 0], device=dev)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    comm.alltoall(sd, rv, algo, G, w_)
            torch.cuda.current_stream().wait_stream(s)
            ts = []
            for _ in range(a.reps):
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            rv.fill_(-1)
            dist.barrier()
            g.replay()
            torch.cuda.synchronize()
            ok &= torch.tensor([1 if torch.equal(rv, want) else 0], device=dev)
            t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            ms = float(t.item())
            res[name] = {"ms": ms, "busbw_gbs": B * (P - 1) / P / (ms / 1e3) / 1e9,
                         "correct": bool(ok.item())}
            del g
        moe.set_tuning(nccl_alltoall=0)
        for name in algos:
            if name != "flat" and "flat" in res:
                res["t_flat_over_t_" + name] = res["flat"]["ms"] / res[name]["ms"]
        dist.barrier()
        torch.cuda.synchronize()
        if recv_sym is not None:
            comm.symm_free(recv_sym)
        if reg is not None:
            comm.mem_free(reg[0])
            comm.mem_free(reg[1])
        rows.append(res)
        if r == 0:
            print(json.dumps(res), flush=True)
        del send, recv, ws, recv_sym, reg
        torch.cuda.empty_cache()
        mib *= 2
    if r == 0 and a.out:
        json.dump(rows, open(a.out, "w"), indent=1)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
