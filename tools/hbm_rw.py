"""HBM write-only / read-only / copy rates at the layout's sizes (torch
kernels, CUDA events, L2 flushed before each timed op).  Context for the
layout's roofline: is 128 MiB of scattered row writes write-bound?"""
import json

import torch


def flush(buf, buf2):
    buf.zero_()
    buf2.sum()


def timed(fn, iters=10):
    a = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    b = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for it in range(iters + 3):
        flush(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[len(ts) // 2]


def main():
    out = {}
    for mb in (64, 128, 512, 2048):
        nb = mb << 20
        w = torch.empty(nb, dtype=torch.uint8, device="cuda")
        us = timed(lambda: w.fill_(1))
        out["write_%dM" % mb] = {"us": round(us, 1), "GBs": round(nb / us / 1e3)}
        r = torch.ones(nb // 4, dtype=torch.float32, device="cuda")
        s = torch.empty((), dtype=torch.float32, device="cuda")
        us = timed(lambda: torch.sum(r, dim=0, out=s))
        out["read_%dM" % mb] = {"us": round(us, 1), "GBs": round(nb / us / 1e3)}
        src = torch.ones(nb // 2, dtype=torch.uint8, device="cuda")
        dst = torch.empty(nb // 2, dtype=torch.uint8, device="cuda")
        us = timed(lambda: dst.copy_(src))
        out["copy_%dM_rw" % mb] = {"us": round(us, 1), "GBs": round(nb / us / 1e3)}
        src2 = torch.ones(nb // 3, dtype=torch.uint8, device="cuda")
        dst2 = torch.empty(2 * (nb // 3), dtype=torch.uint8, device="cuda").view(2, -1)
        us = timed(lambda: dst2.copy_(src2.expand(2, -1)))
        out["dup2_%dM_rw" % mb] = {"us": round(us, 1), "GBs": round(3 * (nb // 3) / us / 1e3)}
        del w, r, src, dst, src2, dst2
    print(json.dumps(out))


if __name__ == "__main__":
    main()
