"""Copy-engine NVLink ceiling in one process: cudaMemcpyPeerAsync (torch
copy_ between devices) one direction, both directions at once, and (with 4
GPUs) every GPU to every other.  GB/s per sending GPU, CUDA events."""
import json

import torch


def run(pairs, nb, iters=10, reps=1):
    n = torch.cuda.device_count()
    src = {i: torch.empty(nb, dtype=torch.uint8, device=i) for i in range(n)}
    dst = {(i, j): torch.empty(nb, dtype=torch.uint8, device=j) for (i, j) in pairs}
    streams = {(i, j): torch.cuda.Stream(device=i) for (i, j) in pairs}
    best = 1e30
    for it in range(iters + 2):
        for i in range(n):
            torch.cuda.synchronize(i)
        ev = {}
        for (i, j) in pairs:
            s = streams[(i, j)]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            with torch.cuda.stream(s):
                for _ in range(reps):
                    dst[(i, j)].copy_(src[i], non_blocking=True)
            e1.record(s)
            ev[(i, j)] = (e0, e1)
        for i in range(n):
            torch.cuda.synchronize(i)
        t = max(a.elapsed_time(b) for a, b in ev.values()) * 1e3 / reps
        if it >= 2:
            best = min(best, t)
    sends = {}
    for (i, j) in pairs:
        sends[i] = sends.get(i, 0) + nb
    return {"us": round(best, 1), "GBs_per_sender": round(max(sends.values()) / best / 1e3, 1)}


def main():
    n = torch.cuda.device_count()
    out = {"gpus": n}
    for i in range(n):
        for j in range(n):
            if i != j:
                torch.cuda.set_device(i)
                try:
                    torch.cuda.memory  # noqa
                except Exception:
                    pass
    for mb in (64, 256):
        nb = mb << 20
        out["uni_%dM" % mb] = run([(0, 1)], nb)
        out["bi_%dM" % mb] = run([(0, 1), (1, 0)], nb)
        out["bi_%dM_x10" % mb] = run([(0, 1), (1, 0)], nb, reps=10)
        if n >= 4:
            out["a2a4_%dM" % mb] = run([(i, j) for i in range(4) for j in range(4) if i != j], nb // 3)
    out["can_p2p"] = torch.cuda.can_device_access_peer(0, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
