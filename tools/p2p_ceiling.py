"""NVLink ceiling for SM-driven one-sided copies at N ranks: the contiguous
P2P AllToAll (k_a2a_p2p: every rank stores its chunk into every peer's
symmetric buffer) at several CTA counts, NCCL's AllToAll of the same bytes,
and the fused dispatch / combine of C2 alone.  GB/s = remote bytes one rank
sends (or pulls) / device time, max over ranks.  Run under
torch.distributed.run."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2203_14685_b200 as moe  # noqa: E402


def timed(fn, comm, iters=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        comm.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    t = torch.tensor([sorted(ts)[len(ts) // 2]], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def main():
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    comm = moe.Comm.from_process_group()
    out = {"P": P}
    for mb in (16, 64, 256):
        B = mb << 20                              # bytes per peer
        send = torch.empty(P * B, dtype=torch.uint8, device="cuda").random_(0, 255)
        recv = comm.symm_empty((P * B,), torch.uint8)
        remote = (P - 1) * B
        for cps in ((1, 2, 4, 8) if mb == 64 else (4, 8)):
            with moe.tuned(a2a_ctas_per_sm=cps):
                us = timed(lambda: comm.alltoall(send, recv, "p2p"), comm)
            out["a2a_p2p_%dM_cps%d" % (mb, cps)] = {"us": round(us, 1),
                                                   "GBs": round(remote / us / 1e3, 1)}
        if mb == 64:
            # back to back: is the fixed cost per copy, or per burst?
            us = timed(lambda: [comm.alltoall(send, recv, "p2p") for _ in range(10)], comm) / 10
            out["a2a_p2p_64M_x10"] = {"us": round(us, 1), "GBs": round(remote / us / 1e3, 1)}
            small_s, small_r = send[:P * 65536], recv[:P * 65536]

            def warm_then():
                comm.alltoall(small_s, small_r, "p2p")
                comm.alltoall(send, recv, "p2p")
            us = timed(warm_then, comm)
            out["a2a_p2p_64M_after_64K"] = {"us": round(us, 1), "GBs": round(remote / us / 1e3, 1)}
            us = timed(lambda: comm.alltoall(small_s, small_r, "p2p"), comm)
            out["a2a_p2p_64K"] = {"us": round(us, 1)}
            sleep = torch.cuda._sleep

            def idle_then():
                sleep(20000)
                comm.alltoall(send, recv, "p2p")
            us = timed(idle_then, comm)
            out["a2a_p2p_64M_after_sleep"] = {"us": round(us, 1)}

            def sleep_only():
                sleep(20000)
            us = timed(sleep_only, comm)
            out["sleep_only"] = {"us": round(us, 1)}
        recv2 = torch.empty_like(send)
        us = timed(lambda: comm.alltoall(send, recv2, "flat"), comm)
        out["a2a_nccl_%dM" % mb] = {"us": round(us, 1), "GBs": round(remote / us / 1e3, 1)}
        comm.symm_free(recv)
        del send, recv2
    # the fused stages of C2 alone (one rank's remote rows = (P-1)/P of 2 S k rows)
    S, d, E, k = 32768, 1024, 8, 2
    cap = moe.capacity(S, E, k, 1.0)
    g = torch.Generator(device="cuda").manual_seed(rank)
    lg = torch.randn((S, E), device="cuda", generator=g)
    x = torch.randn((S, d), device="cuda", generator=g).to(torch.bfloat16)
    r = moe.Gate(S, E, k, cap)(lg)
    buf = comm.symm_empty((P, E // P, cap, d), torch.bfloat16)
    rb = E * cap * d * 2 * (P - 1) / P
    for name, tu in (("default", {}), ("nodedupe", {"p2p_dedupe": 0})):
        with moe.tuned(**tu):
            us = timed(lambda: comm.dispatch_p2p(x, r, buf), comm)
        out["dispatch_" + name] = {"us": round(us, 1), "GBs": round(rb / us / 1e3, 1)}
    y = torch.empty_like(x)
    for name, tu in (("default", {}), ("rev", {"reverse_backwards": 1}), ("ku2", {"reverse_ku": 2}),
                     ("cta_occupancy", {"combine_ctas_per_sm": 0})):
        with moe.tuned(**tu):
            us = timed(lambda: comm.combine_p2p(buf, r, y), comm)
        out["combine_" + name] = {"us": round(us, 1), "GBs": round(rb / us / 1e3, 1)}
    if rank == 0:
        print(json.dumps(out))
    torch.cuda.synchronize()
    dist.barrier()
    comm.symm_free(buf)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
