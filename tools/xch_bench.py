"""Row-exchange microbenchmark (torchrun, one rank per GPU): one equal-block
all-gather of a [world*B, 64] fp32 buffer, B rows owned per rank, by

  * NCCL all_gather_into_tensor,
  * copy-engine pushes (GDX_PUSH=ce), SM unicast pushes (sm), NVSwitch multicast
    pushes (mc) through P2PExchange, each with the device arrival signal + wait.

    torchrun --nproc-per-node 4 tools/xch_bench.py [--rows 1500000] [--ctas 32,148,296]

Prints per mode: ms per exchange (max over ranks) and delivered GB/s per rank
((world-1) * B * 256 bytes received).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1500000)
    ap.add_argument("--ctas", default="32,148,296")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    pg = dist.group.WORLD
    from paper_2311_06837_b200.train import P2PExchange

    B, W = args.rows, 64
    recv = (world - 1) * B * W * 4
    out = {"world": world, "rows_per_rank": B, "bytes_received_per_rank": recv, "modes": {}}

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.reps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    full = torch.zeros(world * B, W, device=dev)
    ms = timed(lambda: dist.all_gather_into_tensor(full, full[rank * B:(rank + 1) * B].clone()))
    out["modes"]["nccl"] = {"ms": round(ms, 3), "GBps": round(recv / ms / 1e6, 1)}
    del full
    for kind in ("ce", "sm", "mc"):
        os.environ["GDX_PUSH"] = kind
        try:
            x = P2PExchange(rank, world, pg, dev)
            buf, deltas = x.buffer(world * B, W)
        except Exception as e:  # multicast unsupported etc.
            out["modes"][kind] = {"error": str(e)[:200]}
            continue
        own = buf[rank * B:(rank + 1) * B]
        for c in ([int(v) for v in args.ctas.split(",")] if kind != "ce" else [0]):
            x.push_ctas = c or x.push_ctas

            def step():
                x.push(own, deltas)
                x.wait()
            ms = timed(step)
            out["modes"][f"{kind}{c or ''}"] = {"ms": round(ms, 3), "GBps": round(recv / ms / 1e6, 1)}
        if kind == "sm":  # sparse push of a random half of the rows to every peer
            g = torch.Generator(device="cpu").manual_seed(rank)
            half = torch.sort(torch.randperm(B, generator=g)[:B // 2])[0].to(torch.int32).to(dev)
            idx = torch.cat([half] * (world - 1))
            off = [i * (B // 2) for i in range(world)]

            def step_sparse():
                x.push(own, deltas, rows=(idx, off))
                x.wait()
            ms = timed(step_sparse)
            out["modes"]["sm_rows_half"] = {"ms": round(ms, 3), "GBps": round(recv / 2 / ms / 1e6, 1)}
        torch.cuda.synchronize()
        dist.barrier()
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
