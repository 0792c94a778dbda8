"""Same box, same workload: the C-ABI trainer (csrc/trainer.cu) vs the torch-
orchestrated FullGraphTrainer, CUDA-graph epochs, CUDA-event time, max over ranks.

    torchrun --nproc-per-node N tools/trainer_compare.py [--config products-gcn]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="reddit-sage")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.native import NativeTrainer
    from paper_2311_06837_b200.train import FullGraphTrainer, ModelConfig

    world, rank, local = bench.dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        opts = dist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True
        dist.init_process_group("nccl", device_id=dev, pg_options=opts)
        pg = dist.group.WORLD
    C = bench.CONFIGS[args.config]
    g = G.gen_random_graph(C["n"], C["degree"], C["seed"])
    cfg = ModelConfig(C["kind"], list(C["dims"]), lr=C["lr"])

    def timeit(step, stream):
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    out = {"config": args.config, "world": world}
    nt = NativeTrainer(g, cfg, rank=rank, world=world, pg=pg)
    out["native_ms"] = timeit(lambda: nt.train_epoch(sync_loss=False), nt.stream())
    ft = FullGraphTrainer(g, cfg, rank=rank, world=world, pg=pg)
    ft.capture(warmup=2)
    out["torch_ms"] = timeit(ft.replay, torch.cuda.current_stream())
    out["native_ms_again"] = timeit(lambda: nt.train_epoch(sync_loss=False), nt.stream())
    if world > 1:   # the one-kernel exchange + aggregation
        nf = NativeTrainer(g, cfg, rank=rank, world=world, pg=pg, fused_exchange=True)
        out["native_fused_ms"] = timeit(lambda: nf.train_epoch(sync_loss=False), nf.stream())
        torch.cuda.synchronize()
        dist.barrier()
        nf.close()
    # aggregation launches of eager epochs (CUDA events on each trainer's stream)
    nt2 = NativeTrainer(g, cfg, rank=rank, world=world, pg=pg, use_graph=False)
    nt2.profile(True)
    for _ in range(3):
        nt2.train_epoch(sync_loss=False)
    ms, n, by = nt2.profile_read()
    out["native_agg_ms_per_epoch"] = ms / 3
    out["native_eager_ms"] = timeit(lambda: nt2.train_epoch(sync_loss=False), nt2.stream())
    ft.graph = None
    ft.enable_kernel_events(True)
    for _ in range(3):
        ft.train_epoch(sync_loss=False)
    ms2, n2, by2 = ft.kernel_event_summary()
    ft.enable_kernel_events(False)
    out["torch_agg_ms_per_epoch"] = ms2 / 3
    out["torch_eager_ms"] = timeit(lambda: ft.train_epoch(sync_loss=False), torch.cuda.current_stream())
    out["agg_launches"] = [n / 3, n2 / 3]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    nt2.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    ft.graph = None
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    nt.close()
    ft.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
