"""Short, deterministic GPU workloads for ncu captures (one GPU):

    python tools/profile_target.py reddit|products|hbm|cobatch [--epochs 3]

reddit / products: the C-ABI trainer's eager epochs on the BASELINE shape (every
aggregation and GEMM of the benchmarked epoch); hbm: the products-shape 64-wide
aggregation pass alone (bench.py's roofline.hbm_regime); cobatch: a papers-shape
cooperative batch step (30 M-vertex graph, 64 batches).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what")
    ap.add_argument("--epochs", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.native import NativeTrainer
    from paper_2311_06837_b200.train import ModelConfig

    if args.what in ("reddit", "products"):
        C = bench.CONFIGS["reddit-sage" if args.what == "reddit" else "products-gcn"]
        g = G.gen_random_graph(C["n"], C["degree"], C["seed"])
        tr = NativeTrainer(g, ModelConfig(C["kind"], list(C["dims"]), lr=C["lr"]), use_graph=False,
                           packed24=bool(C.get("packed24")))
        for _ in range(args.epochs):
            tr.train_epoch(sync_loss=False)
        torch.cuda.synchronize()
        tr.close()
    elif args.what == "hbm":
        bench.hbm_regime_pass(torch, torch.device("cuda", 0), reps=2)
    elif args.what == "cobatch":
        from paper_2311_06837_b200.cobatch import CobatchTrainer
        from paper_2311_06837_b200.graph import Partition
        dims = [128, 64, 64, 172]
        g = G.gen_random_graph(30_000_000, 14.55, 17)
        n = g.num_vertices()
        sp = Partition(np.zeros(n, np.uint32), 1)
        scfg = G.SamplingConfig(1, 15, 3)
        sub = G.extract_sampled(g, sp, 0, scfg)
        plan = G.plan_cobatch_fixed_r(sub, g, 3, scfg, 64, G.ModelSpec(3, 64, 128), target_split="random")
        plan.batches = plan.batches[:2]
        tr = CobatchTrainer(g, ModelConfig("sage", dims, lr=0.1), plan, sp, sp, 0)
        for _ in range(args.epochs):
            tr.train_epoch(sync_loss=False)
        torch.cuda.synchronize()
        if os.environ.get("TIME_EPOCHS"):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                tr.train_epoch(sync_loss=False)
            e1.record()
            torch.cuda.synchronize()
            print(f"cobatch ms per batch step: {e0.elapsed_time(e1) / 5 / len(plan.batches):.3f} "
                  f"(GDX_AGG_LOWDEG={os.environ.get('GDX_AGG_LOWDEG', 'auto')})")
    else:
        raise SystemExit(f"unknown target {args.what}")


if __name__ == "__main__":
    main()
