"""Per-phase device-time breakdown of one eager training epoch (single or multi-GPU).

    torchrun --nproc-per-node N tools/phase_breakdown.py        (or plain python for N=1)

Wraps the trainer's kernel entry points and collectives with CUDA events on the
compute stream (so collective rows include the time the stream waits for NCCL)
and prints, on rank 0, milliseconds per phase per epoch (mean of 5 epochs, max
over ranks).
"""
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        opts = dist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True  # collectives get SMs ahead of the aggregation
        dist.init_process_group("nccl", device_id=dev, pg_options=opts)
        pg = dist.group.WORLD
    import paper_2311_06837_b200 as G
    import paper_2311_06837_b200.train as T

    records = []

    def wrap(name, fn):
        def inner(*a, **k):
            if not ACTIVE[0]:
                return fn(*a, **k)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = fn(*a, **k)
            if hasattr(r, "wait"):
                r.wait()
                nm = name + "(wait)"
            else:
                nm = name
            e1.record()
            records.append((nm, e0, e1))
            return r
        return inner

    ACTIVE = [False]
    orig_gemm = T.gemm_tn

    def gemm(A, B, **kw):
        tag = "gemm_dW" if kw.get("split_k", 1) > 1 or kw.get("a_mn") else (
            "gemm_dH" if kw.get("b_mn") else "gemm_fwd")
        return wrap(tag, orig_gemm)(A, B, **kw)
    T.gemm_tn = gemm
    orig_agg = T.FullGraphTrainer._agg

    def agg(self, csr, src, width, **kw):
        tag = "agg_local" if "row_begin" in kw else ("agg_remote" if "skip" in kw else "agg")
        return wrap(tag, lambda: orig_agg(self, csr, src, width, **kw))()
    T.FullGraphTrainer._agg = agg
    orig_call = T.call
    T.call = lambda name, *a: wrap(name.replace("gdx_", ""), orig_call)(name, *a)
    ex_ag = T.RowExchange.allgather_rows
    T.RowExchange.allgather_rows = lambda self, full: wrap("allgather_sync", ex_ag)(self, full)
    ex_ar = T.RowExchange.allreduce
    T.RowExchange.allreduce = lambda self, t: wrap("allreduce", ex_ar)(self, t)

    cfgname = os.environ.get("GDX_CONFIG", "reddit-sage")
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import CONFIGS
    C = CONFIGS[cfgname]
    n = int(os.environ.get("GDX_N", C["n"]))
    g = G.gen_random_graph(n, C["degree"], C["seed"])
    cfg = T.ModelConfig(C["kind"], C["dims"], lr=C["lr"])
    if C["mode"] == "cobatch":
        # the first GDX_NB batches of an R-batch random-split plan (per-batch cost is what matters)
        import numpy as np
        from paper_2311_06837_b200 import batch_plan as BP
        from paper_2311_06837_b200.cobatch import CobatchTrainer
        from paper_2311_06837_b200.graph import Partition
        R, NB = int(os.environ.get("GDX_R", C["batches"])), int(os.environ.get("GDX_NB", "4"))
        L = len(C["dims"]) - 1
        scfg = G.SamplingConfig(*C["eas"])
        sp = Partition(np.zeros(n, np.uint32), 1)
        ga = np.zeros(n, np.uint32)
        G._lib.call("gdx_host_partition_random", n, world, G.mix64(4 ^ 1), ga.ctypes.data)
        universe = np.ones(n, np.uint8)
        plan = BP.BatchPlan(0, "fetch_then_split", L)
        spec = BP.ModelSpec(L, C["dims"][1], C["dims"][0])
        for grp in BP.split_targets_random(np.arange(n, dtype=np.uint32), R, scfg.seed)[:NB]:
            plan.batches.append(BP.make_batch(g, universe, grp, L, scfg, spec))
        tr = CobatchTrainer(g, cfg, plan, sp, Partition(ga, world), 0, rank=rank, world=world, pg=pg)
    else:
        tr = T.FullGraphTrainer(g, cfg, rank=rank, world=world, pg=pg)
    for _ in range(3):
        tr.train_epoch(sync_loss=False)
    torch.cuda.synchronize()
    ACTIVE[0] = True
    E = 5
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(E):
        tr.train_epoch(sync_loss=False)
    t1.record()
    torch.cuda.synchronize()
    ACTIVE[0] = False
    per = defaultdict(float)
    for nm, a, b in records:
        per[nm] += a.elapsed_time(b) / E
    names = sorted(per)
    vals = torch.tensor([per[n] for n in names] + [t0.elapsed_time(t1) / E], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    if rank == 0:
        out = {n: round(float(v), 4) for n, v in zip(names, vals[:-1])}
        out["epoch_ms_eager"] = round(float(vals[-1]), 4)
        out["sum_of_phases"] = round(float(vals[:-1].sum()), 4)
        print(json.dumps({"world": world, "phases_ms_per_epoch": out}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
