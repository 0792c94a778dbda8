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
    T.gemm_tn = wrap("gemm", T.gemm_tn)
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
    g = G.gen_random_graph(C["n"], C["degree"], C["seed"])
    tr = T.FullGraphTrainer(g, T.ModelConfig(C["kind"], C["dims"], lr=C["lr"]), rank=rank, world=world, pg=pg)
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
