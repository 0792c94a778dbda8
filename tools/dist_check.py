"""Multi-GPU correctness check (run under torchrun, one rank per GPU):

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/dist_check.py

Trains the row-partitioned SAGE/GCN model for a few epochs over NCCL and checks
that (a) every rank ends with bit-identical weights, (b) the loss trajectory
matches the fp64 oracle within 1e-3 (rank 0).  Prints one JSON line on rank 0.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    opts = dist.ProcessGroupNCCL.Options()
    opts.is_high_priority_stream = True  # collectives get SMs ahead of the aggregation
    dist.init_process_group("nccl", device_id=dev, pg_options=opts)
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.train import FullGraphTrainer, ModelConfig, init_weights

    out = {"world": world, "ok": True, "cases": []}
    for kind, n, deg, dims, epochs in (("sage", 5001, 24.0, [96, 64, 64, 41], 5),
                                       ("gcn", 3001, 10.0, [32, 32, 8], 4),
                                       ("sage", 3001, 12.0, [40, 32, 32, 72], 3)):
        g = G.gen_random_graph(n, deg, 5)
        cfg = ModelConfig(kind, dims, lr=0.5)
        w0 = init_weights(cfg, 3)
        tr = FullGraphTrainer(g, cfg, rank=rank, world=world, weights=w0, pg=dist.group.WORLD)
        losses = [tr.train_epoch() for _ in range(epochs)]
        W = torch.from_numpy(np.concatenate([a.ravel() for a in tr.get_weights()])).to(dev)
        Wmax, Wmin = W.clone(), W.clone()
        dist.all_reduce(Wmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(Wmin, op=dist.ReduceOp.MIN)
        same = bool(torch.equal(Wmax, Wmin))
        case = {"kind": kind, "n": n, "losses": losses, "weights_identical_across_ranks": same}
        if rank == 0:
            import oracle as O
            c = O.CSR(n, g.row_offsets(), g.col_indices())
            x = O.make_features(n, dims[0], 1).astype(np.float32).astype(np.float64)
            lab = O.make_labels(n, dims[-1], 2)
            m = O.Model({"sage": O.SAGE, "gcn": O.GCN}[kind], dims)
            w = np.concatenate([a.astype(np.float32).astype(np.float64).ravel() for a in w0])
            ref = [O.train_epoch(c, x, lab, m, w, 0.5, nthreads=8) for _ in range(epochs)]
            case["oracle"] = ref
            case["max_abs_loss_diff"] = float(np.max(np.abs(np.array(losses) - np.array(ref))))
            case["ok"] = same and case["max_abs_loss_diff"] <= 1e-3
            out["ok"] &= case["ok"]
        out["cases"].append(case)
    # cooperative batching (config 5 semantics): one server, `world` GPUs share each batch
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from test_cobatch import _oracle_batch, _plan
    from paper_2311_06837_b200.cobatch import CobatchTrainer
    dims = [48, 32, 32, 72]   # widening output layer: aggregate-first inside the batch
    g, hp, plan = _plan(4000, 10.0, 21, 1, world, 3, 3, G.SamplingConfig(1, 15, 3), dims)
    cfg = ModelConfig("sage", dims, lr=0.5)
    w0 = init_weights(cfg, 3)
    tr = CobatchTrainer(g, cfg, plan, hp.server, hp.gpu, 0, rank=rank, world=world, weights=w0,
                        pg=dist.group.WORLD)
    got = []
    for _ in range(2):
        for i in range(len(plan.batches)):
            tr.train_batch(i)
            got.append(float(tr.loss_acc.item()) / len(plan.batches[i].target_vertices))
    W = torch.from_numpy(np.concatenate([a.ravel() for a in tr.get_weights()])).to(dev)
    Wmax, Wmin = W.clone(), W.clone()
    dist.all_reduce(Wmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(Wmin, op=dist.ReduceOp.MIN)
    same = bool(torch.equal(Wmax, Wmin))
    case = {"kind": "sage-cobatch", "batches": len(plan.batches), "losses": got,
            "weights_identical_across_ranks": same,
            "rows_per_rank": [geo.nloc for geo in tr.geoms]}
    if rank == 0:
        import oracle as O
        n = g.num_vertices()
        x_all = O.make_features(n, dims[0], 1).astype(np.float32).astype(np.float64)
        lab_all = O.make_labels(n, dims[-1], 2)
        m = O.Model(O.SAGE, dims)
        w = np.concatenate([a.astype(np.float32).astype(np.float64).ravel() for a in w0])
        ref = []
        for _ in range(2):
            for b in plan.batches:
                lc, x, lab, layer_rows, nt, _ = _oracle_batch(g, b, 3, x_all, lab_all)
                ref.append(O.train_epoch_masked(lc, x, lab, m, w, 0.5, nt, float(nt), nthreads=8,
                                                layer_rows=layer_rows)[0])
        case["oracle"] = ref
        case["max_abs_loss_diff"] = float(np.max(np.abs(np.array(got) - np.array(ref))))
        case["ok"] = same and case["max_abs_loss_diff"] <= 1e-3
        out["ok"] &= case["ok"]
    out["cases"].append(case)
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not out["ok"]:
        sys.exit(1)


if __name__ == "__main__":
    main()
