"""Microbenchmark of the aggregation kernel (K1) alone on the Reddit-shape graph.

    python tools/agg_bench.py [--widths 64,48] [--reps 20]

Times gdx_aggregate with CUDA events on the launching stream (after warm-up) and
prints ms, edges/s and algorithmic GB/s (SURVEY §8d formula) per width.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--widths", default="32,48,64,128")
    ap.add_argument("--variants", default="4,8")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--n", type=int, default=232965)
    ap.add_argument("--degree", type=float, default=491.99)
    ap.add_argument("--no-probe", action="store_true")
    ap.add_argument("--slices", default="", help="also time row slices [0, r) (multi-GPU shard sizes)")
    args = ap.parse_args()
    import torch
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.device import aggregate, dense, Split

    d = torch.device("cuda", 0)
    g = G.gen_random_graph(args.n, args.degree, 11)
    dg = g.device(d)
    nnz, n = g.num_edges(), g.num_vertices()
    res = []
    for w in [int(x) for x in args.widths.split(",")]:
        src = torch.randn(n, w, device=d)
        out = dense(n, w, d)
        for variant in [int(v) for v in args.variants.split(",")]:
            kw = dict(out=out, self_coef=1.0, variant=variant)
            for _ in range(3):
                aggregate(dg, src, w, **kw)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                aggregate(dg, src, w, **kw)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            alg = 4 * nnz + 8 * (n + 1) + 4 * w * nnz + 4 * w * n
            res.append({"n": n, "deg": args.degree, "width": w, "variant": variant, "ms": round(ms, 4),
                        "gedges_per_s": round(nnz / ms / 1e6, 2),
                        "alg_GBps": round(alg / ms / 1e6, 1)})
    for r in [int(x) for x in args.slices.split(",") if x]:
        w = 64
        src = torch.randn(n, w, device=d)
        out = dense(r, w, d)
        sub = dg.slice_rows(0, r)
        nnz_r = int(sub.row_ptr[-1].item() - sub.row_ptr[0].item())
        for _ in range(3):
            aggregate(sub, src, w, out=out, self_coef=1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            aggregate(sub, src, w, out=out, self_coef=1.0)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        res.append({"slice_rows": r, "nnz": nnz_r, "ms": round(ms, 4), "gedges_per_s": round(nnz_r / ms / 1e6, 2)})
    if args.no_probe:
        print(json.dumps(res))
        return
    # bandwidth ceilings with the library's probe kernel: L2-resident (60 MB) and
    # HBM-resident (4 GB) buffers, coalesced stream and random 256 B row gathers
    from paper_2311_06837_b200._lib import call
    from paper_2311_06837_b200.device import stream_handle
    sink = torch.zeros(4, device=d)
    for mb, reps in ((60, 40), (4096, 2)):
        buf = torch.randn(mb * 262144, device=d)
        for mode in (0, 1):
            call("gdx_probe_bandwidth", buf.data_ptr(), buf.numel() * 4, reps, mode, sink.data_ptr(), stream_handle())
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            call("gdx_probe_bandwidth", buf.data_ptr(), buf.numel() * 4, reps, mode, sink.data_ptr(), stream_handle())
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            res.append({"probe_MB": mb, "mode": ["stream", "gather256"][mode], "ms": round(ms, 3),
                        "GBps": round(reps * buf.numel() * 4 / ms / 1e6, 1)})
        del buf
    # library gather for comparison: index_select of 64-wide rows
    src = torch.randn(n, 64, device=d)
    idx = dg.col[:20_000_000].long()
    for _ in range(2):
        torch.index_select(src, 0, idx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        torch.index_select(src, 0, idx)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res.append({"torch_index_select_rows": 20_000_000, "ms": round(ms, 3),
                "gather_GBps": round(20e6 * 256 / ms / 1e6, 1)})
    print(json.dumps(res))


if __name__ == "__main__":
    main()
