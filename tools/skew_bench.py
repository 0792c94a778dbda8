"""Skewed-graph aggregation: plain warp-per-row vs degree-binned (hub rows chunked).

    python tools/skew_bench.py [--n 2000000 --deg 10 --hubs 16 --hub-deg 500000]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--deg", type=float, default=10.0)
    ap.add_argument("--hubs", type=int, default=16)
    ap.add_argument("--hub-deg", type=int, default=500_000)
    ap.add_argument("--width", type=int, default=64)
    args = ap.parse_args()
    import torch
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from test_balanced import hub_graph
    from paper_2311_06837_b200.device import RowBins, aggregate, dense

    d = torch.device("cuda", 0)
    g = hub_graph(args.n, args.deg, args.hubs, args.hub_deg, 7)
    dg = g.device(d)
    n, w = g.num_vertices(), args.width
    src = torch.rand((n, w), device=d) - 0.5
    out = dense(n, w, d)
    res = {"n": n, "nnz": g.num_edges(), "max_degree": int(np.diff(g.row_offsets()).max()), "width": w}
    for name, b in (("plain", None), ("binned", RowBins(g.row_offsets(), 4096, 1024, w))):
        for _ in range(2):
            aggregate(dg, src, w, out=out, self_coef=1.0, bins=b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            aggregate(dg, src, w, out=out, self_coef=1.0, bins=b)
        e1.record()
        torch.cuda.synchronize()
        res[f"{name}_ms"] = round(e0.elapsed_time(e1) / 5, 3)
    nnz = g.num_edges()
    res["binned_GBps"] = round((4 * nnz + 8 * (n + 1) + 4 * w * nnz + 4 * w * n) / res["binned_ms"] / 1e6, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
