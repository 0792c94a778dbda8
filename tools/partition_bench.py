"""partition_mincut on the BASELINE graph shapes: the engine's host partitioner
(gain-bucket growth) vs the compiled reference (oracle/_ref), same assignment required.

    python tools/partition_bench.py [reddit|products|small] [parts]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = {"reddit": (232965, 491.99, 11), "products": (2449029, 25.26, 13), "small": (10000, 10.0, 7)}


def main():
    import oracle as O
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.partition_host import partition_mincut
    shape = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    parts = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    n, d, seed = SHAPES[shape]
    g = G.gen_random_graph(n, d, seed)
    t0 = time.perf_counter()
    mine = partition_mincut(g, parts, 1).assignment
    t_mine = time.perf_counter() - t0
    rec = {"shape": shape, "n": n, "nnz": int(g.num_edges()), "parts": parts, "engine_s": round(t_mine, 2)}
    if O.ref_available():
        R = O.ref()
        h = R.grr_graph_from_csr(n, g.row_offsets(), g.col_indices())
        ref = np.zeros(n, np.uint32)
        t0 = time.perf_counter()
        assert R.grr_partition_mincut(h, parts, 1, 0.05, ref) == 0
        rec["reference_s"] = round(time.perf_counter() - t0, 2)
        R.grr_graph_free(h)
        rec["identical"] = bool(np.array_equal(mine, ref))
    print(rec)


if __name__ == "__main__":
    main()
