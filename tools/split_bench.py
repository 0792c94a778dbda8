"""Cost of splitting each row into local-source and remote-source passes (the N>1
exchange overlap), isolated on one GPU: Reddit rows [0, B) of a 4-way row partition,
(a) one full pass, (b) local pass [seg_lo, seg_hi) + remote pass (skip + partial),
(c) the same split over two pre-split CSRs (local-source / remote-source edges only)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200._lib import call
    from paper_2311_06837_b200.device import DeviceCSR, aggregate, dense, stream_handle

    d = torch.device("cuda", 0)
    world = int(os.environ.get("WORLD", "4"))
    g = G.gen_random_graph(232965, 491.99, 11)
    n = g.num_vertices()
    B = -(-n // world)
    ro, ci = g.row_offsets(), g.col_indices()
    lro = (ro[:B + 1] - ro[0]).astype(np.uint64)
    lci = ci[:int(ro[B])]
    csr = DeviceCSR.upload(lro, lci, d)
    src = torch.rand((world * B, 64), device=d) - 0.5
    out = dense(B, 64, d)
    P = dense(B, 64, d)
    seg_lo = torch.empty(B, dtype=torch.int64, device=d)
    seg_hi = torch.empty(B, dtype=torch.int64, device=d)
    call("gdx_row_split", csr.row_ptr.data_ptr(), csr.col.data_ptr(), B, 0, B, seg_lo.data_ptr(), seg_hi.data_ptr(),
         stream_handle())
    # pre-split CSRs
    rows = np.repeat(np.arange(B), np.diff(lro).astype(np.int64))
    loc = lci < B
    def sub(mask):
        r = rows[mask]
        c = lci[mask]
        cnt = np.bincount(r, minlength=B)
        p = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint64)
        return DeviceCSR.upload(p, c, d)
    cl, cr = sub(loc), sub(~loc)
    scale = torch.rand(B, device=d)

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    res = {"rows": B, "world": world, "nnz": len(lci), "local_frac": float(loc.mean())}
    res["full_ms"] = timed(lambda: aggregate(csr, src, 64, out=out, self_coef=1.0, post_scale=scale))
    res["local_ms"] = timed(lambda: aggregate(csr, src, 64, out=P, row_begin=seg_lo, row_end=seg_hi))
    res["remote_ms"] = timed(lambda: aggregate(csr, src, 64, out=out, skip=(seg_lo, seg_hi), partial=P, self_coef=1.0,
                                               post_scale=scale))
    res["presplit_local_ms"] = timed(lambda: aggregate(cl, src, 64, out=P))
    res["presplit_remote_ms"] = timed(lambda: aggregate(cr, src, 64, out=out, partial=P, self_coef=1.0,
                                                        post_scale=scale))
    res["split_overhead"] = round((res["local_ms"] + res["remote_ms"]) / res["full_ms"] - 1, 3)
    res["presplit_overhead"] = round((res["presplit_local_ms"] + res["presplit_remote_ms"]) / res["full_ms"] - 1, 3)
    print(json.dumps({k: round(v, 4) if isinstance(v, float) else v for k, v in res.items()}))


if __name__ == "__main__":
    main()
