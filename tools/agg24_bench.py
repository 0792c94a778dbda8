"""Packed-24 vs fp32 gathered rows: the aggregation pass alone (CUDA events), on the
Reddit shape (L2 regime) and the products shape (HBM regime), plus the numerics
(packed-24 result vs the fp32 kernel on the same rounded values, and vs fp32 inputs).

    GDX_P24_MINB=4|6|8 python tools/agg24_bench.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200 import _lib
    from paper_2311_06837_b200._lib import AggregateArgs, call
    from paper_2311_06837_b200.device import aggregate, dense, stream_handle

    d = torch.device("cuda", 0)
    res = []
    for name, n, deg, seed, widths, variant in (("reddit", 232965, 491.99, 11, (64, 48), 0),
                                                  ("products", 2449029, 25.26, 13, (64,), 0)):
        g = G.gen_random_graph(n, deg, seed)
        dg = g.device(d)
        nnz = g.num_edges()
        for w in widths:
            src = (torch.rand((n, w), device=d) - 0.5)
            hi = torch.empty((n, w), dtype=torch.int16, device=d)
            lo = torch.empty((n, w), dtype=torch.uint8, device=d)
            call("gdx_pack24", src.data_ptr(), w, n, w, hi.data_ptr(), lo.data_ptr(), w, stream_handle())
            src24 = torch.empty_like(src)
            call("gdx_unpack24", hi.data_ptr(), lo.data_ptr(), w, n, w, src24.data_ptr(), w, stream_handle())
            out32 = dense(n, w, d)
            out24 = dense(n, w, d)
            var = 1 if w == 48 else variant

            def run32():
                aggregate(dg, src24, w, out=out32, self_coef=1.0, variant=var)

            def run24():
                a = AggregateArgs()
                a.row_ptr, a.col, a.rows, a.width = dg.row_ptr.data_ptr(), dg.col.data_ptr(), n, w
                a.src, a.ld_src, a.src_lo8 = hi.data_ptr(), w, lo.data_ptr()
                a.self_coef = 1.0
                a.out, a.ld_out = out24.data_ptr(), out24.shape[1]
                call("gdx_aggregate_variant", _lib.C.byref(a), var, stream_handle())

            def timed(fn, reps=20):
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                ev = []
                for _ in range(reps):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    fn()
                    b.record()
                    ev.append((a, b))
                torch.cuda.synchronize()
                return float(np.median([a.elapsed_time(b) for a, b in ev]))

            t32, t24 = timed(run32), timed(run24)
            extra = {}
            if w == 48:  # 48 values on a 64-element plane pitch: 3 + 2 aligned sectors per row
                hi64 = torch.zeros((n, 64), dtype=torch.int16, device=d)
                lo64 = torch.zeros((n, 64), dtype=torch.uint8, device=d)
                hi64[:, :w] = hi
                lo64[:, :w] = lo
                out64 = dense(n, w, d)
                for v in (0, 1, 16):
                    def run64(v=v):
                        a = AggregateArgs()
                        a.row_ptr, a.col, a.rows, a.width = dg.row_ptr.data_ptr(), dg.col.data_ptr(), n, w
                        a.src, a.ld_src, a.src_lo8 = hi64.data_ptr(), 64, lo64.data_ptr()
                        a.ld_src_lo8 = 64
                        a.self_coef = 1.0
                        a.out, a.ld_out = out64.data_ptr(), out64.shape[1]
                        call("gdx_aggregate_variant", _lib.C.byref(a), v, stream_handle())
                    extra[f"p24_pitch64_v{v}_ms"] = round(timed(run64), 4)
                    r24 = out24[:, :w].double()
                    extra[f"p24_pitch64_v{v}_err"] = float(((out64[:, :w].double() - r24).abs() /
                                                            (r24.abs() + float(r24.pow(2).mean().sqrt()))).max())
                del hi64, lo64, out64
            ref = out32[:, :w].double()
            rms = float(ref.pow(2).mean().sqrt())
            err_same = float(((out24[:, :w].double() - ref).abs() / (ref.abs() + rms)).max())
            aggregate(dg, src, w, out=out32, self_coef=1.0, variant=var)
            ref2 = out32[:, :w].double()
            err_fp32 = float(((out24[:, :w].double() - ref2).abs() / (ref2.abs() + rms)).max())
            alg32 = 4 * nnz + 8 * (n + 1) + 4 * w * nnz + 4 * w * n
            alg24 = 4 * nnz + 8 * (n + 1) + 3 * w * nnz + 4 * w * n
            res.append({"graph": name, "width": w, "fp32_ms": round(t32, 4), "p24_ms": round(t24, 4),
                        "speedup": round(t32 / t24, 3), "fp32_GBps": round(alg32 / t32 / 1e6, 1),
                        "p24_GBps": round(alg24 / t24 / 1e6, 1), "err_vs_same_values": err_same,
                        "err_vs_fp32_inputs": err_fp32, "minb": os.environ.get("GDX_P24_MINB", "6"), **extra})
            del src, hi, lo, src24, out32, out24
        del dg, g
        torch.cuda.empty_cache()
    for r in res:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
