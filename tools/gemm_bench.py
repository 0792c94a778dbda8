"""Microbenchmark of the tcgen05 GEMM (K2) on the trainer's shapes.

    python tools/gemm_bench.py

For each shape prints ms, algorithmic bytes (A + B operand reads, split bf16 =
4 B/element, + fp32 C write) and FLOP rate (3 bf16 MMAs per product counted as
the 2*M*N*K useful FLOPs).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = [
    # name, m, n, k, a_mn, b_mn, split_k
    ("reddit L1 fwd", 232965, 128, 602, 0, 0, 1),
    ("reddit L2 fwd", 232965, 128, 64, 0, 0, 1),
    ("reddit dH L2", 232965, 64, 128, 0, 1, 1),
    ("reddit dW L1", 128, 602, 232965, 1, 1, 96),
    ("reddit dW L2", 128, 64, 232965, 1, 1, 296),
    ("products L1 fwd", 2449029, 64, 104, 0, 0, 1),
    ("products L2 fwd", 2449029, 64, 64, 0, 0, 1),
    ("products dH", 2449029, 64, 64, 0, 1, 1),
    ("products dW L2", 64, 64, 2449029, 1, 1, 296),
    ("reddit dH L2 fused(mask,scale,split)", 232965, 64, 128, 0, 1, -1),
    ("papers cobatch L1 fwd", 6000000, 128, 128, 0, 0, 1),
    ("papers cobatch L2 fwd", 6000000, 128, 64, 0, 0, 1),
    ("papers cobatch L3 fwd", 6000000, 384, 64, 0, 0, 1),
    ("papers cobatch dH L3", 6000000, 64, 384, 0, 1, 1),
    ("papers cobatch dW L3", 384, 64, 6000000, 1, 1, 296),
    ("papers cobatch dH L2 fused(mask,scale,split)", 6000000, 64, 128, 0, 1, -1),
    ("products dH fused(mask,scale,split)", 2449029, 64, 64, 0, 1, -1),
]


def main():
    import torch
    from paper_2311_06837_b200 import device as D

    d = torch.device("cuda", 0)
    out = []
    only = os.environ.get("GEMM_ONLY")
    for name, m, n, k, a_mn, b_mn, sk in SHAPES:
        if only and only not in name:
            continue
        A = D.Split(k, m, d) if a_mn else D.Split(m, k, d)
        B = D.Split(k, n, d) if b_mn else D.Split(n, k, d)
        for t in (A.hi, A.lo, B.hi, B.lo):
            t.copy_(torch.randint(-16000, 16000, t.shape, dtype=torch.int16, device=d))
        fused = sk < 0
        sk = max(sk, 1)
        rows = sk * m if sk > 1 else m
        C = torch.zeros((rows, D.pad4(n)), dtype=torch.float32, device=d)
        kw = dict(c0=C, split_k=sk, a_mn=bool(a_mn), b_mn=bool(b_mn))
        if fused:
            kw.update(mask=torch.randn(m, D.pad4(n), device=d), row_scale=torch.rand(m, device=d),
                      out_split=D.Split(m, n, d), split_unscaled=True)
        for _ in range(3):
            D.gemm_tn(A, B, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            D.gemm_tn(A, B, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        byts = 4 * (m * k + n * k) + 4 * rows * n
        out.append({"shape": name, "m": m, "n": n, "k": k, "ms": round(ms, 4),
                    "GBps": round(byts / ms / 1e6, 1), "TFLOPs": round(2 * m * n * k / ms / 1e9, 1)})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
