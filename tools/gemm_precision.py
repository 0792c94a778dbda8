"""Diagnostic: accuracy of the tcgen05 split-bf16 GEMM on a dW-shaped product
(C[m][n] = sum over K rows of A[k][m] B[k][n], both MN-major, split-K) against
fp64 on (a) the exact split values hi+lo and (b) the unsplit fp32 inputs.

    python tools/gemm_precision.py [--k 232965 --m 128 --n 602]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=232965)
    ap.add_argument("--m", type=int, default=128)
    ap.add_argument("--n", type=int, default=602)
    ap.add_argument("--splitks", default="1,8,98")
    ap.add_argument("--dist", default="uniform")
    args = ap.parse_args()
    import torch
    from paper_2311_06837_b200.device import Split, gemm_tn

    d = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    K, M, N = args.k, args.m, args.n
    if args.dist == "uniform":
        a = rng.uniform(-0.5, 0.5, (K, M)).astype(np.float32)
        b = rng.uniform(-0.5, 0.5, (K, N)).astype(np.float32)
    else:   # relu-like B (non-negative)
        a = rng.standard_normal((K, M)).astype(np.float32) * 1e-3
        b = np.maximum(rng.standard_normal((K, N)), 0).astype(np.float32)
    A = Split(K, M, d).fill_from(torch.from_numpy(a).to(d), M)
    B = Split(K, N, d).fill_from(torch.from_numpy(b).to(d), N)
    a_split = A.to_float().double().cpu().numpy()
    b_split = B.to_float().double().cpu().numpy()
    exact_split = a_split.T @ b_split
    exact = a.astype(np.float64).T @ b.astype(np.float64)
    out = {"K": K, "M": M, "N": N, "dist": args.dist, "runs": []}
    rms = float(np.sqrt(np.mean(exact ** 2)))
    for sk in [int(x) for x in args.splitks.split(",")]:
        ws = torch.zeros((sk * M, N + (-N) % 4), dtype=torch.float32, device=d)
        gemm_tn(A, B, c0=ws, split_k=sk, a_mn=True, b_mn=True)
        got = ws.view(sk, M, -1)[:, :, :N].double().sum(0).cpu().numpy()
        e_split = got - exact_split
        e_full = got - exact
        out["runs"].append({
            "split_k": sk,
            "max_scaled_vs_split_values": float(np.max(np.abs(e_split) / (np.abs(exact_split) + rms))),
            "mean_err_over_rms_vs_split": float(np.mean(e_split) / rms),
            "corr_err_with_value_vs_split": float(np.corrcoef(e_split.ravel(), exact_split.ravel())[0, 1]),
            "max_scaled_vs_fp32_inputs": float(np.max(np.abs(e_full) / (np.abs(exact) + rms))),
            "rms_err_over_rms": float(np.sqrt(np.mean(e_full ** 2)) / rms)})
    split_err = exact_split - exact
    out["split_only_max_scaled"] = float(np.max(np.abs(split_err) / (np.abs(exact) + rms)))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
