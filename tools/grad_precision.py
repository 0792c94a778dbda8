"""Diagnostic: per-quantity deviation of one GPU training epoch from the fp64 oracle
(same inputs), as max |a-b| / (|b| + rms(b)) -- the parity test's scaled metric.

    python tools/grad_precision.py [--n 232965 --deg 491.99 --kind sage --init uniform]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def scaled(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    rms = float(np.sqrt(np.mean(b * b)))
    return float(np.max(np.abs(a - b) / (np.abs(b) + rms)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=232965)
    ap.add_argument("--deg", type=float, default=491.99)
    ap.add_argument("--seed", type=int, default=11)
    ap.add_argument("--kind", default="sage")
    ap.add_argument("--dims", default="602,64,64,41")
    ap.add_argument("--init", default="uniform")
    ap.add_argument("--lr", type=float, default=0.1)
    args = ap.parse_args()
    import oracle as O
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.train import FullGraphTrainer, ModelConfig

    dims = [int(x) for x in args.dims.split(",")]
    g = G.gen_random_graph(args.n, args.deg, args.seed)
    cfg = ModelConfig(args.kind, dims, lr=args.lr, init=args.init)
    model = O.Model({"sage": O.SAGE, "gcn": O.GCN, "sum": O.SUM}[args.kind], dims)
    w0 = O.stream_weights(model.weight_shapes(), 3, init=args.init)
    tr = FullGraphTrainer(g, cfg, weights=w0)
    tr.keep_activations = True
    lg = tr.train_epoch()
    c = O.CSR(args.n, g.row_offsets(), g.col_indices())
    x = O.make_features(args.n, dims[0], 1).astype(np.float32).astype(np.float64)
    lab = O.make_labels(args.n, dims[-1], 2)
    w = np.concatenate([a.ravel() for a in w0])
    lo, grads, acts, dacts = O.train_epoch(c, x, lab, model, w, args.lr, want_state=True,
                                           nthreads=os.cpu_count())
    out = {"n": args.n, "init": args.init, "loss_gpu": lg, "loss_oracle": lo,
           "acts": [scaled(a.double().cpu().numpy(), b) for a, b in zip(tr.activations, acts)],
           "logit_rms": float(np.sqrt(np.mean(acts[-1] ** 2))),
           "logit_max_abs_err": float(np.max(np.abs(tr.activations[-1].double().cpu().numpy() - acts[-1]))),
           "dW": [], "dW_frob_rel": [], "relu_flips": []}
    for a, b in zip(tr.activations[:-1], acts[:-1]):
        a = a.double().cpu().numpy()
        out["relu_flips"].append(int(np.sum((a > 0) != (b > 0))))
    off = 0
    for gm in tr.get_grads():
        ref = grads[off:off + gm.size].reshape(gm.shape)
        off += gm.size
        out["dW"].append(scaled(gm, ref))
        out["dW_frob_rel"].append(float(np.linalg.norm(gm - ref) / np.linalg.norm(ref)))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
