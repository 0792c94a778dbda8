"""Training extension on the GPU vs the fp64 oracle (parity UNPINNED: the
reference has no backward/loss/SGD).  Contract (BASELINE.json north_star):
per-layer activations and gradients within 1e-4 scaled, training loss within
1e-3 of the oracle over 10 epochs."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def close(a, b, tol=1e-4):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    rms = float(np.sqrt(np.mean(b * b))) if b.size else 0.0
    err = np.abs(a - b) - tol * (np.abs(b) + rms)
    assert err.max() <= 0.0, f"excess {err.max():.3e} rms {rms:.3e}"


KIND = {"sage": O.SAGE, "gcn": O.GCN, "sum": O.SUM}


def run_pair(kind, n, deg, dims, epochs, lr, seed=5):
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.train import FullGraphTrainer, ModelConfig, init_weights

    g = G.gen_random_graph(n, deg, seed)
    c = O.CSR(n, g.row_offsets(), g.col_indices())
    cfg = ModelConfig(kind, list(dims), lr=lr)
    w0 = init_weights(cfg, 3)
    tr = FullGraphTrainer(g, cfg, weights=w0)
    x = O.make_features(n, dims[0], 1).astype(np.float32).astype(np.float64)
    labels = O.make_labels(n, dims[-1], 2)
    model = O.Model(KIND[kind], dims)
    w = np.concatenate([a.astype(np.float32).astype(np.float64).ravel() for a in w0])
    losses_gpu, losses_ref = [], []
    for e in range(epochs):
        tr.keep_activations = e == 0
        lg = tr.train_epoch()
        if e == 0:
            lr_, grads, acts, dacts = O.train_epoch(c, x, labels, model, w, lr, want_state=True, nthreads=4)
            for a_gpu, a_ref in zip(tr.activations, acts):
                close(a_gpu.double().cpu().numpy(), a_ref)
            # updated weights after one step == w0 - lr * grads
            got = np.concatenate([a.ravel() for a in tr.get_weights()])
            close(got, w)
        else:
            lr_ = O.train_epoch(c, x, labels, model, w, lr, nthreads=4)
        losses_gpu.append(lg)
        losses_ref.append(lr_)
    return np.array(losses_gpu), np.array(losses_ref)


@pytest.mark.parametrize("kind", ["sage", "gcn"])
def test_ten_epoch_loss_parity(cuda, kind):
    lg, lr = run_pair(kind, 3000, 20.0, [96, 64, 64, 41], 10, 0.5)
    assert np.all(np.abs(lg - lr) <= 1e-3), (lg, lr)
    assert lg[-1] < lg[0]  # it trains


def test_sum_model_matches_reference_forward(cuda):
    """The reference Sum model (ReLU between layers) through the trainer."""
    lg, lr = run_pair("sum", 1500, 6.0, [16, 16, 8], 3, 1e-4)
    assert np.all(np.abs(lg - lr) <= 1e-3)


def test_reddit_width_layer_parity(cuda):
    """602-wide inputs (Reddit feature width), 41 classes, one epoch."""
    lg, lr = run_pair("sage", 2000, 40.0, [602, 64, 41], 2, 0.1)
    assert np.all(np.abs(lg - lr) <= 1e-3)
