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


@pytest.mark.parametrize("agg_first", ["1", "0"])
def test_widening_output_layer_parity(cuda, monkeypatch, agg_first):
    """SAGE with more classes than hidden units (papers shape: 64 -> 172): the output
    layer runs aggregate-first (exchange and gather at the input width); both orders
    must match the oracle."""
    monkeypatch.setenv("GDX_AGG_FIRST", agg_first)
    lg, lr = run_pair("sage", 2500, 12.0, [40, 32, 32, 72], 4, 0.5)
    assert np.all(np.abs(lg - lr) <= 1e-3), (lg, lr)


def test_sum_model_matches_reference_forward(cuda):
    """The reference Sum model (ReLU between layers) through the trainer."""
    lg, lr = run_pair("sum", 1500, 6.0, [16, 16, 8], 3, 1e-4)
    assert np.all(np.abs(lg - lr) <= 1e-3)


def test_reddit_width_layer_parity(cuda):
    """602-wide inputs (Reddit feature width), 41 classes, one epoch."""
    lg, lr = run_pair("sage", 2000, 40.0, [602, 64, 41], 2, 0.1)
    assert np.all(np.abs(lg - lr) <= 1e-3)


@pytest.mark.parametrize("kind,m,k", [("gcn", 1, 15), ("sage", 2, 4), ("gcn", 3, O.UNLIMITED),
                                      ("sage", 5, 3), ("sum", 2, 6)])
def test_subgraph_training_matches_oracle(cuda, kind, m, k):
    """EAS / preload mode: train on one server's preloaded inner + halo subgraph,
    loss on its inner vertices; the oracle runs the same epoch on the induced
    local graph (hop-ordered local ids, inner first)."""
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.train import FullGraphTrainer, ModelConfig, init_weights

    n, dims = 3000, [48, 32, 32, 8]
    g = G.gen_random_graph(n, 12.0, 9)
    p = G.partition_random(g, 4, 2)
    sub = G.extract_sampled(g, p, 1, G.SamplingConfig(m, k, 5))
    lr = 1e-4 if kind == "sum" else 0.5  # the unnormalised Sum model diverges at large lr
    cfg = ModelConfig(kind, dims, lr=lr)
    w0 = init_weights(cfg, 3)
    tr = FullGraphTrainer(g, cfg, weights=w0, subgraph=sub)
    # the oracle's local graph: same numbering as the engine (hop, id) and induced rows
    hop = sub.hop_array(n)
    order = np.lexsort((np.arange(n), hop))[: len(sub.inner_vertices) + len(sub.halo_vertices)]
    local = np.full(n, -1, np.int64)
    local[order] = np.arange(len(order))
    ro, ci = g.row_offsets(), g.col_indices()
    rows, cols = [], []
    for i, v in enumerate(order):
        nb = local[ci[ro[v]:ro[v + 1]]]
        nb = nb[nb >= 0]
        rows.append(len(nb))
        cols.append(nb)
    lro = np.concatenate([[0], np.cumsum(rows)]).astype(np.uint64)
    lc = O.CSR(len(order), lro, np.concatenate(cols).astype(np.uint32))
    x = O.make_features(n, dims[0], 1).astype(np.float32).astype(np.float64)[order]
    lab = O.make_labels(n, dims[-1], 2)[order]
    model = O.Model(KIND[kind], dims)
    w = np.concatenate([a.astype(np.float32).astype(np.float64).ravel() for a in w0])
    n_inner = len(sub.inner_vertices)
    L = len(dims) - 1
    hop_sorted = hop[order]
    layer_rows = [int(np.sum(hop_sorted <= L - l - 1)) for l in range(L)]  # hop masking
    x[hop_sorted > L] = 0.0  # inputs beyond L hops are unavailable (reference_gnn.cpp:129-131)
    for e in range(6):
        lg = tr.train_epoch()
        loss, grads = O.train_epoch_masked(lc, x, lab, model, w, lr, n_inner, float(n_inner),
                                           nthreads=4, layer_rows=layer_rows)
        assert abs(lg - loss) <= 1e-3, (e, lg, loss)


def test_feature_stream_matches_resident_features(cuda):
    """End-to-end feature loading (bench e2e): features streamed from pinned host memory
    (one contiguous DMA per step, split with ld = F into the padded GEMM operand) train
    like the resident features."""
    import torch

    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.errors import InputError
    from paper_2311_06837_b200.train import FeatureStream, FullGraphTrainer, ModelConfig, init_weights

    g = G.gen_random_graph(2000, 12.0, 9)
    cfg = ModelConfig("sage", [101, 64, 41], lr=0.5)   # odd width: operand pitch != host row
    w0 = init_weights(cfg, 3)
    ref = FullGraphTrainer(g, cfg, weights=w0)
    tr = FullGraphTrainer(g, cfg, weights=w0)
    xh = ref.X[:ref.nloc, :ref.F].cpu().contiguous().pin_memory()
    lh = ref.labels[:ref.nloc].cpu().pin_memory()
    tr.X[:tr.nloc, :tr.F].zero_()
    fs = FeatureStream(tr)
    for _ in range(3):
        fs.prefetch(xh, lh)
        fs.consume()
        torch.testing.assert_close(fs.stage[(fs.consumed - 1) % 2][:tr.nloc, :tr.F].cpu(), xh.cpu(),
                                   rtol=0, atol=0)
        a, b = tr.train_epoch(), ref.train_epoch()
        assert abs(a - b) <= 1e-6 * abs(b), (a, b)   # loss atomics: summation order only
    with pytest.raises(InputError):
        fs.prefetch(xh.cpu().clone(), lh)   # pageable host memory is rejected
