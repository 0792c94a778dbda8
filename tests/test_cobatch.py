"""Cooperative-batching training vs the fp64 oracle.

Parity UNPINNED against the reference (it prices cobatches in simulate_epoch but
has no training code): each batch's step is checked against the oracle's masked
epoch on the batch's induced graph in (peel level, id) order; the peel levels
themselves must reproduce the plan's peel_mfg counts exactly (reference
batch_plan.cpp:75-101)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

KIND = {"sage": O.SAGE, "gcn": O.GCN, "sum": O.SUM}


def _plan(n, deg, seed, servers, gpus, r, layers, cfg_s, dims):
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.partition_host import hierarchical_partition

    g = G.gen_random_graph(n, deg, seed)
    hp = hierarchical_partition(g, servers, gpus, "random", 4)
    sub = G.extract_sampled(g, hp.server, 0, cfg_s)
    plan = G.plan_cobatch_fixed_r(sub, g, layers, cfg_s, r,
                                  G.ModelSpec(layers, dims[1], dims[0]))
    return g, hp, plan


def _peel_levels(g, batch, layers):
    """Host BFS from the targets inside the batch (independent restatement)."""
    n = g.num_vertices()
    ro, ci = g.row_offsets(), g.col_indices()
    inb = np.zeros(n, bool)
    inb[batch.vertices] = True
    d = np.full(n, -1, np.int64)
    d[batch.target_vertices] = 0
    front = list(batch.target_vertices)
    for h in range(1, layers + 1):
        nxt = []
        for v in front:
            for u in ci[ro[v]:ro[v + 1]]:
                if inb[u] and d[u] < 0:
                    d[u] = h
                    nxt.append(u)
        front = nxt
    return d


def _oracle_batch(g, batch, layers, x_all, lab_all):
    d = _peel_levels(g, batch, layers)
    keep = np.nonzero(d >= 0)[0]
    order = keep[np.lexsort((keep, d[keep]))]
    local = np.full(g.num_vertices(), -1, np.int64)
    local[order] = np.arange(len(order))
    ro, ci = g.row_offsets(), g.col_indices()
    rows, cols = [], []
    for v in order:
        nb = local[ci[ro[v]:ro[v + 1]]]
        nb = nb[nb >= 0]
        rows.append(len(nb))
        cols.append(nb)
    lro = np.concatenate([[0], np.cumsum(rows)]).astype(np.uint64)
    lc = O.CSR(len(order), lro, (np.concatenate(cols) if cols else np.zeros(0)).astype(np.uint32))
    ds = d[order]
    layer_rows = [int(np.sum(ds <= layers - l - 1)) for l in range(layers)]
    mfg = [int(np.sum(ds <= layers - l)) for l in range(layers + 1)]
    return lc, x_all[order], lab_all[order], layer_rows, len(batch.target_vertices), mfg


@pytest.mark.parametrize("kind,r,m,k,out", [("sage", 3, 1, 15, 8), ("gcn", 2, 2, 4, 8),
                                            ("sum", 4, 1, 3, 8), ("sage", 3, 1, 15, 72)])
def test_cobatch_training_matches_oracle(cuda, kind, r, m, k, out):
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.cobatch import CobatchTrainer
    from paper_2311_06837_b200.train import ModelConfig, init_weights

    dims = [48, 32, 32, out]   # out = 72: widening output layer (aggregate-first)
    L = len(dims) - 1
    g, hp, plan = _plan(2500, 10.0, 21, 2, 1, r, L, G.SamplingConfig(m, k, 3), dims)
    lr = 1e-4 if kind == "sum" else 0.5
    cfg = ModelConfig(kind, dims, lr=lr)
    w0 = init_weights(cfg, 3)
    tr = CobatchTrainer(g, cfg, plan, hp.server, hp.gpu, 0, weights=w0)
    n = g.num_vertices()
    x_all = O.make_features(n, dims[0], 1).astype(np.float32).astype(np.float64)
    lab_all = O.make_labels(n, dims[-1], 2)
    model = O.Model(KIND[kind], dims)
    w = np.concatenate([a.astype(np.float32).astype(np.float64).ravel() for a in w0])
    for epoch in range(2):
        for i, b in enumerate(plan.batches):
            lc, x, lab, layer_rows, nt, mfg = _oracle_batch(g, b, L, x_all, lab_all)
            # peel levels == the plan's peel_mfg counts (reference semantics)
            assert mfg == list(b.mfg_vertices_per_layer) == tr.geoms[i].mfg
            tr.train_batch(i)
            got = float(tr.loss_acc.item()) / nt
            loss, _ = O.train_epoch_masked(lc, x, lab, model, w, lr, nt, float(nt), nthreads=4,
                                           layer_rows=layer_rows)
            assert abs(got - loss) <= 1e-3, (epoch, i, got, loss)
    wg = np.concatenate([a.ravel() for a in tr.get_weights()])
    rms = np.sqrt(np.mean(w ** 2))
    assert np.all(np.abs(wg - w) <= 1e-4 * (np.abs(w) + rms))


def test_cobatch_geometry_multi_rank(cuda):
    """Rank views of one batch (world 3, built on one GPU): blocks follow split_batch,
    rows are (level, id) ordered, columns are the padded ids of in-batch neighbours."""
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.batch_plan import split_batch
    from paper_2311_06837_b200.cobatch import batch_geometry

    import torch
    L, world = 2, 3
    g, hp, plan = _plan(3000, 8.0, 5, 1, world, 2, L, G.SamplingConfig(1, 6, 7), [16, 16, 4])
    b = plan.batches[0]
    d = _peel_levels(g, b, L)
    shares = split_batch(b.vertices, hp.server, hp.gpu, 0, world)
    dev = torch.device("cuda", 0)
    geos = [batch_geometry(g, b.target_vertices, b.vertices, hp.server, hp.gpu,
                           0, r, world, L, dev, True) for r in range(world)]
    block = geos[0].block
    padded = {}
    for r, geo in enumerate(geos):
        assert geo.block == block
        mine = np.asarray([v for v in shares[r] if d[v] >= 0], np.int64)
        exp = mine[np.lexsort((mine, d[mine]))]
        l2g = geo.l2g.cpu().numpy().astype(np.int64)
        assert np.array_equal(l2g, exp)
        assert geo.rows_out[-1] == int(np.sum(d[exp] == 0)) == geo.loss_rows
        for i, v in enumerate(l2g):
            padded[v] = r * block + i
    ro, ci = g.row_offsets(), g.col_indices()
    for r, geo in enumerate(geos):
        lp = geo.csr.row_ptr.cpu().numpy()
        lc = geo.csr.col.cpu().numpy()
        for i, v in enumerate(geo.l2g.cpu().numpy()):
            nb = sorted(padded[u] for u in ci[ro[v]:ro[v + 1]] if u in padded)
            assert list(lc[lp[i]:lp[i + 1]]) == nb


@pytest.mark.parametrize("kind,out", [("sage", 72), ("gcn", 8)])
def test_cobatch_graph_replay_matches_eager(cuda, kind, out):
    """Per-batch CUDA graphs (LOAD, clears, step, SGD captured per batch) train exactly
    like the eager batches."""
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.cobatch import CobatchTrainer
    from paper_2311_06837_b200.train import ModelConfig, init_weights

    dims = [48, 32, 32, out]
    g, hp, plan = _plan(2500, 10.0, 21, 2, 1, 3, 3, G.SamplingConfig(1, 15, 3), dims)
    cfg = ModelConfig(kind, dims, lr=0.5)
    w0 = init_weights(cfg, 3)
    a = CobatchTrainer(g, cfg, plan, hp.server, hp.gpu, 0, weights=w0)
    b = CobatchTrainer(g, cfg, plan, hp.server, hp.gpu, 0, weights=w0)
    la = [a.train_epoch() for _ in range(4)]
    b.capture(warmup=1)                      # epoch 1 eager, then captured
    lb = [la[0]] + [b.replay_epoch(sync_loss=True) for _ in range(3)]
    np.testing.assert_allclose(lb, la, rtol=2e-6, atol=0)
    wa = np.concatenate([x.ravel() for x in a.get_weights()])
    wb = np.concatenate([x.ravel() for x in b.get_weights()])
    np.testing.assert_allclose(wb, wa, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("kind", ["sage", "gcn"])
def test_cobatch_fused_load_matches_gather_pass(cuda, kind, monkeypatch):
    """GDX_FUSED_LOAD=1 (layer-0 GEMMs read the batch's rows from the resident store
    through TMA gather4) trains bit for bit like the separate LOAD gather pass."""
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.cobatch import CobatchTrainer
    from paper_2311_06837_b200.train import ModelConfig, init_weights

    dims = [72, 32, 32, 9]
    g, hp, plan = _plan(3000, 10.0, 23, 2, 1, 3, 3, G.SamplingConfig(1, 15, 3), dims)
    cfg = ModelConfig(kind, dims, lr=0.5)
    w0 = init_weights(cfg, 3)
    res = []
    for fused in ("0", "1"):
        monkeypatch.setenv("GDX_FUSED_LOAD", fused)
        tr = CobatchTrainer(g, cfg, plan, hp.server, hp.gpu, 0, weights=w0)
        assert tr._fused_load == (fused == "1")
        losses = [tr.train_epoch() for _ in range(3)]
        res.append((losses, np.concatenate([x.ravel() for x in tr.get_weights()])))
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1])
