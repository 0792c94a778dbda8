"""Degree-binned load balancing (gdx_row_bins + gdx_aggregate_balanced) on skewed,
hub-heavy graphs: the chunked hub rows + row-listed light rows must equal the plain
kernels (fp32 summation order only) and fp64, with every epilogue feature, split
passes and hop prefixes; the C-ABI trainer with chunked hubs matches the oracle."""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def hub_graph(n, deg, hubs, hub_deg, seed):
    """ER(n, deg) plus `hubs` vertices joined to hub_deg random vertices each."""
    from paper_2311_06837_b200.graph import Graph
    rng = np.random.default_rng(seed)
    m = int(n * deg / 2)
    e = [rng.integers(0, n, (m, 2))]
    for h in range(hubs):
        v = rng.choice(n, hub_deg, replace=False)
        e.append(np.stack([np.full(hub_deg, h * (n // hubs)), v], 1))
    return Graph.from_edges(np.concatenate(e), n)


def scaled_close(a, b, tol):
    """|a - b| <= tol (|b| + rms(b)): fp32 summation order differs between the chunked and
    the whole-row reductions (hub rows sum ~10^4 terms)."""
    rms = float(np.sqrt(np.mean(np.asarray(b, np.float64) ** 2)))
    err = np.max(np.abs(a - b) / (np.abs(b) + rms))
    assert err <= tol, err


def _args(n, w, cuda):
    import torch
    rng = torch.Generator(device=cuda).manual_seed(0)
    src = torch.rand((n, w), device=cuda, generator=rng) - 0.5
    scale = torch.rand(n, device=cuda, generator=rng)
    add = torch.rand((n, w), device=cuda, generator=rng) - 0.5
    return src, scale, add


@pytest.mark.parametrize("w", [64, 48, 16])
def test_balanced_equals_plain_and_fp64(cuda, w):
    import torch
    from paper_2311_06837_b200.device import RowBins, Split, aggregate, dense

    g = hub_graph(30000, 6.0, 3, 9000, 1)
    dg = g.device(cuda)
    n = g.num_vertices()
    assert int(np.diff(g.row_offsets()).max()) > 8000
    bins = RowBins(g.row_offsets(), heavy_degree=500, chunk_edges=1024, max_width=64)
    assert bins.n_heavy >= 3 and bins.n_chunks > bins.n_heavy
    src, scale, add = _args(n, w, cuda)
    kw = dict(self_coef=1.0, post_scale=scale, add=add, relu=True)
    outs = []
    for b in (None, bins):
        out = dense(n, w, cuda)
        sp = Split(n, w, cuda)
        aggregate(dg, src, w, out=out, out_split=sp, bins=b, **kw)
        outs.append((out[:, :w].double().cpu().numpy(), sp.to_float().double().cpu().numpy()))
    (a, asp), (b, bsp) = outs
    scaled_close(b, a, 1e-4)     # the north_star activation contract
    scaled_close(bsp, b, 1e-5)
    # fp64 reference of the same op
    ro, ci = g.row_offsets().astype(np.int64), g.col_indices()
    x = src[:, :w].double().cpu().numpy()
    rows = np.repeat(np.arange(n), np.diff(ro))
    agg = np.zeros((n, w))
    np.add.at(agg, rows, x[ci])
    ref = np.maximum((agg + x) * scale.double().cpu().numpy()[:, None] + add[:, :w].double().cpu().numpy(), 0)
    rms = np.sqrt(np.mean(ref ** 2))
    assert np.max(np.abs(b - ref) / (np.abs(ref) + rms)) <= 1e-4
    assert np.max(np.abs(a - ref) / (np.abs(ref) + rms)) <= 1e-4


def test_balanced_split_passes_and_prefix(cuda):
    """The exchange's local/remote split (row_begin/row_end, skip + partial) and a hop
    prefix (rows < total) through the bins."""
    import torch
    from paper_2311_06837_b200._lib import call
    from paper_2311_06837_b200.device import RowBins, aggregate, dense, stream_handle

    g = hub_graph(20000, 5.0, 2, 12000, 2)
    dg = g.device(cuda)
    n, w = g.num_vertices(), 64
    bins = RowBins(g.row_offsets(), heavy_degree=300, chunk_edges=512, max_width=64)
    src, scale, _ = _args(n, w, cuda)
    lo, hi = 5000, 12000
    seg_lo = torch.empty(n, dtype=torch.int64, device=cuda)
    seg_hi = torch.empty(n, dtype=torch.int64, device=cuda)
    call("gdx_row_split", dg.row_ptr.data_ptr(), dg.col.data_ptr(), n, lo, hi, seg_lo.data_ptr(),
         seg_hi.data_ptr(), stream_handle())
    for rows in (n, 15001):
        sub = dg.slice_rows(0, rows)
        res = []
        for b in (None, bins):
            P = dense(n, w, cuda)
            out = dense(n, w, cuda)
            aggregate(sub, src, w, out=P, row_begin=seg_lo, row_end=seg_hi, bins=b)
            aggregate(sub, src, w, out=out, skip=(seg_lo, seg_hi), partial=P, self_coef=1.0, post_scale=scale,
                      bins=b)
            res.append(out[:rows, :w].double().cpu().numpy())
        scaled_close(res[1], res[0], 1e-4)


def test_native_trainer_with_chunked_hubs_matches_oracle(cuda):
    import paper_2311_06837_b200 as G  # noqa: F401
    from paper_2311_06837_b200.native import NativeTrainer
    from paper_2311_06837_b200.train import FullGraphTrainer, ModelConfig

    g = hub_graph(20000, 8.0, 3, 8000, 3)
    n, dims, lr = g.num_vertices(), [64, 32, 32, 8], 0.5
    cfg = ModelConfig("gcn", dims, lr=lr)
    model = O.Model(O.GCN, dims)
    w0 = O.stream_weights(model.weight_shapes(), 3)
    nat = NativeTrainer(g, cfg, weights=w0, heavy_degree=256)
    assert nat.info()[9] >= 3          # hub rows run chunked
    ref = FullGraphTrainer(g, cfg, weights=w0)
    c = O.CSR(n, g.row_offsets(), g.col_indices())
    x = O.make_features(n, dims[0], 1).astype(np.float32).astype(np.float64)
    lab = O.make_labels(n, dims[-1], 2)
    w = np.concatenate([a.ravel() for a in w0])
    for e in range(5):
        a, b = nat.train_epoch(), ref.train_epoch()
        lo = O.train_epoch(c, x, lab, model, w, lr, nthreads=os.cpu_count())
        assert abs(a - b) <= 1e-5 * abs(b), (e, a, b)
        assert abs(a - lo) <= 1e-3, (e, a, lo)
    nat.close()
    ref.close()


@pytest.mark.parametrize("w", [64, 32, 128, 48, 16])
def test_flat_low_degree_kernel_equals_row_groups(cuda, w):
    """GDX_AGG_FLAT (edge-flat walk over RG-row groups) sums every row's edges in the same
    ascending order as the row-group kernel: identical results, epilogue included, on a
    low-degree graph with empty rows and a few long ones."""
    import torch
    from paper_2311_06837_b200.device import Split, aggregate, dense

    g = hub_graph(100003, 2.6, 5, 300, 4)
    dg = g.device(cuda)
    n = g.num_vertices()
    src, scale, add = _args(n, w, cuda)
    res = []
    for variant in (1, 3):
        out = dense(n, w, cuda)
        sp = Split(n, w, cuda)
        aggregate(dg, src, w, out=out, out_split=sp, self_coef=1.0, post_scale=scale, add=add, relu=True,
                  variant=variant)
        res.append((out[:, :w].cpu().numpy(), sp.hi.cpu().numpy(), sp.lo.cpu().numpy()))
    for a, b in zip(*res):
        assert np.array_equal(a, b)
