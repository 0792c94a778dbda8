"""Pins the oracle (C restatement) before trusting it: bit-exact against the
compiled reference (oracle/_ref) and the reference tests' known answers, plus
finite-difference checks of the unpinned training extension.  CPU only."""
import ctypes as C

import numpy as np
import pytest

import oracle as O

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def ref_graph(c):
    return O.ref().grr_graph_from_csr(c.n, c.row_offsets, c.cols)


@needs_ref
@pytest.mark.parametrize("n,d,seed", [(1, 0.0, 3), (2, 1.0, 1), (120, 6.0, 2200), (1000, 50.0, 9),
                                      (10000, 10.0, 7)])
def test_generator_matches_reference(n, d, seed):
    R = O.ref()
    c = O.gen_random_graph(n, d, seed)
    h = R.grr_gen_random_graph(n, d, seed)
    ro = np.zeros(n + 1, np.uint64)
    ci = np.zeros(max(R.grr_graph_nnz(h), 1), np.uint32)
    R.grr_graph_copy(h, ro, ci)
    R.grr_graph_free(h)
    assert np.array_equal(ro, c.row_offsets) and np.array_equal(ci[:c.nnz], c.cols)


@needs_ref
def test_planted_and_from_edges_match_reference():
    R = O.ref()
    c = O.gen_planted(120, 4, 0.25, 0.02, 31)
    h = R.grr_gen_planted(120, 4, 0.25, 0.02, 31)
    ro = np.zeros(121, np.uint64)
    ci = np.zeros(R.grr_graph_nnz(h), np.uint32)
    R.grr_graph_copy(h, ro, ci)
    R.grr_graph_free(h)
    assert np.array_equal(ro, c.row_offsets) and np.array_equal(ci, c.cols)
    edges = np.array([[0, 1], [1, 2], [2, 2], [3, 1], [0, 1]], np.uint32)
    c2 = O.from_edges(edges, 4)
    h = R.grr_graph_from_edges(np.ascontiguousarray(edges.ravel()), 5, 4)
    ro = np.zeros(5, np.uint64)
    ci = np.zeros(R.grr_graph_nnz(h), np.uint32)
    R.grr_graph_copy(h, ro, ci)
    R.grr_graph_free(h)
    assert np.array_equal(ro, c2.row_offsets) and np.array_equal(ci, c2.cols)


@needs_ref
def test_streams_match_reference():
    R = O.ref()
    a = np.zeros(50 * 9)
    R.grr_make_features(50, 9, 4, a)
    assert np.array_equal(a.reshape(50, 9), O.make_features(50, 9, 4))
    w = np.zeros(7 * 5 + 2 * 7 * 7)
    assert R.grr_make_layer_weights(3, 5, 7, 11, w) == 0
    assert np.array_equal(w, np.concatenate([x.ravel() for x in O.make_layer_weights(3, 5, 7, 11)]))
    assert R.grr_mix64(12345) == O.mix64(12345)
    p = np.zeros(100, np.uint32)
    h = R.grr_gen_random_graph(100, 3.0, 1)
    R.grr_partition_random(h, 7, 5, p)
    R.grr_graph_free(h)
    assert np.array_equal(p, O.partition_random(100, 7, 5))


@needs_ref
@pytest.mark.parametrize("n,deg,F,H,L,seed", [(80, 6.0, 5, 7, 3, 33), (10000, 10.0, 64, 64, 2, 7),
                                              (300, 12.0, 20, 9, 4, 1)])
def test_forward_full_bit_exact_vs_reference(n, deg, F, H, L, seed):
    R = O.ref()
    c = O.gen_random_graph(n, deg, seed)
    x = O.make_features(n, F, seed + 1)
    ws = O.make_layer_weights(L, F, H, O.mix64(seed + 2))
    out = O.forward_full(c, x, ws, L, nthreads=4)
    h = ref_graph(c)
    rr = np.zeros(n * H)
    assert R.grr_forward_full(h, x, n, F, np.concatenate([w.ravel() for w in ws]), L, H, L, rr) == 0
    R.grr_graph_free(h)
    assert np.array_equal(out, rr.reshape(n, H))


def _ref_hops(c, assign, parts, server, m, k, seed, full):
    R = O.ref()
    h = ref_graph(c)
    hop = np.zeros(c.n, np.uint32)
    ind = C.c_uint64(0)
    if full:
        rc = R.grr_extract_full(h, assign, parts, server, m, hop, C.byref(ind))
    else:
        rc = R.grr_extract_sampled(h, assign, parts, server, m, k, seed, hop, C.byref(ind))
    R.grr_graph_free(h)
    assert rc == 0, R.grr_last_error()
    return hop, ind.value


@needs_ref
@pytest.mark.parametrize("seed", range(5))
def test_extraction_bit_exact_vs_reference(seed):
    c = O.gen_random_graph(150, 8.0, 500 + seed)
    assign = O.partition_random(150, 4, seed)
    for s in range(4):
        for L in range(4):
            hop, ind = O.extract_full(c, assign, s, L)
            rhop, rind = _ref_hops(c, assign, 4, s, L, 0, 0, True)
            assert np.array_equal(hop, rhop) and ind == rind
        for m in (0, 1, 2, 3):
            for k in (0, 1, 2, 5, O.UNLIMITED):
                hop, ind = O.extract_sampled(c, assign, s, m, k, seed)
                rhop, rind = _ref_hops(c, assign, 4, s, m, k, seed, False)
                assert np.array_equal(hop, rhop) and ind == rind


@needs_ref
def test_server_local_bit_exact_vs_reference():
    R = O.ref()
    c = O.gen_planted(60, 2, 0.5, 0.3, 12)
    assign = np.array([0] * 30 + [1] * 30, np.uint32)
    x = O.make_features(60, 4, 3)
    ws = O.make_layer_weights(3, 4, 4, 6)
    flat = np.concatenate([w.ravel() for w in ws])
    for (m, k) in ((1, 1), (2, 3), (3, O.UNLIMITED)):
        hop, _ = O.extract_sampled(c, assign, 0, m, k, 2)
        ours = O.forward_server_local(c, x, ws, 3, hop)
        h = ref_graph(c)
        out = np.zeros(30 * 4)
        assert R.grr_forward_server_local(h, hop, 0, m, int(k != O.UNLIMITED), x, 4, flat, 4, 3, 0, out) == 0
        R.grr_graph_free(h)
        assert np.array_equal(ours, out.reshape(30, 4))


@needs_ref
def test_cobatch_plan_and_split_vs_reference():
    """Single-batch plan == batch_closure + peel_mfg; split_batch pinned through the
    reference simulator's per-GPU moved / preloaded counts (sim.cpp:223-266)."""
    R = O.ref()
    c = O.gen_random_graph(400, 7.0, 12)
    servers, gpus = 2, 3
    hsp = np.zeros(400, np.uint32)
    hgp = np.zeros(400, np.uint32)
    h = ref_graph(c)
    assert R.grr_hierarchical_partition(h, servers, gpus, 0, 5, hsp, hgp) == 0
    plans = []
    for s in range(servers):
        hop, _ = O.extract_sampled(c, hsp, s, 1, 3, 5)
        p = R.grr_plan_cobatch_fixed_r(h, hop, s, 1, 1, 2, 1, 3, 5, 1, 8, 8)
        assert p
        nt, nv, nbytes = C.c_uint64(), C.c_uint64(), C.c_uint64()
        R.grr_plan_batch_sizes(p, 0, C.byref(nt), C.byref(nv), C.byref(nbytes))
        t = np.zeros(nt.value, np.uint32)
        v = np.zeros(nv.value, np.uint32)
        mfg = np.zeros(3, np.uint64)
        R.grr_plan_batch_copy(p, 0, t, v, mfg)
        universe = (hop != O.UNSEEN).astype(np.uint8)
        clo = O.batch_closure(c, universe, t, 1, 3, 5)
        assert np.array_equal(clo, v)
        assert np.array_equal(O.peel_mfg(c, clo, t, 2), mfg)
        plans.append((p, v))
    moved = np.zeros(servers * gpus, np.uint64)
    pre = np.zeros(servers * gpus, np.uint64)
    arr = (C.c_void_p * servers)(*[p for p, _ in plans])
    assert R.grr_simulate_cobatch_moved(h, hsp, hgp, servers, gpus, 2, arr, moved, pre) == 0
    # recount from the oracle's split_batch (sim.cpp:237-262)
    for s, (p, v) in enumerate(plans):
        owner = O.split_batch(v, hsp, hgp, s, gpus)
        own = np.full(400, -1)
        own[v] = owner
        for w in range(gpus):
            share = v[owner == w]
            deps = set()
            for x in share:
                for u in c.cols[c.row_offsets[x]:c.row_offsets[x + 1]]:
                    if own[u] >= 0 and own[u] != w:
                        deps.add(int(u))
            assert moved[s * gpus + w] == len(deps) * 2
            assert pre[s * gpus + w] == int(np.sum(hsp[share] != s))
    for p, _ in plans:
        R.grr_plan_free(p)
    R.grr_graph_free(h)


# ---- known answers from the reference's unit tests ------------------------------------
def test_kats_forward():
    g = O.from_edges(np.zeros((0, 2), np.uint32), 1)
    assert np.array_equal(O.forward_full(g, np.array([[1.0, -2.0]]), [np.eye(2)], 1), [[1.0, 0.0]])
    g = O.from_edges([[0, 1]], 2)
    assert np.array_equal(O.forward_full(g, np.array([[1.0], [2.0]]), [np.eye(1)], 1), [[3.0], [3.0]])


def test_kats_extraction():
    path = O.from_edges([[0, 1], [1, 2], [2, 3]], 4)
    hop, ind = O.extract_full(path, np.array([0, 0, 1, 1], np.uint32), 0, 1)
    assert list(hop) == [0, 0, 1, O.UNSEEN] and ind == 4
    toy = O.from_edges([[0, 1], [0, 2], [1, 3], [2, 3], [2, 4], [3, 4], [4, 5], [4, 7], [5, 6], [6, 7]], 8)
    a = np.array([0, 0, 0, 0, 1, 1, 1, 1], np.uint32)
    hop, _ = O.extract_full(toy, a, 0, 2)
    assert list(np.nonzero((hop != 0) & (hop != O.UNSEEN))[0]) == [4, 5, 7]
    seen = set()
    for seed in range(32):
        hop, _ = O.extract_sampled(toy, a, 0, 2, 1, seed)
        halo = list(np.nonzero((hop != 0) & (hop != O.UNSEEN))[0])
        assert len(halo) == 2 and halo[0] == 4
        seen.add(tuple(halo))
    assert (4, 5) in seen


def test_kat_batch_memory():
    # estimate_batch_memory (batch_plan.cpp:13-20): 4 layers x 100 x 64 x 4 B = 102400
    assert sum(100 * 64 * 4 for _ in range(4)) == 102400


# ---- training extension: reduction to the reference and gradient checks -----------------
def test_sum_model_reduces_to_forward_full():
    c = O.gen_random_graph(200, 6.0, 3)
    x = O.make_features(200, 8, 1)
    ws = O.make_layer_weights(3, 8, 8, 2)
    m = O.Model(O.SUM, [8, 8, 8, 8], relu_last=True)
    acts = O.model_forward(c, x, m, np.concatenate([w.ravel() for w in ws]))
    assert np.array_equal(acts[-1], O.forward_full(c, x, ws, 3))


@pytest.mark.parametrize("kind", [O.SAGE, O.GCN, O.SUM])
def test_training_gradients_finite_difference(kind):
    c = O.gen_random_graph(40, 4.0, 9)
    dims = [5, 4, 3]
    m = O.Model(kind, dims)
    rng = np.random.default_rng(kind)
    x = rng.uniform(-1, 1, (40, 5))
    labels = rng.integers(0, 3, 40).astype(np.int32)
    w = rng.uniform(-0.5, 0.5, m.weight_count())
    wc = w.copy()
    loss, grads, acts, dacts = O.train_epoch(c, x, labels, m, wc, 0.0, want_state=True)
    eps = 1e-6
    for i in rng.choice(len(w), 12, replace=False):
        wp, wm = w.copy(), w.copy()
        wp[i] += eps
        wm[i] -= eps
        lp = O.train_epoch(c, x, labels, m, wp, 0.0)
        lm = O.train_epoch(c, x, labels, m, wm, 0.0)
        assert abs((lp - lm) / (2 * eps) - grads[i]) <= 1e-6 + 1e-5 * abs(grads[i])


def test_labels_match_keyed_stream():
    if not O.ref_available():
        pytest.skip("needs oracle/_ref")
    lab = O.make_labels(300, 41, 5)
    ref = [(int(O.rng_draws(5, v, 0x6c61626c, 1)[0]) * 41) >> 64 for v in range(300)]
    assert np.array_equal(lab, ref)


def test_stream_weights_continue_the_weight_stream():
    """stream_weights (the bench / test initial weights) is make_layer_weights'
    stream (reference_gnn.cpp:18-32) continued across matrices."""
    ref = O.make_layer_weights(2, 5, 4, 77)
    got = O.stream_weights([(4, 5), (4, 4)], 77, fp32=False)
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))
    r32 = O.stream_weights([(4, 5), (4, 4)], 77)
    assert all(np.array_equal(a, b.astype(np.float32).astype(np.float64)) for a, b in zip(r32, ref))


def test_feature_rows_are_rows_of_make_features():
    full = O.make_features(300, 7, 9)
    ids = np.array([0, 5, 299, 17, 17], np.uint32)
    assert np.array_equal(O.feature_rows(ids, 7, 9), full[ids])
