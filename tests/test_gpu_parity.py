"""GPU engine vs the reference (oracle/_ref, the reference sources compiled
unmodified) and the C restatement (oracle port), through the public API.

Mirrors /root/reference/proj/tests/test_reference_gnn.cpp and test_extract.cpp:
known answers, bit-exact index sets, exactness of server-local evaluation.
FP parity: |a-b| <= 1e-4 (|b| + rms(b)) against the fp64 reference on the same
fp32-rounded inputs.
"""
import numpy as np
import pytest

import oracle as O
import paper_2311_06837_b200 as G

pytestmark = pytest.mark.gpu
TOL = 1e-4


def close(a, b, tol=TOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape
    rms = float(np.sqrt(np.mean(b * b))) if b.size else 0.0
    err = np.abs(a - b) - tol * (np.abs(b) + rms)
    assert (err.max() if err.size else -1) <= 0.0, f"excess {err.max():.3e}"


def to_graph(c: O.CSR) -> G.Graph:
    return G.Graph(c.n, c.row_offsets, c.cols)


def r32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def ref_forward(c, x, ws, L):
    return O.forward_full(c, r32(x), [r32(w) for w in ws], L)


# ---- test_reference_gnn.cpp known answers ---------------------------------------
def test_isolated_vertex_relu(cuda):
    g = G.Graph.from_edges([], 1)
    out = G.forward_full(g, np.array([[1.0, -2.0]]), [np.eye(2)], 1)
    assert out[0, 0] == 1.0 and out[0, 1] == 0.0


def test_edge_pair_sums(cuda):
    g = G.Graph.from_edges([(0, 1)], 2)
    out = G.forward_full(g, np.array([[1.0], [2.0]]), [np.eye(1)], 1)
    assert out[0, 0] == 3.0 and out[1, 0] == 3.0


def test_zero_layers_identity(cuda):
    g = G.gen_random_graph(20, 3.0, 1)
    x = G.make_features(20, 4, 9)
    assert np.array_equal(G.forward_full(g, x, [], 0), x)


def test_shape_errors(cuda):
    g = G.Graph.from_edges([(0, 1)], 2)
    with pytest.raises(G.InputError):
        G.forward_full(g, np.zeros((2, 3)), [np.eye(2)], 1)
    with pytest.raises(G.InputError):
        G.forward_full(g, np.zeros((1, 3)), [np.eye(3)], 1)


# ---- forward_full vs the compiled reference -------------------------------------------
@pytest.mark.parametrize("n,deg,F,H,L,seed", [
    (10000, 10.0, 64, 64, 2, 7),     # config 1 shape (reference Sum model)
    (3000, 25.0, 100, 64, 3, 13),    # narrowing first layer (transform-first)
    (500, 6.0, 4, 7, 3, 5),          # widening layers (aggregate-first)
    (2000, 40.0, 602, 64, 1, 11),    # Reddit-width first layer
])
def test_forward_full_matches_reference(cuda, n, deg, F, H, L, seed):
    c = O.gen_random_graph(n, deg, seed)
    g = G.gen_random_graph(n, deg, seed)
    assert np.array_equal(g.row_offsets(), c.row_offsets) and np.array_equal(g.col_indices(), c.cols)
    x = G.make_features(n, F, seed + 1)
    ws = G.make_layer_weights(L, F, H, G.mix64(seed + 2))
    out = G.forward_full(g, x, ws, L)
    ref = ref_forward(c, x, ws, L)
    if O.ref_available():
        R = O.ref()
        h = R.grr_graph_from_csr(c.n, c.row_offsets, c.cols)
        rr = np.zeros(n * H)
        flat = np.concatenate([r32(w).ravel() for w in ws])
        assert R.grr_forward_full(h, np.ascontiguousarray(r32(x)), n, F, flat, L, H, L, rr) == 0
        R.grr_graph_free(h)
        assert np.array_equal(rr.reshape(n, H), ref)  # port == reference, bit-exact
    close(out, ref)


# ---- server-local evaluation -------------------------------------------------------------
def test_server_local_full_closure_bit_exact_vs_full(cuda):
    g = G.gen_random_graph(80, 6.0, 33)
    p = G.partition_random(g, 3, 2)
    x = G.make_features(80, 5, 4)
    w = G.make_layer_weights(3, 5, 7, 5)
    full = G.forward_full(g, x, w, 3)
    for s in range(3):
        sub = G.extract_full(g, p, s, 3)
        local = G.forward_server_local(sub, g, x, w, 3, True)
        assert np.array_equal(local, full[sub.inner_vertices])  # bit exact, as the reference test


def test_server_local_matches_reference_sampled(cuda):
    c = O.gen_planted(60, 2, 0.5, 0.3, 12)
    g = to_graph(c)
    p = G.Partition(np.array([0] * 30 + [1] * 30, np.uint32), 2)
    x = G.make_features(60, 4, 3)
    w = G.make_layer_weights(3, 4, 4, 6)
    full = G.forward_full(g, x, w, 3)
    sub = G.extract_sampled(g, p, 0, G.SamplingConfig(1, 1, 2))
    local = G.forward_server_local(sub, g, x, w, 3)
    hop = sub.hop_array(60)
    ref = O.forward_server_local(c, r32(x), [r32(a) for a in w], 3, hop)
    close(local, ref)
    assert np.max(np.abs(local - full[sub.inner_vertices])) > 0.0


def test_server_local_contract(cuda):
    g = G.gen_random_graph(40, 5.0, 21)
    p = G.partition_random(g, 2, 6)
    x = G.make_features(40, 4, 1)
    w = G.make_layer_weights(4, 4, 4, 2)
    with pytest.raises(G.ContractError):
        G.forward_server_local(G.extract_full(g, p, 0, 2), g, x, w, 4, True)
    with pytest.raises(G.ContractError):
        G.forward_server_local(G.extract_sampled(g, p, 0, G.SamplingConfig(4, 2, 3)), g, x, w, 4, True)


@pytest.mark.parametrize("seed", range(5))
def test_equivalence_check_exact(cuda, seed):
    g = G.gen_random_graph(120, 6.0, 2200 + seed)
    p = G.partition_random(g, 4, seed)
    rep = G.equivalence_check(g, p, 4, seed, 8, 8)
    assert rep.max_deviation == 0.0 and len(rep.per_server_max_dev) == 4


def test_deep_hop_limit_masks_far_inputs(cuda):
    """hop_limit > layers: vertices beyond L hops are in the subgraph but must not be read."""
    c = O.gen_random_graph(300, 4.0, 8)
    g = to_graph(c)
    p = G.partition_random(g, 4, 1)
    x = G.make_features(300, 6, 2)
    w = G.make_layer_weights(2, 6, 5, 3)
    sub = G.extract_full(g, p, 1, 5)
    local = G.forward_server_local(sub, g, x, w, 2)
    ref = O.forward_server_local(c, r32(x), [r32(a) for a in w], 2, sub.hop_array(300))
    close(local, ref)


# ---- extraction: bit-exact vs the reference -------------------------------------------------
def _ref_extract(c, assign, parts, server, m, k, seed, full=False):
    if not O.ref_available():
        if full:
            return O.extract_full(c, assign, server, m)
        return O.extract_sampled(c, assign, server, m, k, seed)
    import ctypes as C
    R = O.ref()
    h = R.grr_graph_from_csr(c.n, c.row_offsets, c.cols)
    hop = np.zeros(c.n, np.uint32)
    ind = C.c_uint64(0)
    if full:
        rc = R.grr_extract_full(h, assign, parts, server, m, hop, C.byref(ind))
    else:
        rc = R.grr_extract_sampled(h, assign, parts, server, m, k, seed, hop, C.byref(ind))
    R.grr_graph_free(h)
    assert rc == 0
    return hop, int(ind.value)


@pytest.mark.parametrize("seed", range(6))
def test_extract_sampled_bit_exact(cuda, seed):
    c = O.gen_random_graph(400, 14.0, 1300 + seed)
    g = to_graph(c)
    p = G.partition_random(g, 4, seed)
    for m in (0, 1, 2, 3):
        for k in (0, 1, 2, 5, 15, G.kUnlimitedFanout):
            sub = G.extract_sampled(g, p, seed % 4, G.SamplingConfig(m, k, seed))
            hop, ind = _ref_extract(c, p.assignment, 4, seed % 4, m, k, seed)
            assert np.array_equal(sub.hop_array(c.n), hop), (m, k)
            assert sub.induced_edges == ind
            assert sub.sampled == (k != G.kUnlimitedFanout) and sub.hop_limit == m


@pytest.mark.parametrize("seed", range(4))
def test_extract_full_bit_exact(cuda, seed):
    c = O.gen_random_graph(300, 5.0, 500 + seed)
    g = to_graph(c)
    p = G.partition_random(g, 4, seed)
    for L in range(0, 5):
        for s in range(4):
            sub = G.extract_full(g, p, s, L)
            hop, ind = _ref_extract(c, p.assignment, 4, s, L, 0, 0, full=True)
            assert np.array_equal(sub.hop_array(c.n), hop)
            assert sub.induced_edges == ind


def test_extract_high_degree_sampling(cuda):
    """Reddit-like degrees (the shuffle replays ~500 swaps per frontier vertex)."""
    c = O.gen_random_graph(3000, 400.0, 11)
    g = to_graph(c)
    p = G.partition_random(g, 8, 1)
    for m, k in ((1, 15), (2, 3)):
        sub = G.extract_sampled(g, p, 3, G.SamplingConfig(m, k, 3))
        hop, ind = _ref_extract(c, p.assignment, 8, 3, m, k, 3)
        assert np.array_equal(sub.hop_array(c.n), hop)
        assert sub.induced_edges == ind


def toy8():
    return G.Graph.from_edges([(0, 1), (0, 2), (1, 3), (2, 3), (2, 4), (3, 4), (4, 5), (4, 7),
                               (5, 6), (6, 7)], 8)


def test_toy8_fixture(cuda):
    g = toy8()
    p = G.Partition(np.array([0, 0, 0, 0, 1, 1, 1, 1], np.uint32), 2)
    full2 = G.extract_full(g, p, 0, 2)
    assert list(full2.halo_vertices) == [4, 5, 7]
    saw45 = False
    for seed in range(32):
        sub = G.extract_sampled(g, p, 0, G.SamplingConfig(2, 1, seed))
        assert len(sub.halo_vertices) == 2 and sub.halo_vertices[0] == 4
        assert set(sub.halo_vertices) <= set(full2.halo_vertices)
        saw45 |= list(sub.halo_vertices) == [4, 5]
    assert saw45


def test_path4_and_helpers(cuda):
    g = G.Graph.from_edges([(0, 1), (1, 2), (2, 3)], 4)
    p = G.Partition(np.array([0, 0, 1, 1], np.uint32), 2)
    sub = G.extract_full(g, p, 0, 1)
    assert list(sub.inner_vertices) == [0, 1] and list(sub.halo_vertices) == [2]
    assert list(sub.halo_hops) == [1]
    assert sub.is_inner(0) and sub.is_halo(2) and not sub.contains(3)
    assert sub.hop_of(1) == 0 and sub.hop_of(2) == 1
    with pytest.raises(G.InputError):
        sub.hop_of(3)
    assert sub.induced_edges == 4
    assert G.neighbor_explosion_profile(g, p, 0, 3) == [(1, 3), (2, 4), (3, 4)]


def test_extract_bad_server(cuda):
    g = G.gen_random_graph(20, 3.0, 2)
    p = G.partition_random(g, 2, 1)
    with pytest.raises(G.InputError):
        G.extract_full(g, p, 5, 1)


# ---- cooperative batching -------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(4))
def test_batch_closure_and_peel(cuda, seed):
    c = O.gen_random_graph(500, 9.0, 40 + seed)
    g = to_graph(c)
    p = G.partition_random(g, 2, seed)
    sub = G.extract_sampled(g, p, 0, G.SamplingConfig(2, 4, seed))
    universe = np.zeros(c.n, np.uint8)
    universe[sub.all_vertices()] = 1
    targets = sub.inner_vertices[::3]
    for m, k in ((1, 3), (2, 2), (3, G.kUnlimitedFanout)):
        got = G.batch_closure(g, universe, targets, G.SamplingConfig(m, k, seed))
        ref = O.batch_closure(c, universe, targets, m, k, seed)
        assert np.array_equal(got, ref)
        for L in (1, 2, 3):
            assert G.peel_mfg(g, got, targets, L) == [int(v) for v in O.peel_mfg(c, got, targets, L)]


@pytest.mark.parametrize("gpus", [1, 2, 3, 8])
def test_split_batch_bit_exact(cuda, gpus):
    c = O.gen_random_graph(2000, 8.0, gpus)
    g = to_graph(c)
    servers = 2
    sp = G.partition_random(g, servers, 3)
    gp_assign = np.zeros(c.n, np.uint32)
    rng = np.random.default_rng(gpus)
    for s in range(servers):
        idx = np.nonzero(sp.assignment == s)[0]
        gp_assign[idx] = s * gpus + rng.integers(0, gpus, len(idx)).astype(np.uint32)
    gp = G.Partition(gp_assign, servers * gpus)
    for s in range(servers):
        sub = G.extract_sampled(g, sp, s, G.SamplingConfig(1, 5, 7))
        bv = sub.all_vertices()
        shares = G.split_batch(bv, sp, gp, s, gpus)
        owner = O.split_batch(bv, sp.assignment, gp.assignment, s, gpus)
        for w in range(gpus):
            assert np.array_equal(shares[w], bv[owner == w])
