"""Committed golden fixtures (tests/golden/, generated from the unmodified reference
by tools/make_golden.py) checked against the oracle port (CPU) and the B200
engine (GPU).  These hold even where oracle/_ref cannot be built."""
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


def graph(name):
    z = load(f"graph_{name}.npz")
    return O.CSR(int(z["n"]), z["row_offsets"], z["cols"]), z


@pytest.mark.parametrize("name", ["er_10k_d10_s7", "er_120_d6_s2200", "er_400_d14_s1300", "er_3000_d400_s11"])
def test_generator_golden(name):
    c, z = graph(name)
    mine = O.gen_random_graph(int(z["n"]), float(z["degree"]), int(z["seed"]))
    assert np.array_equal(mine.row_offsets, c.row_offsets) and np.array_equal(mine.cols, c.cols)


def test_forward_full_golden_port():
    c, _ = graph("er_10k_d10_s7")
    z = load("forward_full_config1.npz")
    x = O.make_features(c.n, 64, int(z["feature_seed"]))
    ws = O.make_layer_weights(2, 64, 64, int(z["weight_seed"]))
    assert np.array_equal(O.forward_full(c, x, ws, 2, nthreads=4), z["out"])
    assert float(z["equivalence_max_dev"]) == 0.0


def test_extraction_golden_port():
    c, _ = graph("er_400_d14_s1300")
    z = load("extract_er400.npz")
    for m, k, hop, ind in zip(z["sampled_m"], z["sampled_k"], z["sampled_hop"], z["sampled_induced"]):
        h, i = O.extract_sampled(c, z["partition"], int(z["server_sampled"]), int(m), int(k), int(z["seed"]))
        assert np.array_equal(h, hop) and i == ind
    for L, hop, ind in zip(z["full_layers"], z["full_hop"], z["full_induced"]):
        h, i = O.extract_full(c, z["partition"], int(z["server_full"]), int(L))
        assert np.array_equal(h, hop) and i == ind


def test_server_local_golden_port():
    z = load("server_local_planted.npz")
    c = O.CSR(60, z["row_offsets"], z["cols"])
    ws = [z["w"][i * 16:(i + 1) * 16].reshape(4, 4) for i in range(3)]
    for hop, out in zip(z["hop"], z["out"]):
        assert np.array_equal(O.forward_server_local(c, z["x"], ws, 3, hop), out)


def test_cobatch_golden_port():
    c, _ = graph("er_120_d6_s2200")
    z = load("cobatch_er120.npz")
    for s in range(2):
        hop = z[f"hop_s{s}"]
        universe = (hop != O.UNSEEN).astype(np.uint8)
        t = z[f"s{s}_r1_b0_targets"]
        v = O.batch_closure(c, universe, t, 1, 3, 5)
        assert np.array_equal(v, z[f"s{s}_r1_b0_vertices"])
        assert np.array_equal(O.peel_mfg(c, v, t, 2), z[f"s{s}_r1_b0_mfg"])
        # r = 3: the reference's min-cut target groups -> same closures / MFG counts
        for b in range(int(z[f"s{s}_r3_batches"][0])):
            tb = z[f"s{s}_r3_b{b}_targets"]
            vb = O.batch_closure(c, universe, tb, 1, 3, 5)
            assert np.array_equal(vb, z[f"s{s}_r3_b{b}_vertices"])
            assert np.array_equal(O.peel_mfg(c, vb, tb, 2), z[f"s{s}_r3_b{b}_mfg"])


def _split_moved(c, z, owner_fn):
    sp, gp = z["server_partition"], z["gpu_partition"]
    moved = np.zeros(6, np.uint64)
    pre = np.zeros(6, np.uint64)
    for s in range(2):
        v = z[f"s{s}_r1_b0_vertices"]
        owner = owner_fn(v, sp, gp, s)
        own = np.full(c.n, -1)
        own[v] = owner
        for w in range(3):
            share = v[owner == w]
            deps = {int(u) for x in share for u in c.cols[c.row_offsets[x]:c.row_offsets[x + 1]]
                    if own[u] >= 0 and own[u] != w}
            moved[s * 3 + w] = 2 * len(deps)
            pre[s * 3 + w] = int(np.sum(sp[share] != s))
    return moved, pre


def test_split_batch_golden_port():
    c, _ = graph("er_120_d6_s2200")
    z = load("cobatch_er120.npz")
    moved, pre = _split_moved(c, z, lambda v, sp, gp, s: O.split_batch(v, sp, gp, s, 3))
    assert np.array_equal(moved, z["sim_internal_moved"]) and np.array_equal(pre, z["sim_features_preloaded"])


# ---- the B200 engine against the same fixtures ---------------------------------------------
@pytest.mark.gpu
def test_engine_golden(cuda):
    import paper_2311_06837_b200 as G

    c, _ = graph("er_10k_d10_s7")
    z = load("forward_full_config1.npz")
    g = G.Graph(c.n, c.row_offsets, c.cols)
    x = G.make_features(c.n, 64, int(z["feature_seed"]))
    ws = G.make_layer_weights(2, 64, 64, int(z["weight_seed"]))
    out = G.forward_full(g, x, ws, 2)
    ref = z["out"]  # fp64 reference on fp64 inputs; GPU runs fp32 inputs: 1e-4 scaled
    rms = np.sqrt(np.mean(ref ** 2))
    assert np.all(np.abs(out - ref) <= 1e-4 * (np.abs(ref) + rms))
    p = G.Partition(z["mincut2"], 2)
    assert G.equivalence_check(g, p, 2, 3, 64, 64).max_deviation == 0.0

    c, _ = graph("er_400_d14_s1300")
    e = load("extract_er400.npz")
    g = G.Graph(c.n, c.row_offsets, c.cols)
    part = G.Partition(e["partition"], 4)
    for m, k, hop, ind in zip(e["sampled_m"], e["sampled_k"], e["sampled_hop"], e["sampled_induced"]):
        sub = G.extract_sampled(g, part, int(e["server_sampled"]), G.SamplingConfig(int(m), int(k), int(e["seed"])))
        assert np.array_equal(sub.hop_array(c.n), hop) and sub.induced_edges == ind
    for L, hop, ind in zip(e["full_layers"], e["full_hop"], e["full_induced"]):
        sub = G.extract_full(g, part, int(e["server_full"]), int(L))
        assert np.array_equal(sub.hop_array(c.n), hop) and sub.induced_edges == ind
    prof = G.neighbor_explosion_profile(g, part, int(e["profile_server"]), 6)
    assert [s for _, s in prof] == [int(v) for v in e["profile"]]

    c, _ = graph("er_3000_d400_s11")
    r = load("extract_reddit_degree.npz")
    g = G.Graph(c.n, c.row_offsets, c.cols)
    for (m, k), hop, ind in zip(r["mk"], r["hop"], r["induced"]):
        sub = G.extract_sampled(g, G.Partition(r["partition"], 8), int(r["server"]),
                                G.SamplingConfig(int(m), int(k), int(r["seed"])))
        assert np.array_equal(sub.hop_array(c.n), hop) and sub.induced_edges == ind

    c, _ = graph("er_120_d6_s2200")
    cz = load("cobatch_er120.npz")
    g = G.Graph(c.n, c.row_offsets, c.cols)
    sp, gp = G.Partition(cz["server_partition"], 2), G.Partition(cz["gpu_partition"], 6)
    for s in range(2):
        universe = (cz[f"hop_s{s}"] != O.UNSEEN).astype(np.uint8)
        t = cz[f"s{s}_r1_b0_targets"]
        v = G.batch_closure(g, universe, t, G.SamplingConfig(1, 3, 5))
        assert np.array_equal(v, cz[f"s{s}_r1_b0_vertices"])
        assert G.peel_mfg(g, v, t, 2) == [int(a) for a in cz[f"s{s}_r1_b0_mfg"]]

    # plan_cobatch_fixed_r with the reference's min-cut target split (r = 1 and 3)
    for s in range(2):
        hop = cz[f"hop_s{s}"]
        sub = G.DependencySubgraph(s, np.nonzero(hop == 0)[0].astype(np.uint32),
                                   np.nonzero((hop != 0) & (hop != O.UNSEEN))[0].astype(np.uint32),
                                   hop[(hop != 0) & (hop != O.UNSEEN)], 0, 1, True)
        for r in (1, 3):
            plan = G.plan_cobatch_fixed_r(sub, g, 2, G.SamplingConfig(1, 3, 5), r, G.ModelSpec(2, 8, 8))
            assert plan.batch_count() == int(cz[f"s{s}_r{r}_batches"][0])
            for b, bt in enumerate(plan.batches):
                assert np.array_equal(bt.target_vertices, cz[f"s{s}_r{r}_b{b}_targets"])
                assert np.array_equal(bt.vertices, cz[f"s{s}_r{r}_b{b}_vertices"])
                assert bt.mfg_vertices_per_layer == [int(a) for a in cz[f"s{s}_r{r}_b{b}_mfg"]]
                assert bt.est_memory_bytes == int(cz[f"s{s}_r{r}_b{b}_bytes"][0])

    def owner_dev(v, sp_a, gp_a, s):
        shares = G.split_batch(v, sp, gp, s, 3)
        out = np.zeros(len(v), np.uint32)
        for w, sh in enumerate(shares):
            out[np.searchsorted(v, sh)] = w
        return out
    moved, pre = _split_moved(c, cz, owner_dev)
    assert np.array_equal(moved, cz["sim_internal_moved"]) and np.array_equal(pre, cz["sim_features_preloaded"])

    s = load("server_local_planted.npz")
    g = G.Graph(60, s["row_offsets"], s["cols"])
    ws = [s["w"][i * 16:(i + 1) * 16].reshape(4, 4) for i in range(3)]
    for hop, out, (m, k) in zip(s["hop"], s["out"], s["mk"]):
        sub = G.DependencySubgraph(0, np.nonzero(hop == 0)[0].astype(np.uint32),
                                   np.nonzero((hop != 0) & (hop != O.UNSEEN))[0].astype(np.uint32),
                                   hop[(hop != 0) & (hop != O.UNSEEN)], 0, int(m), k >= 0)
        got = G.forward_server_local(sub, g, s["x"], ws, 3)
        rr = np.sqrt(np.mean(out ** 2))
        assert np.all(np.abs(got - out) <= 1e-4 * (np.abs(out) + rr))
