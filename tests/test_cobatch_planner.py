"""Device cooperative-batch planner (gdx_cobatch_eval: every group of one R in
batched launches) against the compiled reference's plan_cobatch /
plan_cobatch_fixed_r (batch_plan.cpp:146-180), on the fixtures and budgets of the
reference's own test_batch_plan.cpp:60-170.  Integer outputs: bit-exact -- batch
count, targets, vertex universes, MFG counts, byte estimates, and the
CapacityError message naming the vertex."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

UNL = 0xFFFFFFFF
KUNLIMITED_MEMORY = (1 << 64) - 1


def _ref_plan(g, sub, layers, cfg, hidden, feat, r=0, budget=0):
    n = g.num_vertices()
    h = O.ref().grr_graph_from_csr(n, g.row_offsets(), g.col_indices())
    try:
        return O.ref_plan(h, sub.hop_array(n), sub.server_id, sub.hop_limit, sub.sampled, layers,
                          cfg.max_hop, cfg.fanout & 0xFFFFFFFF, cfg.seed, hidden, feat, r=r,
                          budget=budget)
    finally:
        O.ref().grr_graph_free(h)


def _same(plan, ref):
    assert not isinstance(ref, str), ref
    assert plan.batch_count() == len(ref)
    for b, (t, v, mfg, by) in zip(plan.batches, ref):
        assert np.array_equal(b.target_vertices, t)
        assert np.array_equal(b.vertices, v)
        assert [int(x) for x in b.mfg_vertices_per_layer] == mfg
        assert b.est_memory_bytes == by


def _planted(n, parts, p_in, p_out, seed):
    """gen_planted_partition_graph (graph.cpp:156-185) via the port (bit-identical to
    the reference, tests/test_oracle.py)."""
    from paper_2311_06837_b200.graph import Graph
    c = O.gen_planted(n, parts, p_in, p_out, seed)
    return Graph(n, c.row_offsets, c.cols)


def _fixture(name):
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.graph import Graph, Partition
    from paper_2311_06837_b200.partition_host import partition_mincut

    if name == "er80":          # test_batch_plan.cpp:60-76
        g = G.gen_random_graph(80, 6.0, 3)
        sub = G.extract_full(g, G.partition_random(g, 2, 4), 0, 2)
        return g, sub, 2, G.SamplingConfig(2, UNL, 0), 8, 8
    if name == "path":          # :78-101
        g = Graph.from_edges([(0, 1), (1, 2), (2, 3)], 4, True)
        p = Partition(np.array([0, 0, 1, 1], np.uint32), 2)
        return g, G.extract_full(g, p, 0, 1), 1, G.SamplingConfig(1, UNL, 0), 4, 4
    if name == "planted100":    # :103-110
        g = _planted(100, 2, 0.3, 0.05, 8)
        cfg = G.SamplingConfig(1, 5, 7)
        return g, G.extract_sampled(g, G.partition_random(g, 2, 2), 1, cfg), 4, cfg, 16, 16
    if name == "planted120":    # :146-163
        g = _planted(120, 4, 0.25, 0.02, 31)
        cfg = G.SamplingConfig(1, 3, 5)
        return g, G.extract_sampled(g, partition_mincut(g, 2, 3), 0, cfg), 2, cfg, 8, 8
    if name == "er400m2":       # deeper sampled closure: two hops, fanout 4
        g = G.gen_random_graph(400, 12.0, 21)
        cfg = G.SamplingConfig(2, 4, 9)
        return g, G.extract_sampled(g, G.partition_random(g, 3, 1), 2, cfg), 3, cfg, 32, 16
    raise KeyError(name)


@pytest.mark.parametrize("name", ["er80", "path", "planted100", "planted120", "er400m2"])
def test_plan_cobatch_budget_scan_matches_reference(cuda, name):
    import paper_2311_06837_b200 as G

    g, sub, layers, cfg, hidden, feat = _fixture(name)
    m = G.ModelSpec(layers, hidden, feat)
    full = G.plan_cobatch(sub, g, layers, cfg, KUNLIMITED_MEMORY, m)
    _same(full, _ref_plan(g, sub, layers, cfg, hidden, feat, budget=KUNLIMITED_MEMORY))
    fb = full.batches[0].est_memory_bytes
    for budget in (fb - 1, fb * 3 // 4, fb // 2, fb // 3):
        ref = _ref_plan(g, sub, layers, cfg, hidden, feat, budget=max(budget, 1))
        if isinstance(ref, str):
            assert ref.startswith("capacity"), ref
            with pytest.raises(G.CapacityError) as e:
                G.plan_cobatch(sub, g, layers, cfg, max(budget, 1), m)
            assert str(e.value) in ref
            continue
        _same(G.plan_cobatch(sub, g, layers, cfg, max(budget, 1), m), ref)


@pytest.mark.parametrize("name,r", [("er80", 3), ("planted120", 5), ("er400m2", 7), ("er400m2", 40)])
def test_plan_cobatch_fixed_r_matches_reference(cuda, name, r):
    import paper_2311_06837_b200 as G

    g, sub, layers, cfg, hidden, feat = _fixture(name)
    plan = G.plan_cobatch_fixed_r(sub, g, layers, cfg, r, G.ModelSpec(layers, hidden, feat))
    _same(plan, _ref_plan(g, sub, layers, cfg, hidden, feat, r=r))


def test_plan_cobatch_capacity_error_names_vertex(cuda):
    """test_batch_plan.cpp:112-121: a 3-vertex path on one server, budget 8 bytes."""
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.graph import Graph, Partition

    g = Graph.from_edges([(0, 1), (1, 2)], 3, True)
    sub = G.extract_full(g, Partition(np.zeros(3, np.uint32), 1), 0, 1)
    ref = _ref_plan(g, sub, 1, G.SamplingConfig(1, UNL, 0), 4, 4, budget=8)
    with pytest.raises(G.CapacityError) as e:
        G.plan_cobatch(sub, g, 1, G.SamplingConfig(1, UNL, 0), 8, G.ModelSpec(1, 4, 4))
    assert "single-target batch for vertex" in str(e.value) and str(e.value) in ref


def test_chunked_evaluation_matches_one_chunk(cuda, monkeypatch):
    """A workspace that holds one group at a time gives the same plan as all at once."""
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200 import batch_plan as BP

    g, sub, layers, cfg, hidden, feat = _fixture("er400m2")
    m = G.ModelSpec(layers, hidden, feat)
    a = G.plan_cobatch_fixed_r(sub, g, layers, cfg, 9, m)
    monkeypatch.setattr(BP, "_workspace_bytes", lambda dev: 1)
    b = G.plan_cobatch_fixed_r(sub, g, layers, cfg, 9, m)
    for x, y in zip(a.batches, b.batches):
        assert np.array_equal(x.vertices, y.vertices)
        assert x.mfg_vertices_per_layer == y.mfg_vertices_per_layer
