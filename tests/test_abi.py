"""CPU-only checks of the drop-in boundary: libgdx.so loads and exports every
entry point include/gdx.h declares; host preprocessing entry points are
bit-identical to the reference; error codes map to the reference taxonomy."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gdx.h")).read()
    return sorted(set(re.findall(r"\b(gdx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2311_06837_b200 import _lib
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    from paper_2311_06837_b200 import native
    bound = set(_lib._SIGS) | set(native._SIGS)
    assert set(syms) <= bound, sorted(set(syms) - bound)


def test_version_and_error_channel():
    from paper_2311_06837_b200 import _lib
    from paper_2311_06837_b200.errors import InputError
    assert _lib.lib().gdx_version() >= 1
    with pytest.raises(InputError):
        _lib.call("gdx_host_partition_random", 3, 0, 1, None)
    assert b"parts must be >= 1" in _lib.lib().gdx_last_error()


@pytest.mark.parametrize("n,d,seed", [(1, 0.0, 1), (2, 1.0, 3), (50, 5.0, 71), (10000, 10.0, 7),
                                      (3000, 250.0, 11)])
def test_host_generator_bit_exact(n, d, seed):
    import oracle as O
    import paper_2311_06837_b200 as G
    g = G.gen_random_graph(n, d, seed)
    c = O.gen_random_graph(n, d, seed)
    assert np.array_equal(g.row_offsets(), c.row_offsets)
    assert np.array_equal(g.col_indices(), c.cols)


def test_host_generator_errors():
    import paper_2311_06837_b200 as G
    with pytest.raises(G.InputError):
        G.gen_random_graph(0, 1.0, 1)
    with pytest.raises(G.InputError):
        G.gen_random_graph(10, 10.0, 1)


@pytest.mark.parametrize("n,parts,seed", [(10, 3, 1), (1000, 8, 5), (7, 7, 2)])
def test_host_partition_random_bit_exact(n, parts, seed):
    import oracle as O
    import paper_2311_06837_b200 as G
    g = G.Graph(n, np.zeros(n + 1, np.uint64), np.zeros(0, np.uint32))
    assert np.array_equal(G.partition_random(g, parts, seed).assignment, O.partition_random(n, parts, seed))


def test_from_edges_matches_reference_rules():
    import oracle as O
    import paper_2311_06837_b200 as G
    edges = [(0, 1), (1, 0), (2, 2), (3, 1), (0, 1), (4, 2)]
    g = G.Graph.from_edges(edges, 5)
    c = O.from_edges(edges, 5)
    assert np.array_equal(g.row_offsets(), c.row_offsets) and np.array_equal(g.col_indices(), c.cols)
    with pytest.raises(G.InputError):
        G.Graph.from_edges([(0, 9)], 5)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2311_06837_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "granndis_oracle" not in src, f


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2311_06837_b200 import _lib
    from paper_2311_06837_b200.errors import InternalError
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(InternalError):
        _lib.lib()


@pytest.mark.parametrize("n,d,seed,parts", [(120, 6.0, 2200, 2), (10000, 10.0, 7, 2), (3000, 20.0, 1, 8),
                                            (500, 3.0, 4, 7), (20000, 30.0, 9, 4), (2000, 1.5, 3, 5)])
def test_host_partition_mincut_and_hierarchical_bit_exact(n, d, seed, parts):
    import oracle as O
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.partition_host import hierarchical_partition, partition_mincut
    if not O.ref_available():
        pytest.skip("needs oracle/_ref")
    R = O.ref()
    g = G.gen_random_graph(n, d, seed)
    h = R.grr_graph_from_csr(n, g.row_offsets(), g.col_indices())
    ref = np.zeros(n, np.uint32)
    assert R.grr_partition_mincut(h, parts, 1, 0.05, ref) == 0
    assert np.array_equal(partition_mincut(g, parts, 1).assignment, ref)
    sp, gp = np.zeros(n, np.uint32), np.zeros(n, np.uint32)
    R.grr_hierarchical_partition(h, 2, 3, 1, 5, sp, gp)
    R.grr_graph_free(h)
    hp = hierarchical_partition(g, 2, 3, "mincut", 5)
    assert np.array_equal(hp.server.assignment, sp) and np.array_equal(hp.gpu.assignment, gp)


def test_golden_mincut_partition():
    import os
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.partition_host import partition_mincut
    gold = os.path.join(ROOT, "tests", "golden")
    z = np.load(os.path.join(gold, "graph_er_10k_d10_s7.npz"))
    f = np.load(os.path.join(gold, "forward_full_config1.npz"))
    g = G.Graph(int(z["n"]), z["row_offsets"], z["cols"])
    assert np.array_equal(partition_mincut(g, 2, 1).assignment, f["mincut2"])


def test_every_push_path_takes_seven_peers():
    """One box of 8 GPUs = 7 peers per rank: every peer-store entry point accepts 7 and
    rejects 8 (checked before any device work, so this runs on CPU)."""
    import ctypes as C

    from paper_2311_06837_b200 import _lib
    from paper_2311_06837_b200.errors import InputError
    L = _lib.lib()
    d7 = (C.c_int64 * 8)(*([256] * 8))
    for npeers, ok in ((7, True), (8, False)):
        rc = L.gdx_push_peers(None, 16, d7, npeers, None, None, 1, None)
        msg = L.gdx_last_error().decode()
        assert rc == 1 and (("at most 7" in msg) != ok), (npeers, msg)
        rc = L.gdx_push_rows(None, 16, None, None, d7, npeers, None, None, 1, None)
        msg = L.gdx_last_error().decode()
        assert rc == 1 and (("at most 7" in msg) != ok), (npeers, msg)
        rc = L.gdx_softmax_xent_fused_peers(None, 0, 0, 1, None, 1.0, None, None, 0, None, None, 0, None,
                                            npeers, d7, None)
        msg = L.gdx_last_error().decode()
        assert rc == 1, msg
    # the trainer: world <= 8 is accepted by the argument checks, 9 is not
    from paper_2311_06837_b200 import native
    native._bind()
    dims = (C.c_uint32 * 3)(8, 8, 4)
    ro = (C.c_uint64 * 3)(0, 1, 2)
    ci = (C.c_uint32 * 2)(1, 0)
    gr = native.TrainerGraph(2, 2, C.cast(ro, C.c_void_p), C.cast(ci, C.c_void_p))
    for world, ok in ((8, True), (9, False)):
        cfg = native.TrainerConfig(2, 2, dims, 0.1, 0, world, 0, 1, 2, 1, 0, 0, 0.0)
        h = C.c_void_p()
        rc = L.gdx_trainer_create(C.byref(cfg), C.byref(gr), C.byref(h))
        msg = L.gdx_last_error().decode()
        assert ("world must be 1..8" in msg) != ok, (world, rc, msg)
        if rc == 0:
            L.gdx_trainer_destroy(h)


@pytest.mark.parametrize("m,k,seed", [(1, 3, 5), (2, 4, 9), (3, 2, 1), (2, 0xFFFFFFFF, 0)])
def test_host_sample_trace_attribution(m, k, seed):
    """gdx_host_sample_trace (extract.hpp:49-64): the taken vertices are exactly the halo
    of extract_sampled (oracle, bit-exact to the reference), each once, at its hop, and a
    step's vertex is in the frontier of its hop."""
    import oracle as O
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.extract import sample_trace

    n = 400
    g = G.gen_random_graph(n, 8.0, 13)
    p = G.partition_random(g, 3, 2)
    inner = (p.assignment == 1).astype(np.uint8)
    cfg = G.SamplingConfig(m, k, seed)
    tr = sample_trace(g, inner, cfg)
    c = O.CSR(n, g.row_offsets(), g.col_indices())
    hop, _ = O.extract_sampled(c, p.assignment, 1, m, k, seed)
    taken = [(u, s.hop) for s in tr for u in s.taken]
    assert len({u for u, _ in taken}) == len(taken)
    halo = {int(v): int(hop[v]) for v in range(n) if hop[v] not in (0, 0xFFFFFFFF)}
    assert dict(taken) == halo
    for s in tr:
        assert (s.hop == 1 and inner[s.frontier_vertex]) or hop[s.frontier_vertex] == s.hop - 1


def test_trainer_create_validates_before_device_work():
    """gdx_trainer_create's argument checks (status + message, no GPU needed): model kind,
    layer dims, class count, world/rank, CSR pointers."""
    import ctypes as C

    from paper_2311_06837_b200 import _lib, native
    L = native._bind()
    ro = (C.c_uint64 * 3)(0, 1, 2)
    ci = (C.c_uint32 * 2)(1, 0)
    gr = native.TrainerGraph(2, 2, C.cast(ro, C.c_void_p), C.cast(ci, C.c_void_p))

    def create(kind=2, dims=(8, 8, 4), world=1, rank=0, graph=gr):
        d = (C.c_uint32 * len(dims))(*dims)
        cfg = native.TrainerConfig(kind, len(dims) - 1, d, 0.1, rank, world, 0, 1, 2, 1, 0, 0, 0.0)
        h = C.c_void_p()
        rc = L.gdx_trainer_create(C.byref(cfg), C.byref(graph), C.byref(h))
        if rc == 0:
            L.gdx_trainer_destroy(h)
        return rc, L.gdx_last_error().decode()

    assert create(kind=7) == (1, "gdx_trainer_create: unknown model kind")
    assert create(dims=(8, 0, 4))[0] == 1 and "dims must be >= 1" in create(dims=(8, 0, 4))[1]
    assert "classes must be <= 256" in create(dims=(8, 8, 300))[1]
    assert "rank < world" in create(world=2, rank=2)[1]
    bad = native.TrainerGraph(2, 2, None, None)
    assert "null CSR" in create(graph=bad)[1]
