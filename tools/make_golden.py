"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref, built from
/root/reference/proj/src by oracle/Makefile).  Run here (where /root/reference exists):

    python tools/make_golden.py

Each fixture stores the inputs' generating parameters and the reference's outputs:
graphs (CSR), partitions, forward_full / forward_server_local outputs (fp64),
extract_full / extract_sampled hop labels and induced-edge counts, neighbour
explosion profiles, cooperative batch plans, and the simulator's per-GPU moved
counts that pin split_batch.  Small sizes only (the files are committed).
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def ref_csr(R, h):
    n = R.grr_graph_n(h)
    ro = np.zeros(n + 1, np.uint64)
    ci = np.zeros(max(R.grr_graph_nnz(h), 1), np.uint32)
    R.grr_graph_copy(h, ro, ci)
    return ro, ci[:int(ro[-1])]


def main():
    R = O.ref()
    os.makedirs(OUT, exist_ok=True)

    # 1. graphs from the reference generators
    graphs = {}
    for name, (n, d, seed) in {"er_10k_d10_s7": (10000, 10.0, 7), "er_120_d6_s2200": (120, 6.0, 2200),
                               "er_400_d14_s1300": (400, 14.0, 1300), "er_3000_d400_s11": (3000, 400.0, 11)}.items():
        h = R.grr_gen_random_graph(n, d, seed)
        ro, ci = ref_csr(R, h)
        graphs[name] = (h, n, d, seed)
        np.savez_compressed(os.path.join(OUT, f"graph_{name}.npz"), n=n, degree=d, seed=seed,
                            row_offsets=ro, cols=ci)

    # 2. forward_full (config 1 shape, reference Sum model) + equivalence
    h, n, _, _ = graphs["er_10k_d10_s7"]
    x = np.zeros(n * 64)
    R.grr_make_features(n, 64, 3, x)
    w = np.zeros(2 * 64 * 64)
    R.grr_make_layer_weights(2, 64, 64, R.grr_mix64(4), w)
    out = np.zeros(n * 64)
    assert R.grr_forward_full(h, x, n, 64, w, 2, 64, 2, out) == 0
    part = np.zeros(n, np.uint32)
    assert R.grr_partition_mincut(h, 2, 1, 0.05, part) == 0
    dev = R.grr_equivalence_check(h, part, 2, 2, 3, 64, 64)
    np.savez_compressed(os.path.join(OUT, "forward_full_config1.npz"), feature_seed=3,
                        weight_seed=R.grr_mix64(4), F=64, H=64, layers=2, out=out.reshape(n, 64),
                        mincut2=part, equivalence_max_dev=dev)

    # 3. extraction: hop labels for (m, k) grid, partitions from the reference
    h, n, _, _ = graphs["er_400_d14_s1300"]
    part = np.zeros(n, np.uint32)
    R.grr_partition_random(h, 4, 3, part)
    cases = []
    for m in (0, 1, 2, 3):
        for k in (0, 1, 2, 5, 15, O.UNLIMITED):
            hop = np.zeros(n, np.uint32)
            ind = C.c_uint64(0)
            assert R.grr_extract_sampled(h, part, 4, 1, m, k, 9, hop, C.byref(ind)) == 0
            cases.append((m, k, hop.copy(), ind.value))
    full = []
    for L in range(5):
        hop = np.zeros(n, np.uint32)
        ind = C.c_uint64(0)
        assert R.grr_extract_full(h, part, 4, 2, L, hop, C.byref(ind)) == 0
        full.append((L, hop.copy(), ind.value))
    prof = np.zeros(6, np.uint64)
    R.grr_neighbor_explosion_profile(h, part, 4, 0, 6, prof)
    np.savez_compressed(os.path.join(OUT, "extract_er400.npz"), partition=part, server_sampled=1, seed=9,
                        sampled_m=np.array([c[0] for c in cases]), sampled_k=np.array([c[1] for c in cases], np.uint64),
                        sampled_hop=np.stack([c[2] for c in cases]), sampled_induced=np.array([c[3] for c in cases], np.uint64),
                        server_full=2, full_layers=np.array([f[0] for f in full]),
                        full_hop=np.stack([f[1] for f in full]), full_induced=np.array([f[2] for f in full], np.uint64),
                        profile_server=0, profile=prof)

    # 4. Reddit-degree sampling (deep shuffles)
    h, n, _, _ = graphs["er_3000_d400_s11"]
    part = np.zeros(n, np.uint32)
    R.grr_partition_random(h, 8, 1, part)
    hops, inds = [], []
    for (m, k) in ((1, 15), (2, 3)):
        hop = np.zeros(n, np.uint32)
        ind = C.c_uint64(0)
        R.grr_extract_sampled(h, part, 8, 3, m, k, 3, hop, C.byref(ind))
        hops.append(hop)
        inds.append(ind.value)
    np.savez_compressed(os.path.join(OUT, "extract_reddit_degree.npz"), partition=part, server=3, seed=3,
                        mk=np.array([[1, 15], [2, 3]]), hop=np.stack(hops), induced=np.array(inds, np.uint64))

    # 5. forward_server_local on sampled / full subgraphs (planted graph of test_reference_gnn)
    hp = R.grr_gen_planted(60, 2, 0.5, 0.3, 12)
    ro, ci = ref_csr(R, hp)
    assign = np.array([0] * 30 + [1] * 30, np.uint32)
    x = np.zeros(60 * 4)
    R.grr_make_features(60, 4, 3, x)
    w = np.zeros(3 * 16)
    R.grr_make_layer_weights(3, 4, 4, 6, w)
    outs, hops = [], []
    for (m, k) in ((1, 1), (2, 3), (3, O.UNLIMITED)):
        hop = np.zeros(60, np.uint32)
        ind = C.c_uint64(0)
        R.grr_extract_sampled(hp, assign, 2, 0, m, k, 2, hop, C.byref(ind))
        out = np.zeros(30 * 4)
        assert R.grr_forward_server_local(hp, hop, 0, m, int(k != O.UNLIMITED), x, 4, w, 4, 3, 0, out) == 0
        outs.append(out.reshape(30, 4))
        hops.append(hop)
    np.savez_compressed(os.path.join(OUT, "server_local_planted.npz"), row_offsets=ro, cols=ci, x=x.reshape(60, 4),
                        w=w, hop=np.stack(hops), out=np.stack(outs), mk=np.array([[1, 1], [2, 3], [3, -1]]))

    # 6. cooperative plans (r = 1 and r = 3) and the simulator's moved counts
    h, n, _, _ = graphs["er_120_d6_s2200"]
    sp = np.zeros(n, np.uint32)
    gp = np.zeros(n, np.uint32)
    R.grr_hierarchical_partition(h, 2, 3, 1, 5, sp, gp)
    rec = {"server_partition": sp, "gpu_partition": gp}
    plans = []
    for s in range(2):
        hop = np.zeros(n, np.uint32)
        ind = C.c_uint64(0)
        R.grr_extract_sampled(h, sp, 2, s, 1, 3, 5, hop, C.byref(ind))
        rec[f"hop_s{s}"] = hop
        for r in (1, 3):
            p = R.grr_plan_cobatch_fixed_r(h, hop, s, 1, 1, 2, 1, 3, 5, r, 8, 8)
            nb = R.grr_plan_batches(p)
            for b in range(nb):
                nt, nv, nbytes = C.c_uint64(), C.c_uint64(), C.c_uint64()
                R.grr_plan_batch_sizes(p, b, C.byref(nt), C.byref(nv), C.byref(nbytes))
                t = np.zeros(nt.value, np.uint32)
                v = np.zeros(nv.value, np.uint32)
                mfg = np.zeros(3, np.uint64)
                R.grr_plan_batch_copy(p, b, t, v, mfg)
                rec[f"s{s}_r{r}_b{b}_targets"] = t
                rec[f"s{s}_r{r}_b{b}_vertices"] = v
                rec[f"s{s}_r{r}_b{b}_mfg"] = mfg
                rec[f"s{s}_r{r}_b{b}_bytes"] = np.array([nbytes.value], np.uint64)
            rec[f"s{s}_r{r}_batches"] = np.array([nb])
            if r == 1:
                plans.append(p)
            else:
                R.grr_plan_free(p)
    moved = np.zeros(6, np.uint64)
    pre = np.zeros(6, np.uint64)
    arr = (C.c_void_p * 2)(*plans)
    assert R.grr_simulate_cobatch_moved(h, sp, gp, 2, 3, 2, arr, moved, pre) == 0
    rec["sim_internal_moved"] = moved
    rec["sim_features_preloaded"] = pre
    np.savez_compressed(os.path.join(OUT, "cobatch_er120.npz"), **rec)
    for p in plans:
        R.grr_plan_free(p)
    for (hh, *_rest) in graphs.values():
        R.grr_graph_free(hh)
    R.grr_graph_free(hp)
    print("golden fixtures written to", OUT)
    for f in sorted(os.listdir(OUT)):
        print(f"  {f}: {os.path.getsize(os.path.join(OUT, f))} bytes")


if __name__ == "__main__":
    main()
