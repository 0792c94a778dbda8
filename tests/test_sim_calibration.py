"""Simulator calibration: the reference's own simulate_epoch
(sim.cpp:165-283, compiled in oracle/_ref) fed with rates measured on B200 this round
(profiles/r01_calibration.json), compared with the measured multi-GPU epochs.

compute_vps is calibrated from the measured 1-GPU epoch (the simulator charges
owned_vertices * layers / compute_vps * backward_factor); internal_bw_vps is the
measured NVLink ingress per GPU in 64-wide fp32 vertex vectors.  The simulator has no
compute/communication overlap, the engine overlaps the exchange with the local-source
aggregation, so the measured N>1 epochs should not exceed the prediction by much and
should not fall far below the pure-compute share.  CPU only (no GPU needed)."""
import json
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
CAL = os.path.join(HERE, "..", "profiles", "r01_calibration.json")

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def simulate(R, h, n, N, compute_vps, bw_vps, layers, hidden, feature):
    sp = np.zeros(n, np.uint32)
    B = -(-n // N)
    gp = (np.arange(n, dtype=np.int64) // B).astype(np.uint32)  # the engine's row blocks
    tot = (np.ctypeslib.ctypes.c_double * 5)()
    wk = (np.ctypeslib.ctypes.c_double * (6 * N))()
    rc = R.grr_simulate_epoch(h, sp, gp, 1, N, compute_vps, bw_vps, bw_vps, layers, hidden, feature,
                              0, 1, 15, 0, tot, wk)
    assert rc == 0, R.grr_last_error()
    return list(tot)


@pytest.mark.parametrize("idx", [0, 1])
def test_simulator_with_b200_rates(idx):
    cal = json.load(open(CAL))
    c = cal["configs"][idx]
    R = O.ref()
    h = R.grr_gen_random_graph(c["n"], c["degree"], c["seed"])
    try:
        n, L = c["n"], c["layers"]
        ms1 = c["epoch_ms"]["1"]
        compute_vps = n * L * 2.0 / (ms1 * 1e-3)      # backward_factor 2 (SimOptions default)
        rows = []
        for key, ms in sorted(c["epoch_ms"].items(), key=lambda kv: int(kv[0])):
            N = int(key)
            bw = cal["nvlink_ingress_GBps"].get(key, 1.0) * 1e9 / cal["row_bytes"] if N > 1 else 1.0
            comp, internal, external, sync, total = simulate(R, h, n, N, compute_vps, bw, L, c["hidden"],
                                                             c["feature"])
            rows.append((N, ms, total * 1e3, comp * 1e3, internal * 1e3))
        print(f"\n{c['name']}: N  measured_ms  simulated_ms (compute + NVLink)")
        for N, ms, tot, comp, internal in rows:
            print(f"  {N}  {ms:9.3f}  {tot:9.3f} ({comp:.3f} + {internal:.3f})")
        N1 = rows[0]
        assert abs(N1[2] - N1[1]) <= 1e-6 * N1[1]            # calibration point
        for N, ms, tot, comp, internal in rows[1:]:
            assert internal > 0.0                             # ER graph: every GPU fetches
            assert 0.8 * comp <= ms <= 1.25 * tot, (N, ms, tot, comp)
    finally:
        R.grr_graph_free(h)
