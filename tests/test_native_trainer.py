"""The C-ABI trainer (gdx_trainer_*, csrc/trainer.cu) -- the epoch bench.py measures --
against the torch-orchestrated twin (train.FullGraphTrainer, same kernels in the
same order), the fp64 oracle, and a C++ host program that uses include/gdx.h only
(tests/cxx/trainer_epoch.cpp).  Parity unpinned against the reference itself (no
training path)."""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KIND = {"sage": O.SAGE, "gcn": O.GCN, "sum": O.SUM}


def _pair(kind, n, deg, dims, lr, epochs, use_graph=True, subgraph=None, seed=5, init="uniform"):
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.native import NativeTrainer
    from paper_2311_06837_b200.train import FullGraphTrainer, ModelConfig

    g = G.gen_random_graph(n, deg, seed)
    cfg = ModelConfig(kind, list(dims), lr=lr, init=init)
    w0 = O.stream_weights(O.Model(KIND[kind], dims).weight_shapes(), 3, init=init)
    sub = subgraph(g) if subgraph else None
    nat = NativeTrainer(g, cfg, weights=w0, subgraph=sub, use_graph=use_graph)
    ref = FullGraphTrainer(g, cfg, weights=w0, subgraph=sub)
    ln = [nat.train_epoch() for _ in range(epochs)]
    lp = [ref.train_epoch() for _ in range(epochs)]
    wn, wp = nat.get_weights(), ref.get_weights()
    gn, gp = nat.get_grads(), ref.get_grads()
    captured = nat.graph_captured
    nat.close()
    ref.close()
    return np.array(ln), np.array(lp), wn, wp, gn, gp, captured


@pytest.mark.parametrize("kind,dims", [("sage", [96, 64, 64, 41]), ("gcn", [32, 32, 8]), ("sum", [16, 16, 8]),
                                       ("sage", [40, 32, 32, 72])])
def test_native_epoch_matches_torch_orchestrated_trainer(cuda, kind, dims):
    """Same kernels, same order: losses agree to fp64-atomic summation order, weights
    and gradients to fp32 rounding (aggregate-first output layer included)."""
    lr = 1e-4 if kind == "sum" else 0.5
    ln, lp, wn, wp, gn, gp, captured = _pair(kind, 3001, 14.0, dims, lr, 5)
    assert captured  # epochs 3.. replay a CUDA graph
    np.testing.assert_allclose(ln, lp, rtol=2e-6, atol=0)
    for a, b in zip(wn, wp):
        np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)
    for a, b in zip(gn, gp):
        scale = np.abs(b).max() + 1e-30
        assert np.abs(a - b).max() <= 1e-4 * scale


def test_native_eager_and_graph_replay_agree(cuda):
    ln, lp, *_ = _pair("sage", 2500, 20.0, [64, 32, 41], 0.5, 6, use_graph=False)
    lg, _, *_ = _pair("sage", 2500, 20.0, [64, 32, 41], 0.5, 6, use_graph=True)
    np.testing.assert_allclose(ln, lg, rtol=2e-6, atol=0)


@pytest.mark.parametrize("kind,m,k", [("gcn", 1, 15), ("sage", 2, 4), ("sum", 2, 6)])
def test_native_subgraph_mode_matches_torch_trainer(cuda, kind, m, k):
    """EAS / preload mode: the rank's preloaded subgraph, hop-prefix masks, loss on inner."""
    import paper_2311_06837_b200 as G

    def sub(g):
        return G.extract_sampled(g, G.partition_random(g, 4, 2), 1, G.SamplingConfig(m, k, 5))
    lr = 1e-4 if kind == "sum" else 0.5
    ln, lp, wn, wp, *_ = _pair(kind, 3000, 12.0, [48, 32, 32, 8], lr, 4, subgraph=sub, seed=9)
    np.testing.assert_allclose(ln, lp, rtol=2e-6, atol=0)
    for a, b in zip(wn, wp):
        np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)


def test_native_loss_matches_oracle_ten_epochs(cuda):
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.native import NativeTrainer
    from paper_2311_06837_b200.train import ModelConfig

    n, dims, lr = 4000, [128, 64, 64, 41], 0.1
    g = G.gen_random_graph(n, 60.0, 11)
    tr = NativeTrainer(g, ModelConfig("sage", dims, lr=lr))   # weights from the (3, "weig") stream
    c = O.CSR(n, g.row_offsets(), g.col_indices())
    x = O.make_features(n, dims[0], 1).astype(np.float32).astype(np.float64)
    lab = O.make_labels(n, dims[-1], 2)
    model = O.Model(O.SAGE, dims)
    w = np.concatenate([a.ravel() for a in O.stream_weights(model.weight_shapes(), 3)])
    for e in range(10):
        lg = tr.train_epoch()
        lo = O.train_epoch(c, x, lab, model, w, lr, nthreads=os.cpu_count())
        assert abs(lg - lo) <= 1e-3, (e, lg, lo)
    tr.close()


def test_native_staged_host_inputs_match_resident(cuda):
    """End-to-end inputs: the feature block and labels copied from pinned host memory each
    step (one contiguous DMA, double-buffered) train exactly like the resident ones."""
    import torch

    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.native import NativeTrainer
    from paper_2311_06837_b200.train import ModelConfig

    n, dims = 2000, [101, 64, 41]   # odd width: host row pitch != operand pitch
    g = G.gen_random_graph(n, 12.0, 9)
    cfg = ModelConfig("sage", dims, lr=0.5)
    a = NativeTrainer(g, cfg)
    b = NativeTrainer(g, cfg)
    x = torch.from_numpy(O.make_features(n, dims[0], 1).astype(np.float32)).pin_memory().numpy()
    lab = torch.from_numpy(O.make_labels(n, dims[-1], 2)).pin_memory().numpy()
    b.stage_inputs(x, lab)
    for i in range(4):
        if i + 1 < 4:
            b.stage_inputs(x, lab)
        lb = b.step_staged()
        la = a.train_epoch()
        assert abs(la - lb) <= 1e-6 * abs(la), (i, la, lb)
    a.close()
    b.close()


def test_cxx_host_program_runs_the_epoch(cuda):
    """tests/cxx/trainer_epoch.cpp: a C++ host (gdx.h only) runs SAGE epochs; its losses
    equal the Python-driven native trainer's and the oracle's."""
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.native import NativeTrainer
    from paper_2311_06837_b200.train import ModelConfig

    exe = os.path.join(ROOT, "build", "trainer_epoch")
    if not os.path.exists(exe):
        pytest.skip("build/trainer_epoch not built")
    n, deg, dims, lr = 3000, 25.0, [602, 64, 64, 41], 0.1
    r = subprocess.run([exe, str(n), str(deg), "11", "sage", str(lr), "4", ",".join(map(str, dims))],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = json.loads(r.stdout.strip().splitlines()[-1])["losses"]
    g = G.gen_random_graph(n, deg, 11)
    tr = NativeTrainer(g, ModelConfig("sage", dims, lr=lr))
    py = [tr.train_epoch() for _ in range(4)]
    tr.close()
    np.testing.assert_allclose(got, py, rtol=2e-6, atol=0)
    c = O.CSR(n, g.row_offsets(), g.col_indices())
    x = O.make_features(n, dims[0], 1).astype(np.float32).astype(np.float64)
    model = O.Model(O.SAGE, dims)
    w = np.concatenate([a.ravel() for a in O.stream_weights(model.weight_shapes(), 3)])
    lo = O.train_epoch(c, x, O.make_labels(n, dims[-1], 2), model, w, lr, nthreads=os.cpu_count())
    assert abs(got[0] - lo) <= 1e-3


@pytest.mark.parametrize("kind,dims", [("sage", [128, 64, 64, 41]), ("gcn", [48, 64, 64, 10]),
                                       ("gcn", [48, 64, 64, 47])])
def test_native_packed24_matches_oracle_and_fp32(cuda, kind, dims):
    """cfg.packed24: the 64- and 48-wide gathered Z / dZ rows stored packed-24 (written by
    the forward GEMM and the fused dH GEMM epilogues and, for the output layer's dZ, the
    softmax kernel; read by the packed-24 aggregation).
    Losses stay within the oracle tolerance and within 24-bit rounding of the fp32 rows."""
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.native import NativeTrainer
    from paper_2311_06837_b200.train import ModelConfig

    n, lr = 4000, 0.1
    g = G.gen_random_graph(n, 60.0, 11)
    cfg = ModelConfig(kind, dims, lr=lr)
    a = NativeTrainer(g, cfg, packed24=True)
    b = NativeTrainer(g, cfg, packed24=False)
    c = O.CSR(n, g.row_offsets(), g.col_indices())
    x = O.make_features(n, dims[0], 1).astype(np.float32).astype(np.float64)
    lab = O.make_labels(n, dims[-1], 2)
    model = O.Model(KIND[kind], dims)
    w = np.concatenate([v.ravel() for v in O.stream_weights(model.weight_shapes(), 3)])
    for e in range(5):
        la, lb = a.train_epoch(), b.train_epoch()
        lo = O.train_epoch(c, x, lab, model, w, lr, nthreads=os.cpu_count())
        assert abs(la - lo) <= 1e-3, (e, la, lo)
        assert abs(la - lb) <= 2e-4 * abs(lb), (e, la, lb)
    assert a.graph_captured
    a.close()
    b.close()
