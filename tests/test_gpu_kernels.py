"""GPU parity of the individual kernels through the C ABI (K1 aggregate, K2 tcgen05
GEMM, K7 init) against fp64 / exact references.  Tolerance: |a-b| <= 1e-4 (|b| + rms(b))."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def close(a, b, tol=TOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    rms = float(np.sqrt(np.mean(b * b))) if b.size else 0.0
    err = np.abs(a - b) - tol * (np.abs(b) + rms)
    worst = float(err.max()) if err.size else -1.0
    assert worst <= 0.0, f"max excess {worst:.3e} (rms {rms:.3e})"


@pytest.fixture(scope="module")
def gdx(cuda):
    import torch
    from paper_2311_06837_b200 import device as D
    torch.manual_seed(0)
    return D


def _split(D, x, cuda):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(cuda)
    s = D.Split(x.shape[0], x.shape[1], cuda)
    return s.fill_from(t, x.shape[1])


@pytest.mark.parametrize("m,n,k", [(1, 8, 16), (128, 64, 64), (300, 128, 602), (1000, 41, 64),
                                   (257, 96, 128), (64, 608, 200), (4000, 128, 608), (129, 256, 1000)])
def test_gemm_tcgen05_matches_fp64(gdx, cuda, m, n, k):
    import torch
    rng = np.random.default_rng(m * 7 + n + k)
    a = rng.uniform(-0.5, 0.5, (m, k))
    b = rng.uniform(-0.5, 0.5, (n, k))
    A, B = _split(gdx, a, cuda), _split(gdx, b, cuda)
    c = gdx.dense(m, n, cuda)
    gdx.gemm_tn(A, B, c0=c)
    torch.cuda.synchronize()
    ref = a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T
    close(c[:m, :n].double().cpu().numpy(), ref)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(128, 64, 64), (300, 128, 602), (96, 602, 5000), (130, 256, 700)])
def test_gemm_operand_majors(gdx, cuda, a_mn, b_mn, m, n, k):
    """MN-major operands (A stored [k][m], B stored [k][n]) as used by dW = G^T H."""
    import torch
    rng = np.random.default_rng(m + n + k + 10 * a_mn + 20 * b_mn)
    a = rng.uniform(-0.5, 0.5, (m, k))
    b = rng.uniform(-0.5, 0.5, (n, k))
    A = _split(gdx, a.T.copy() if a_mn else a, cuda)
    B = _split(gdx, b.T.copy() if b_mn else b, cuda)
    c = gdx.dense(m, n, cuda)
    gdx.gemm_tn(A, B, c0=c, a_mn=bool(a_mn), b_mn=bool(b_mn))
    torch.cuda.synchronize()
    ref = a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T
    close(c[:m, :n].double().cpu().numpy(), ref)


@pytest.mark.parametrize("split_k", [3, 64])
def test_gemm_mn_splitk(gdx, cuda, split_k):
    """The trainer's weight-gradient shape: M = 96, N = 602, K = rows, split-K."""
    import torch
    from paper_2311_06837_b200._lib import call
    rng = np.random.default_rng(split_k)
    m, n, k = 96, 602, 20000
    g = rng.uniform(-1, 1, (k, m))
    h = rng.uniform(-1, 1, (k, n))
    A, B = _split(gdx, g, cuda), _split(gdx, h, cuda)
    ld = 608
    ws = torch.zeros(split_k * m, ld, dtype=torch.float32, device=cuda)
    gdx.gemm_tn(A, B, c0=ws, split_k=split_k, a_mn=True, b_mn=True)
    out = torch.zeros(m, ld, dtype=torch.float32, device=cuda)
    call("gdx_splitk_reduce", ws.data_ptr(), split_k, m * ld, m, n, ld, out.data_ptr(), None, 0.0,
         None, None, gdx.stream_handle())
    torch.cuda.synchronize()
    ref = g.astype(np.float32).astype(np.float64).T @ h.astype(np.float32).astype(np.float64)
    close(out[:m, :n].double().cpu().numpy(), ref)


def test_gemm_epilogue_split_scale_relu(gdx, cuda):
    import torch
    rng = np.random.default_rng(5)
    m, n, k = 333, 128, 96
    a = rng.uniform(-1, 1, (m, k))
    b = rng.uniform(-1, 1, (n, k))
    scale = rng.uniform(0.1, 2.0, m).astype(np.float32)
    A, B = _split(gdx, a, cuda), _split(gdx, b, cuda)
    c0, c1 = gdx.dense(m, 64, cuda), gdx.dense(m, 64, cuda)
    sp = gdx.Split(m, n, cuda)
    sc = torch.from_numpy(scale).to(cuda)
    gdx.gemm_tn(A, B, c0=c0, c1=c1, split=64, row_scale=sc, relu=True, out_split=sp)
    torch.cuda.synchronize()
    ref = np.maximum((a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T)
                     * scale[:, None], 0)
    close(c0[:m, :64].double().cpu().numpy(), ref[:, :64])
    close(c1[:m, :64].double().cpu().numpy(), ref[:, 64:])
    close(sp.to_float().double().cpu().numpy(), ref)


@pytest.mark.parametrize("split_k", [2, 7])
def test_gemm_splitk_reduce(gdx, cuda, split_k):
    import torch
    from paper_2311_06837_b200._lib import call
    rng = np.random.default_rng(split_k)
    m, n, k = 128, 64, 5000
    a = rng.uniform(-1, 1, (m, k))
    b = rng.uniform(-1, 1, (n, k))
    A, B = _split(gdx, a, cuda), _split(gdx, b, cuda)
    ws = torch.zeros(split_k * m * 64, dtype=torch.float32, device=cuda).view(split_k * m, 64)
    gdx.gemm_tn(A, B, c0=ws, split_k=split_k)
    out = gdx.dense(m, n, cuda)
    call("gdx_splitk_reduce", ws.data_ptr(), split_k, m * 64, m, n, 64, out.data_ptr(), None, 0.0,
         None, None, gdx.stream_handle())
    torch.cuda.synchronize()
    ref = a.astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T
    close(out[:m, :n].double().cpu().numpy(), ref)


def _rand_csr(n, deg, seed):
    import oracle as O
    return O.gen_random_graph(n, deg, seed)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("width", [1, 3, 4, 8, 12, 41, 44, 48, 64, 128, 130, 192, 256, 602])
def test_aggregate_widths(gdx, cuda, width, variant):
    """Warp-per-row (variant 0, auto) and lane-group-per-row (GDX_AGG_ROWS) kernels."""
    import torch
    from paper_2311_06837_b200.device import DeviceCSR
    g = _rand_csr(700, 9.0, width)
    rng = np.random.default_rng(width)
    x = rng.uniform(-1, 1, (g.n, width)).astype(np.float32)
    add = rng.uniform(-1, 1, (g.n, width)).astype(np.float32)
    scale = rng.uniform(0.5, 1.5, g.n).astype(np.float32)
    dg = DeviceCSR.upload(g.row_offsets, g.cols, cuda)
    X = gdx.dense(g.n, width, cuda)
    X[:, :width] = torch.from_numpy(x).to(cuda)
    Add = gdx.dense(g.n, width, cuda)
    Add[:, :width] = torch.from_numpy(add).to(cuda)
    out = gdx.dense(g.n, width, cuda)
    sp = gdx.Split(g.n, width, cuda)
    gdx.aggregate(dg, X, width, out=out, out_split=sp, self_coef=1.0,
                  post_scale=torch.from_numpy(scale).to(cuda), add=Add, relu=True, variant=variant)
    torch.cuda.synchronize()
    ro, ci = g.row_offsets.astype(np.int64), g.cols.astype(np.int64)
    xd = x.astype(np.float64)
    ref = xd.copy()
    for v in range(g.n):
        ref[v] += xd[ci[ro[v]:ro[v + 1]]].sum(0)
    ref = np.maximum(ref * scale[:, None] + add, 0)
    close(out[:, :width].double().cpu().numpy(), ref)
    close(sp.to_float().double().cpu().numpy(), ref)


def test_aggregate_slice_and_self_base(gdx, cuda):
    """Owned-row slice [lo, hi) with the self term taken at self_base + row (multi-GPU layout)."""
    import torch
    from paper_2311_06837_b200.device import DeviceCSR
    g = _rand_csr(500, 12.0, 3)
    x = np.random.default_rng(1).uniform(-1, 1, (g.n, 64)).astype(np.float32)
    dg = DeviceCSR.upload(g.row_offsets, g.cols, cuda)
    X = torch.from_numpy(x).to(cuda)
    lo, hi = 123, 377
    out = gdx.dense(hi - lo, 64, cuda)
    gdx.aggregate(dg.slice_rows(lo, hi), X, 64, out=out, self_coef=1.0, self_base=lo)
    torch.cuda.synchronize()
    ro, ci = g.row_offsets.astype(np.int64), g.cols.astype(np.int64)
    ref = np.stack([x[v].astype(np.float64) + x[ci[ro[v]:ro[v + 1]]].astype(np.float64).sum(0)
                    for v in range(lo, hi)])
    close(out[:, :64].double().cpu().numpy(), ref)


def test_init_streams_bit_exact(cuda):
    import oracle as O
    from paper_2311_06837_b200 import make_features, make_layer_weights
    assert np.array_equal(make_features(313, 7, 9), O.make_features(313, 7, 9))
    ws = make_layer_weights(3, 5, 4, 77)
    wo = O.make_layer_weights(3, 5, 4, 77)
    for a, b in zip(ws, wo):
        assert np.array_equal(a, b)


def test_labels_bit_exact(cuda):
    import torch
    import oracle as O
    from paper_2311_06837_b200._lib import call
    from paper_2311_06837_b200.device import stream_handle
    out = torch.empty(5000, dtype=torch.int32, device=cuda)
    call("gdx_init_labels", 11, 0, 5000, 41, out.data_ptr(), stream_handle())
    assert np.array_equal(out.cpu().numpy(), O.make_labels(5000, 41, 11))


@pytest.mark.parametrize("m,mask_ld,unscaled", [(517, 64, True), (1_100_003, 64, True), (1_100_003, 64, False),
                                                 (517, 65, True), (1_100_003, 65, True)])
def test_gemm_mask_epilogue_fused_backward(gdx, cuda, m, mask_ld, unscaled):
    """dH GEMM epilogue of the trainer: ReLU-backward mask, split copy (unscaled or scaled),
    row scale. A 16-byte mask pitch takes the TMA variant (mask tile TMA-loaded, c0 and
    the split copy TMA-stored); pitch 65 the register epilogue (EW 16, or the staged
    EW 8 form at >= 4 M rows)."""
    import torch
    rng = np.random.default_rng(11)
    n, k = 64, 96
    g = rng.uniform(-1, 1, (m, k))
    w = rng.uniform(-1, 1, (k, n))          # stored [k][n]: MN-major B
    mask = rng.uniform(-1, 1, (m, n)).astype(np.float32)
    scale = rng.uniform(0.1, 2.0, m).astype(np.float32)
    A, B = _split(gdx, g, cuda), _split(gdx, w, cuda)
    out = gdx.dense(m, n, cuda)
    sp = gdx.Split(m, n, cuda)
    mk = torch.zeros((m, mask_ld), dtype=torch.float32, device=cuda)
    mk[:, :n] = torch.from_numpy(mask).to(cuda)
    gdx.gemm_tn(A, B, c0=out, b_mn=True, mask=mk[:, :n],
                row_scale=torch.from_numpy(scale).to(cuda), out_split=sp, split_unscaled=unscaled)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([rng.integers(0, m, 4000), np.arange(max(0, m - 300), m)]))
    dh = g[rows].astype(np.float32).astype(np.float64) @ w.astype(np.float32).astype(np.float64)
    gref = np.where(mask[rows] > 0, dh, 0.0)
    ri = torch.from_numpy(rows).to(cuda)
    close(sp.to_float()[ri].double().cpu().numpy(), gref if unscaled else gref * scale[rows, None])
    close(out[ri, :n].double().cpu().numpy(), gref * scale[rows, None])


@pytest.mark.parametrize("relu,split", [(False, 64), (True, 64), (False, 40)])
def test_gemm_staged_split_outputs(gdx, cuda, relu, split):
    """Long forward GEMM (staged epilogue: TMA bulk stores of swizzled 32 x 16 boxes, the
    register path for groups straddling the split): c0/c1 column split + split copy."""
    import torch
    rng = np.random.default_rng(5)
    m, n, k = 1_050_001, 128, 64
    a = rng.uniform(-1, 1, (m, k))
    b = rng.uniform(-1, 1, (n, k))
    A, B = _split(gdx, a, cuda), _split(gdx, b, cuda)
    c0, c1 = gdx.dense(m, split, cuda), gdx.dense(m, n - split, cuda)
    sp = gdx.Split(m, n, cuda)
    gdx.gemm_tn(A, B, c0=c0, c1=c1, split=split, relu=relu, out_split=sp)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([rng.integers(0, m, 4000), np.arange(m - 200, m)]))
    ref = a[rows].astype(np.float32).astype(np.float64) @ b.astype(np.float32).astype(np.float64).T
    if relu:
        ref = np.maximum(ref, 0)
    ri = torch.from_numpy(rows).to(cuda)
    close(c0[ri, :split].double().cpu().numpy(), ref[:, :split])
    close(c1[ri, :n - split].double().cpu().numpy(), ref[:, split:])
    close(sp.to_float()[ri].double().cpu().numpy(), ref)


def _gathered_split(gdx, S, idx, cuda):
    """rows idx of split S as a fresh Split (what gdx_gather_split_rows produces)."""
    import torch
    out = gdx.Split(idx.numel(), S.cols, cuda)
    ii = idx.long()
    out.hi.view(-1, out.ld)[:idx.numel()] = S.hi.view(-1, S.ld)[ii][:, :out.ld]
    out.lo.view(-1, out.ld)[:idx.numel()] = S.lo.view(-1, S.ld)[ii][:, :out.ld]
    return out


@pytest.mark.parametrize("m,k,n", [(1000, 128, 128), (517, 100, 64), (300, 64, 256)])
def test_gemm_gathered_a_rows(gdx, cuda, m, k, n):
    """TMA gather4 of a K-major A (the cooperative batch's LOAD fused into its forward
    GEMM): bit-identical to gathering the rows first, c0/c1 split outputs included."""
    import torch
    rng = np.random.default_rng(m + k)
    src_rows = 5000
    A = _split(gdx, rng.uniform(-1, 1, (src_rows, k)), cuda)
    B = _split(gdx, rng.uniform(-1, 1, (n, k)), cuda)
    idx = torch.from_numpy(rng.integers(0, src_rows, m).astype(np.int32)).to(cuda)
    split = n // 2
    outs = []
    for gathered in (True, False):
        c0, c1 = gdx.dense(m, split, cuda), gdx.dense(m, n - split, cuda)
        if gathered:
            gdx.gemm_tn(A, B, c0=c0, c1=c1, split=split, a_rows=idx)
        else:
            gdx.gemm_tn(_gathered_split(gdx, A, idx, cuda), B, c0=c0, c1=c1, split=split)
        outs.append((c0.clone(), c1.clone()))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    c = gdx.dense(m, n, cuda)
    gdx.gemm_tn(A, B, c0=c, a_rows=idx, simt=True)   # the SIMT reference gathers too
    close(torch.cat(outs[0], 1).double().cpu().numpy(), c[:, :n].double().cpu().numpy())


@pytest.mark.parametrize("kk,n,sk", [(1000, 128, 4), (4099, 64, 8), (200, 256, 1)])
def test_gemm_gathered_b_rows(gdx, cuda, kk, n, sk):
    """TMA gather4 of an MN-major B over k (the cooperative batch's dW GEMM reading its
    input rows from the resident store): bit-identical to gathering first."""
    import torch
    rng = np.random.default_rng(kk)
    src_rows, m = 9000, 64
    G = _split(gdx, rng.uniform(-1, 1, (kk, m)), cuda)      # [k][m]: MN-major A
    X = _split(gdx, rng.uniform(-1, 1, (src_rows, n)), cuda)  # source [rows][n]
    idx = torch.from_numpy(rng.choice(src_rows, kk, replace=False).astype(np.int32)).to(cuda)
    outs = []
    for gathered in (True, False):
        ws = torch.zeros((sk * m, gdx.pad4(n)), dtype=torch.float32, device=cuda)
        if gathered:
            gdx.gemm_tn(G, X, c0=ws, split_k=sk, a_mn=True, b_mn=True, b_rows=idx)
        else:
            gdx.gemm_tn(G, _gathered_split(gdx, X, idx, cuda), c0=ws, split_k=sk, a_mn=True, b_mn=True)
        outs.append(ws.clone())
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    tot = outs[0].view(sk, m, -1).sum(0)[:, :n].double().cpu().numpy()
    xg = X.to_float()[idx.long()].double().cpu().numpy()
    close(tot, G.to_float().double().cpu().numpy().T @ xg)


def _interleaved_p24(cuda, ref, m, n):
    """packed-24 planes of fp32 `ref` [m, n] in the trainer's interleaved rows (3 n bytes
    per row: high plane then low plane) via gdx_pack24 -- (buffer, hi addr, lo addr)."""
    import torch
    from paper_2311_06837_b200._lib import call
    from paper_2311_06837_b200.device import stream_handle
    hi = torch.zeros(m * n, dtype=torch.int16, device=cuda)
    lo = torch.zeros(m * n, dtype=torch.uint8, device=cuda)
    call("gdx_pack24", ref.data_ptr(), ref.stride(0), m, n, hi.data_ptr(), lo.data_ptr(), n, stream_handle())
    buf = torch.zeros((m, 3 * n), dtype=torch.uint8, device=cuda)
    buf[:, :2 * n] = hi.view(torch.uint8).view(m, 2 * n)
    buf[:, 2 * n:] = lo.view(m, n)
    return buf.view(-1)


@pytest.mark.parametrize("case", ["sage-fwd", "gcn-fwd", "dh-mask"])
def test_gemm_packed24_outputs(gdx, cuda, case):
    """Packed-24 GEMM outputs (generic epilogue: SAGE forward's c1 / GCN forward's
    row-scaled c0; TMA-store mask epilogue: the dH GEMM) are exactly the packed-24
    rounding of the fp32 outputs, in the trainer's interleaved row layout."""
    import torch
    rng = np.random.default_rng(7)
    m, k = 1000, 96
    n = 128 if case == "sage-fwd" else 64
    A = _split(gdx, rng.uniform(-1, 1, (m, k)), cuda)
    kw, bmn = {}, case == "dh-mask"
    B = _split(gdx, rng.uniform(-1, 1, (k, n)) if bmn else rng.uniform(-1, 1, (n, k)), cuda)
    if case == "gcn-fwd":
        kw["row_scale"] = torch.rand(m, device=cuda) + 0.5
    if case == "dh-mask":
        kw.update(mask=torch.randn(m, n, device=cuda), row_scale=torch.rand(m, device=cuda) + 0.5,
                  out_split=gdx.Split(m, n, cuda), split_unscaled=True)
    w24 = 64
    buf = torch.zeros(m * 3 * w24, dtype=torch.uint8, device=cuda)
    p24 = (buf.data_ptr(), buf.data_ptr() + 2 * w24, 3 * w24 // 2, 3 * w24)
    ref = gdx.dense(m, n, cuda)
    if case == "sage-fwd":
        S = gdx.dense(m, 64, cuda)
        gdx.gemm_tn(A, B, c0=S, split=64, p24=p24 + (1,))
        gdx.gemm_tn(A, B, c0=ref, **kw)
        want = ref[:, 64:128].contiguous()
        torch.cuda.synchronize()
        assert torch.equal(S, ref[:, :64])
    else:
        gdx.gemm_tn(A, B, b_mn=bmn, p24=p24 + (0,), **kw)
        gdx.gemm_tn(A, B, c0=ref, b_mn=bmn, **kw)
        want = ref[:, :64].contiguous()
    exp = _interleaved_p24(cuda, want, m, w24)
    torch.cuda.synchronize()
    assert torch.equal(buf, exp)


def test_aggregate_packed24_interleaved_rows(gdx, cuda):
    """ld_src_lo8: a packed-24 source in interleaved rows aggregates exactly like the
    same values in two separate planes."""
    import torch
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200._lib import call
    from paper_2311_06837_b200.device import stream_handle
    n, w = 3000, 64
    g = G.gen_random_graph(n, 30.0, 5)
    dg = g.device(cuda)
    x = torch.randn(n, w, device=cuda)
    inter = _interleaved_p24(cuda, x, n, w)
    hi = torch.zeros(n * w, dtype=torch.int16, device=cuda)
    lo = torch.zeros(n * w, dtype=torch.uint8, device=cuda)
    call("gdx_pack24", x.data_ptr(), w, n, w, hi.data_ptr(), lo.data_ptr(), w, stream_handle())
    outs = []
    for src, lo8, ldl in ((hi.view(n, w), lo, 0), (torch.as_strided(inter.view(torch.int16), (n, w), (3 * w // 2, 1)),
                                                    inter.data_ptr() + 2 * w, 3 * w)):
        out = gdx.dense(n, w, cuda)
        gdx.aggregate(dg, src, w, out=out, self_coef=1.0, src_lo8=lo8, ld_src_lo8=ldl)
        outs.append(out)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("width", [64, 30])
def test_grad_prepare(gdx, cuda, width):
    """g = dH * (H > 0) -> split(g) and gs = g * scale (vector and scalar forms)."""
    import torch
    from paper_2311_06837_b200._lib import call
    rng = np.random.default_rng(width)
    n = 1000
    dh = rng.uniform(-1, 1, (n, width)).astype(np.float32)
    h = rng.uniform(-1, 1, (n, width)).astype(np.float32)
    sc = rng.uniform(0.5, 2, n).astype(np.float32)
    DH, H = (torch.from_numpy(a).to(cuda) for a in (dh, h))
    S = torch.from_numpy(sc).to(cuda)
    gs = torch.zeros(n, width, device=cuda)
    sp = gdx.Split(n, width, cuda)
    call("gdx_grad_prepare", DH.data_ptr(), width, H.data_ptr(), width, n, width, S.data_ptr(), None, 0,
         gs.data_ptr(), width, sp.hi.data_ptr(), sp.lo.data_ptr(), sp.ld, gdx.stream_handle())
    torch.cuda.synchronize()
    g = np.where(h > 0, dh, 0).astype(np.float64)
    close(sp.to_float().double().cpu().numpy(), g)
    close(gs.double().cpu().numpy(), g * sc[:, None])


def test_gather_split_rows_exact(gdx, cuda):
    """The cooperative-batch LOAD: rows idx of a split store, bit-exact."""
    import torch
    from paper_2311_06837_b200._lib import call
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (5000, 128)).astype(np.float32)
    src = _split(gdx, x, cuda)
    idx = np.sort(rng.choice(5000, 777, replace=False)).astype(np.int32)
    I = torch.from_numpy(idx).to(cuda)
    out = gdx.Split(777, 128, cuda)
    call("gdx_gather_split_rows", src.hi.data_ptr(), src.lo.data_ptr(), src.ld, I.data_ptr(), 777, 128,
         out.hi.data_ptr(), out.lo.data_ptr(), out.ld, gdx.stream_handle())
    torch.cuda.synchronize()
    a = src.hi.view(5000, src.ld)[I.long()].cpu().numpy()
    b = out.hi.view(777, out.ld).cpu().numpy()
    assert np.array_equal(a, b)
    assert np.array_equal(src.lo.view(5000, src.ld)[I.long()].cpu().numpy(), out.lo.view(777, out.ld).cpu().numpy())


@pytest.mark.parametrize("classes,ld", [(1, 8), (8, 8), (41, 48), (47, 64), (64, 64), (72, 72),
                                        (128, 128), (172, 176)])
def test_softmax_xent_fused(gdx, cuda, classes, ld):
    """Fused loss head: loss sum, g = (softmax - onehot)/count as split copy and as
    gs = g * row_scale (vector form up to 128 classes, warp form beyond)."""
    import torch
    from paper_2311_06837_b200._lib import call
    rng = np.random.default_rng(classes)
    n = 3001
    z = rng.normal(0, 2, (n, classes)).astype(np.float32)
    y = rng.integers(0, classes, n).astype(np.int32)
    sc = rng.uniform(0.5, 2, n).astype(np.float32)
    Z = torch.zeros(n, ld, device=cuda)
    Z[:, :classes] = torch.from_numpy(z).to(cuda)
    Y, S = torch.from_numpy(y).to(cuda), torch.from_numpy(sc).to(cuda)
    gs = torch.zeros(n, ld, device=cuda)
    sp = gdx.Split(n, ld, cuda)
    loss = torch.zeros(1, dtype=torch.float64, device=cuda)
    call("gdx_softmax_xent_fused", Z.data_ptr(), ld, n, classes, Y.data_ptr(), 1.0 / n, None, 0, S.data_ptr(),
         gs.data_ptr(), ld, sp.hi.data_ptr(), sp.lo.data_ptr(), sp.ld, loss.data_ptr(), gdx.stream_handle())
    torch.cuda.synchronize()
    zd = z.astype(np.float64)
    m = zd.max(1, keepdims=True)
    lse = m[:, 0] + np.log(np.exp(zd - m).sum(1))
    p = np.exp(zd - lse[:, None])
    g = p.copy()
    g[np.arange(n), y] -= 1.0
    g /= n
    assert abs(float(loss.item()) - float((lse - zd[np.arange(n), y]).sum())) <= 1e-4 * n
    close(sp.to_float()[:, :classes].double().cpu().numpy(), g)
    close(gs[:, :classes].double().cpu().numpy(), g * sc[:, None])
    assert float(gs[:, classes:].abs().max().item() if ld > classes else 0.0) == 0.0


@pytest.mark.parametrize("classes,ld", [(41, 64), (47, 64), (8, 8), (64, 64), (100, 128)])
def test_softmax_xent_fused_p24(gdx, cuda, classes, ld):
    """Packed-24 gs (the trainer's interleaved rows: u16 high plane then u8 low plane,
    3 ld bytes per row) is the fp32 gs of gdx_softmax_xent_fused rounded by gdx_pack24:
    bit-exact; the split copy and the loss are unchanged."""
    import torch
    from paper_2311_06837_b200._lib import call
    rng = np.random.default_rng(classes + 1000)
    n = 2999
    z = rng.normal(0, 2, (n, classes)).astype(np.float32)
    y = rng.integers(0, classes, n).astype(np.int32)
    sc = rng.uniform(0.5, 2, n).astype(np.float32)
    Z = torch.zeros(n, (classes + 3) // 4 * 4, device=cuda)
    Z[:, :classes] = torch.from_numpy(z).to(cuda)
    Y, S = torch.from_numpy(y).to(cuda), torch.from_numpy(sc).to(cuda)
    gs = torch.zeros(n, ld, device=cuda)
    sp, sp24 = gdx.Split(n, ld, cuda), gdx.Split(n, ld, cuda)
    loss, loss24 = (torch.zeros(1, dtype=torch.float64, device=cuda) for _ in range(2))
    call("gdx_softmax_xent_fused", Z.data_ptr(), Z.shape[1], n, classes, Y.data_ptr(), 1.0 / n, None, 0,
         S.data_ptr(), gs.data_ptr(), ld, sp.hi.data_ptr(), sp.lo.data_ptr(), sp.ld, loss.data_ptr(),
         gdx.stream_handle())
    rows = torch.zeros(n, 3 * ld, dtype=torch.uint8, device=cuda)  # interleaved packed-24 rows
    base = rows.data_ptr()
    call("gdx_softmax_xent_fused_p24", Z.data_ptr(), Z.shape[1], n, classes, Y.data_ptr(), 1.0 / n, S.data_ptr(),
         base, 3 * ld // 2, base + 2 * ld, 3 * ld, sp24.hi.data_ptr(), sp24.lo.data_ptr(), sp24.ld,
         loss24.data_ptr(), gdx.stream_handle())
    hi = torch.empty(n, ld, dtype=torch.int16, device=cuda)
    lo = torch.empty(n, ld, dtype=torch.uint8, device=cuda)
    call("gdx_pack24", gs.data_ptr(), ld, n, ld, hi.data_ptr(), lo.data_ptr(), ld, gdx.stream_handle())
    torch.cuda.synchronize()
    got = rows.cpu().numpy()
    assert np.array_equal(got[:, :2 * ld].view(np.int16), hi.cpu().numpy())
    assert np.array_equal(got[:, 2 * ld:], lo.cpu().numpy())
    assert torch.equal(sp.hi, sp24.hi) and torch.equal(sp.lo, sp24.lo)
    assert float(loss.item()) == pytest.approx(float(loss24.item()), rel=1e-12)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_bandwidth_probe_modes(gdx, cuda, mode):
    """The roofline probes (stream, random 256-byte rows, random 192-byte packed-24 rows)
    run on an L2-resident buffer, reject non-4 KiB sizes, and report a plausible rate."""
    import torch
    from paper_2311_06837_b200._lib import call
    from paper_2311_06837_b200.errors import InputError
    nbytes = 8 << 20
    buf = torch.rand(nbytes // 4, device=cuda)
    sink = torch.zeros(4, device=cuda)
    with pytest.raises(InputError):
        call("gdx_probe_bandwidth", buf.data_ptr(), nbytes - 4, 1, mode, sink.data_ptr(), gdx.stream_handle())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call("gdx_probe_bandwidth", buf.data_ptr(), nbytes, 8, mode, sink.data_ptr(), gdx.stream_handle())
    e1.record()
    torch.cuda.synchronize()
    gbs = 8 * nbytes / e0.elapsed_time(e1) / 1e6
    assert 100.0 < gbs < 100000.0, gbs
