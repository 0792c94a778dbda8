"""The reference GNN layer API (reference_gnn.hpp) on the B200 engine.

Model (reference_gnn.cpp:64-89): h^l(v) = relu(W^l (h^{l-1}(v) + sum_{u in N(v)} h^{l-1}(u))).

Each layer is one tcgen05 GEMM (K2) and one fused gather-reduce (K1).  The
order is chosen by width: when the layer narrows (H <= F_in) the transform
runs first, Z = H^{l-1} W^T, and the aggregation gathers H-wide rows with the
self term, ReLU and the split-bf16 copy for the next GEMM fused in; when it
widens, the aggregation runs first and ReLU moves into the GEMM epilogue.
Both orders are the same linear map; results are fp32 within the scaled 1e-4
contract of an fp64 evaluation (tests/test_gpu_parity.py).

Matrices cross the API as numpy fp64 (the reference ``Matrix``), row-major.
"""
from __future__ import annotations

import numpy as np
import torch

from ._lib import call
from .device import DeviceCSR, Split, aggregate, dense, gemm_tn, pad4, require_cuda, stream_handle
from .errors import ContractError, InputError
from .extract import DependencySubgraph, extract_full, UNSEEN
from .graph import Graph, Partition

Matrix = np.ndarray
FEAT_TAG = 0x66656174   # "feat", reference_gnn.cpp:13
WEIG_TAG = 0x77656967   # "weig", reference_gnn.cpp:24


def _dev():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def make_features(n: int, dim: int, seed: int) -> Matrix:
    """reference_gnn.cpp:11-16, generated on device by SplitMix64 jump-ahead (K7)."""
    d = _dev()
    out = torch.empty(max(n * dim, 1), dtype=torch.float64, device=d)
    call("gdx_init_uniform_f64", seed, FEAT_TAG, 0, 0, n, dim, -0.5, 0.5, out.data_ptr(), dim,
         stream_handle())
    return out[:n * dim].cpu().numpy().reshape(n, dim)


def make_layer_weights(num_layers: int, feature_dim: int, hidden_dim: int, seed: int) -> list:
    """reference_gnn.cpp:18-32: layer 0 is hidden x feature_dim, later layers hidden x hidden,
    drawn consecutively from stream (seed, "weig")."""
    if feature_dim == 0 or hidden_dim == 0:
        raise InputError("make_layer_weights: dimensions must be >= 1")
    d = _dev()
    ws, first = [], 0
    for l in range(num_layers):
        i = feature_dim if l == 0 else hidden_dim
        out = torch.empty(hidden_dim * i, dtype=torch.float64, device=d)
        call("gdx_init_uniform_f64", seed, WEIG_TAG, 0, first, hidden_dim, i, -0.5, 0.5,
             out.data_ptr(), i, stream_handle())
        ws.append(out.cpu().numpy().reshape(hidden_dim, i))
        first += hidden_dim * i
    return ws


def _check_shapes(x: Matrix, w, layers: int):
    """reference_gnn.cpp:36-50."""
    if layers == 0:
        return
    if len(w) < layers:
        raise InputError(f"forward: {layers} layers requested, {len(w)} weight matrices given")
    width = x.shape[1]
    for l in range(layers):
        if w[l].shape[1] != width:
            raise InputError(f"forward: layer {l + 1} expects width {w[l].shape[1]}, got {width}")
        width = w[l].shape[0]


def _weights_split(W: np.ndarray, d) -> Split:
    Wt = torch.from_numpy(np.ascontiguousarray(W, np.float32)).to(d)
    s = Split(W.shape[0], W.shape[1], d)
    return s.fill_from(Wt, W.shape[1])


def _run_layers(csr_for_rows, n_local: int, h: torch.Tensor, width: int, w, layers: int,
                rows_in, rows_out, d) -> tuple[torch.Tensor, int]:
    """Shared layer loop.  rows_in[l]/rows_out[l]: prefix of rows read / computed at
    layer l (rows outside the computed prefix stay zero, which is how the
    hop mask of forward_server_local is honoured without per-edge checks)."""
    for l in range(layers):
        W = w[l]
        H = W.shape[0]
        B = _weights_split(W, d)
        r_in, r_out = rows_in[l], rows_out[l]
        g = csr_for_rows(r_out)
        out = dense(n_local, H, d)
        if H <= width:
            A = Split(n_local, width, d).fill_from(h, h.shape[1]) if r_in else Split(n_local, width, d)
            Z = dense(n_local, H, d)
            if r_in:
                gemm_tn(A, B, c0=Z, m=r_in)
            if r_out:
                aggregate(g, Z, H, out=out, self_coef=1.0, relu=True)
        else:
            A = Split(n_local, width, d)
            if r_out:
                aggregate(g, h, width, out_split=A, self_coef=1.0)
                gemm_tn(A, B, c0=out, relu=True, m=r_out)
        h, width = out, H
    return h, width


def forward_full(g: Graph, x: Matrix, w, layers: int) -> Matrix:
    """reference_gnn.cpp:64-89 on the GPU.  layers = 0 returns the input unchanged."""
    x = np.asarray(x, np.float64)
    if x.shape[0] != g.num_vertices():
        raise InputError("forward_full: feature rows do not match vertex count")
    _check_shapes(x, w, layers)
    if layers == 0:
        return x.copy()
    d = _dev()
    n = g.num_vertices()
    dg = g.device(d)
    h = dense(n, x.shape[1], d)
    h[:n, :x.shape[1]] = torch.from_numpy(x.astype(np.float32)).to(d)
    out, width = _run_layers(lambda r: dg.slice_rows(0, r), n, h, x.shape[1], w, layers,
                             [n] * layers, [n] * layers, d)
    return out[:n, :width].double().cpu().numpy()


class LocalSubgraph:
    """Device form of a DependencySubgraph: local ids ordered by (hop, id), the
    induced CSR in global neighbour order, and hop-class prefix sizes."""

    def __init__(self, sub: DependencySubgraph, g: Graph, d):
        n = g.num_vertices()
        hop_np = sub.hop_array(n)
        self.max_hop = int(sub.halo_hops.max()) if len(sub.halo_hops) else 0
        dg = g.device(d)
        hop = torch.from_numpy(hop_np.view(np.int32)).to(d)
        self.l2g = torch.empty(max(n, 1), dtype=torch.int32, device=d)
        self.local_of = torch.empty(max(n, 1), dtype=torch.int32, device=d)
        self.hop_start = np.zeros(self.max_hop + 2, np.uint64)
        from . import _lib
        ln = _lib.u32(0)
        call("gdx_order_by_hop", hop.data_ptr(), n, self.max_hop, self.l2g.data_ptr(),
             self.local_of.data_ptr(), self.hop_start.ctypes.data, _lib.C.byref(ln), stream_handle())
        self.n = int(ln.value)
        counts = torch.zeros(max(self.n, 1), dtype=torch.int64, device=d)
        call("gdx_local_csr", dg.row_ptr.data_ptr(), dg.col.data_ptr(), self.l2g.data_ptr(), self.n,
             self.local_of.data_ptr(), counts.data_ptr(), None, None, stream_handle())
        self.lptr = torch.zeros(self.n + 1, dtype=torch.int64, device=d)
        total = _lib.u64(0)
        call("gdx_exclusive_scan_u64", counts.data_ptr(), self.n, self.lptr.data_ptr(),
             _lib.C.byref(total), stream_handle())
        self.lcol = torch.empty(max(int(total.value), 1), dtype=torch.int32, device=d)
        call("gdx_local_csr", dg.row_ptr.data_ptr(), dg.col.data_ptr(), self.l2g.data_ptr(), self.n,
             self.local_of.data_ptr(), None, self.lptr.data_ptr(), self.lcol.data_ptr(),
             stream_handle())
        self.csr = DeviceCSR(self.lptr, self.lcol, self.n)

    def upto(self, h: int) -> int:
        """Number of local vertices with hop <= h."""
        if h < 0:
            return 0
        return int(self.hop_start[min(h, self.max_hop) + 1])


def forward_server_local(sub: DependencySubgraph, g: Graph, x: Matrix, w, layers: int,
                         require_exact: bool = False) -> Matrix:
    """reference_gnn.cpp:91-147: the same computation restricted to inner + halo;
    at layer l only rows with hop <= L-l are produced and neighbours with
    hop > L-l+1 are unavailable.  Rows are returned for inner vertices, ascending."""
    x = np.asarray(x, np.float64)
    if x.shape[0] != g.num_vertices():
        raise InputError("forward_server_local: feature rows do not match vertex count")
    _check_shapes(x, w, layers)
    if require_exact and (sub.sampled or sub.hop_limit < layers):
        raise ContractError(f"forward_server_local: subgraph too shallow or sampled for exact "
                            f"{layers}-layer computation")
    if layers == 0:  # no layer runs: the inner rows verbatim (reference_gnn.cpp:140-146)
        return x[np.asarray(sub.inner_vertices, np.int64)].copy()
    d = _dev()
    loc = LocalSubgraph(sub, g, d)
    F = x.shape[1]
    xg = torch.from_numpy(x.astype(np.float32)).to(d)
    h = dense(loc.n, F, d)
    first = loc.upto(layers)  # layer 1 reads hop <= L
    if first:
        call("gdx_gather_rows", xg.data_ptr(), F, loc.l2g.data_ptr(), first, F, h.data_ptr(),
             h.shape[1], stream_handle())
    rows_in = [loc.upto(layers - l) for l in range(layers)]        # hop <= L-l+1 (1-based l)
    rows_out = [loc.upto(layers - l - 1) for l in range(layers)]   # hop <= L-l
    out, width = _run_layers(lambda r: loc.csr.slice_rows(0, r), loc.n, h, F, w, layers,
                             rows_in, rows_out, d)
    n_inner = loc.upto(0)
    if layers == 0:
        return out[:n_inner, :F].double().cpu().numpy()
    return out[:n_inner, :width].double().cpu().numpy()


class EquivalenceReport:
    def __init__(self, per_server, max_dev):
        self.per_server_max_dev = per_server
        self.max_deviation = max_dev


def equivalence_check(g: Graph, server_partition: Partition, layers: int, seed: int,
                      feature_dim: int = 8, hidden_dim: int = 8) -> EquivalenceReport:
    """reference_gnn.cpp:149-172 on the engine: full closure per server must
    reproduce the whole-graph outputs on inner vertices (0 deviation expected)."""
    from .rng import mix64
    x = make_features(g.num_vertices(), feature_dim, seed)
    w = make_layer_weights(layers, feature_dim, hidden_dim, mix64(seed + 1))
    full = forward_full(g, x, w, layers)
    per = []
    for s in range(server_partition.num_parts):
        sub = extract_full(g, server_partition, s, layers)
        local = forward_server_local(sub, g, x, w, layers, require_exact=True)
        dev = float(np.max(np.abs(local - full[sub.inner_vertices]))) if local.size else 0.0
        per.append(dev)
    return EquivalenceReport(per, max(per) if per else 0.0)
