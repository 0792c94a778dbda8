"""CPU checkers for the GraNNDis hot path -- TEST INFRASTRUCTURE ONLY.

Two checkers, both built by ``oracle/Makefile``:

* ``port``  -- ``_build/liboracle.so``, the C restatement in ``granndis_oracle.c``
  (each function cites the reference file:line it follows);
* ``ref``   -- ``_ref/libgranndis_ref.so``, the UNMODIFIED reference sources
  (``/root/reference/proj/src``) compiled in place plus ``ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this package.  The product package
``paper_2311_06837_b200`` never does: it fails loudly without its CUDA library.

Parity status: RNG, generators, forward_full, forward_server_local, extraction,
batch closure / peel and split_batch are pinned to the reference (bit-exact);
the training extension (SAGE, normalised GCN, loss, backward, SGD) is
"parity unpinned" -- no reference implementation exists.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
UNSEEN = 0xFFFFFFFF
UNLIMITED = 0xFFFFFFFF
SUM, SAGE, GCN = 0, 1, 2

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


def build(quiet: bool = True) -> None:
    """Compile the checkers (the reference one only where /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-C", _HERE, "-s"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _load(rel: str) -> C.CDLL:
    path = os.path.join(_HERE, rel)
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


class _ModelC(C.Structure):
    _fields_ = [("kind", C.c_int), ("layers", C.c_uint32), ("dims", C.POINTER(C.c_uint32)),
                ("relu_last", C.c_int)]


_port = None
_ref = None


def port() -> C.CDLL:
    global _port
    if _port is None:
        L = _load("_build/liboracle.so")
        L.gro_mix64.restype = C.c_uint64
        L.gro_mix64.argtypes = [C.c_uint64]
        L.gro_gen_random_graph_count.restype = C.c_uint64
        L.gro_gen_random_graph_count.argtypes = [C.c_uint32, C.c_double, C.c_uint64, _u64p]
        L.gro_gen_random_graph_fill.argtypes = [C.c_uint32, C.c_double, C.c_uint64, _u64p, _u32p]
        L.gro_gen_planted_count.restype = C.c_uint64
        L.gro_gen_planted_count.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                            C.c_uint64, _u64p]
        L.gro_gen_planted_fill.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                           C.c_uint64, _u64p, _u32p]
        L.gro_from_edges.restype = C.c_uint64
        L.gro_from_edges.argtypes = [_u32p, C.c_uint64, C.c_uint32, _u64p, _u32p]
        L.gro_partition_random.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _u32p]
        L.gro_make_features.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _f64p]
        L.gro_feature_rows.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64, _f64p, C.c_int]
        L.gro_make_layer_weights.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, _f64p]
        L.gro_forward_full.argtypes = [C.c_uint32, _u64p, _u32p, _f64p, C.c_uint32, _f64p,
                                       C.c_uint32, C.c_uint32, _f64p, C.c_int]
        L.gro_forward_server_local.argtypes = [C.c_uint32, _u64p, _u32p, _f64p, C.c_uint32, _f64p,
                                               C.c_uint32, C.c_uint32, _u32p, _f64p]
        L.gro_extract_full.restype = C.c_uint64
        L.gro_extract_full.argtypes = [C.c_uint32, _u64p, _u32p, _u32p, C.c_uint32, C.c_uint32,
                                       _u32p]
        L.gro_extract_sampled.restype = C.c_uint64
        L.gro_extract_sampled.argtypes = [C.c_uint32, _u64p, _u32p, _u32p, C.c_uint32,
                                          C.c_uint32, C.c_uint32, C.c_uint64, _u32p]
        L.gro_batch_closure.restype = C.c_uint64
        L.gro_batch_closure.argtypes = [C.c_uint32, _u64p, _u32p, _u8p, _u32p, C.c_uint64,
                                        C.c_uint32, C.c_uint32, C.c_uint64, _u8p]
        L.gro_peel_mfg.argtypes = [C.c_uint32, _u64p, _u32p, _u8p, _u32p, C.c_uint64,
                                   C.c_uint32, _u64p]
        L.gro_split_batch.argtypes = [_u32p, C.c_uint64, _u32p, _u32p, C.c_uint32, C.c_uint32,
                                      _u32p]
        L.gro_weight_count.restype = C.c_uint64
        L.gro_weight_count.argtypes = [C.POINTER(_ModelC)]
        L.gro_model_forward.argtypes = [C.c_uint32, _u64p, _u32p, _f64p, C.POINTER(_ModelC),
                                        _f64p, C.c_void_p, C.c_int]
        L.gro_train_epoch.restype = C.c_double
        L.gro_train_epoch.argtypes = [C.c_uint32, _u64p, _u32p, _f64p, _i32p, C.c_uint32,
                                      C.POINTER(_ModelC), _f64p, C.c_double, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_uint32, C.c_int]
        L.gro_train_epoch_masked.restype = C.c_double
        L.gro_train_epoch_masked.argtypes = [C.c_uint32, _u64p, _u32p, _f64p, _i32p, C.c_uint32,
                                             C.POINTER(_ModelC), _f64p, C.c_double, C.c_void_p,
                                             C.c_uint32, C.c_double, C.c_void_p, C.c_int]
        _port = L
    return _port


def ref_available() -> bool:
    return os.path.exists(os.path.join(_HERE, "_ref/libgranndis_ref.so"))


def ref() -> C.CDLL:
    """The compiled reference (oracle/_ref).  Raises if it was never built."""
    global _ref
    if _ref is None:
        path = os.path.join(_HERE, "_ref/libgranndis_ref.so")
        if not os.path.exists(path):
            raise RuntimeError("oracle/_ref/libgranndis_ref.so missing: run make -C oracle "
                               "where /root/reference is mounted")
        L = C.CDLL(path)
        vp = C.c_void_p
        L.grr_last_error.restype = C.c_char_p
        L.grr_gen_random_graph.restype = vp
        L.grr_gen_random_graph.argtypes = [C.c_uint32, C.c_double, C.c_uint64]
        L.grr_gen_planted.restype = vp
        L.grr_gen_planted.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_uint64]
        L.grr_graph_from_edges.restype = vp
        L.grr_graph_from_edges.argtypes = [_u32p, C.c_uint64, C.c_uint32]
        L.grr_graph_from_csr.restype = vp
        L.grr_graph_from_csr.argtypes = [C.c_uint32, _u64p, _u32p]
        L.grr_graph_n.restype = C.c_uint32
        L.grr_graph_n.argtypes = [vp]
        L.grr_graph_nnz.restype = C.c_uint64
        L.grr_graph_nnz.argtypes = [vp]
        L.grr_graph_copy.argtypes = [vp, _u64p, _u32p]
        L.grr_graph_free.argtypes = [vp]
        L.grr_partition_random.argtypes = [vp, C.c_uint32, C.c_uint64, _u32p]
        L.grr_partition_mincut.argtypes = [vp, C.c_uint32, C.c_uint64, C.c_double, _u32p]
        L.grr_hierarchical_partition.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_int, C.c_uint64,
                                                 _u32p, _u32p]
        L.grr_mix64.restype = C.c_uint64
        L.grr_mix64.argtypes = [C.c_uint64]
        L.grr_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.grr_shuffle.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u32p, C.c_uint64]
        L.grr_make_features.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _f64p]
        L.grr_make_layer_weights.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, _f64p]
        L.grr_forward_full.argtypes = [vp, _f64p, C.c_uint32, C.c_uint32, _f64p, C.c_uint32,
                                       C.c_uint32, C.c_uint32, _f64p]
        L.grr_forward_server_local.argtypes = [vp, _u32p, C.c_uint32, C.c_uint32, C.c_int, _f64p,
                                               C.c_uint32, _f64p, C.c_uint32, C.c_uint32, C.c_int,
                                               _f64p]
        L.grr_equivalence_check.restype = C.c_double
        L.grr_equivalence_check.argtypes = [vp, _u32p, C.c_uint32, C.c_uint32, C.c_uint64,
                                            C.c_uint32, C.c_uint32]
        L.grr_extract_full.argtypes = [vp, _u32p, C.c_uint32, C.c_uint32, C.c_uint32, _u32p,
                                       C.POINTER(C.c_uint64)]
        L.grr_extract_sampled.argtypes = [vp, _u32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_uint64, _u32p, C.POINTER(C.c_uint64)]
        L.grr_neighbor_explosion_profile.argtypes = [vp, _u32p, C.c_uint32, C.c_uint32,
                                                     C.c_uint32, _u64p]
        L.grr_plan_cobatch_fixed_r.restype = vp
        L.grr_plan_cobatch_fixed_r.argtypes = [vp, _u32p, C.c_uint32, C.c_uint32, C.c_int,
                                               C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                               C.c_uint32, C.c_uint32, C.c_uint32]
        L.grr_plan_cobatch.restype = vp
        L.grr_plan_cobatch.argtypes = [vp, _u32p, C.c_uint32, C.c_uint32, C.c_int,
                                       C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                       C.c_uint64, C.c_uint32, C.c_uint32]
        L.grr_plan_batches.restype = C.c_uint32
        L.grr_plan_batches.argtypes = [vp]
        L.grr_plan_batch_sizes.argtypes = [vp, C.c_uint32, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.grr_plan_batch_copy.argtypes = [vp, C.c_uint32, _u32p, _u32p, _u64p]
        L.grr_plan_free.argtypes = [vp]
        L.grr_simulate_cobatch_moved.argtypes = [vp, _u32p, _u32p, C.c_uint32, C.c_uint32,
                                                 C.c_uint32, C.POINTER(vp), _u64p, _u64p]
        L.grr_simulate_epoch.argtypes = [vp, _u32p, _u32p, C.c_uint32, C.c_uint32, C.c_double,
                                         C.c_double, C.c_double, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_int, C.c_uint32, C.c_uint32, C.c_uint64,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _ref = L
    return _ref


# ---------------------------------------------------------------------------
@dataclass
class CSR:
    """Host CSR in the reference layout (graph.hpp:21-60)."""
    n: int
    row_offsets: np.ndarray  # u64[n+1]
    cols: np.ndarray         # u32[nnz]

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets).astype(np.int64)


def gen_random_graph(n: int, avg_degree: float, seed: int) -> CSR:
    L = port()
    ro = np.zeros(n + 1, np.uint64)
    nnz = L.gro_gen_random_graph_count(n, avg_degree, seed, ro)
    cols = np.zeros(max(nnz, 1), np.uint32)
    L.gro_gen_random_graph_fill(n, avg_degree, seed, ro, cols)
    return CSR(n, ro, cols[:nnz])


def gen_planted(n: int, parts: int, p_in: float, p_out: float, seed: int) -> CSR:
    L = port()
    ro = np.zeros(n + 1, np.uint64)
    nnz = L.gro_gen_planted_count(n, parts, p_in, p_out, seed, ro)
    cols = np.zeros(max(nnz, 1), np.uint32)
    L.gro_gen_planted_fill(n, parts, p_in, p_out, seed, ro, cols)
    return CSR(n, ro, cols[:nnz])


def from_edges(edges, n: int) -> CSR:
    e = np.ascontiguousarray(np.asarray(edges, np.uint32).reshape(-1, 2))
    ro = np.zeros(n + 1, np.uint64)
    cols = np.zeros(max(2 * len(e), 1), np.uint32)
    nnz = port().gro_from_edges(e.reshape(-1), len(e), n, ro, cols)
    return CSR(n, ro, cols[:nnz].copy())


def partition_random(n: int, parts: int, seed: int) -> np.ndarray:
    out = np.zeros(n, np.uint32)
    port().gro_partition_random(n, parts, seed, out)
    return out


def mix64(x: int) -> int:
    return int(port().gro_mix64(x))


def make_features(n: int, dim: int, seed: int) -> np.ndarray:
    out = np.zeros(n * dim, np.float64)
    port().gro_make_features(n, dim, seed, out)
    return out.reshape(n, dim)


def feature_rows(ids, dim: int, seed: int, nthreads: int = 0) -> np.ndarray:
    """Rows `ids` of make_features(n, dim, seed) without generating the rest."""
    ids = np.ascontiguousarray(ids, np.uint32)
    out = np.zeros(max(len(ids), 1) * dim, np.float64)
    port().gro_feature_rows(ids.ctypes.data, len(ids), dim, seed, out, nthreads or (os.cpu_count() or 1))
    return out[:len(ids) * dim].reshape(len(ids), dim)


def make_layer_weights(layers: int, F: int, H: int, seed: int) -> list[np.ndarray]:
    total = sum(H * (F if l == 0 else H) for l in range(layers))
    out = np.zeros(max(total, 1), np.float64)
    port().gro_make_layer_weights(layers, F, H, seed, out)
    ws, off = [], 0
    for l in range(layers):
        i = F if l == 0 else H
        ws.append(out[off:off + H * i].reshape(H, i).copy())
        off += H * i
    return ws


def stream_weights(shapes, seed: int, fp32: bool = True, init: str = "uniform") -> list[np.ndarray]:
    """Matrices of the given (rows, cols) shapes filled by consecutive U(-.5,.5) draws
    of the weight stream (seed, "weig") -- make_layer_weights' stream
    (reference_gnn.cpp:18-32) continued across matrices, which is how the engine's
    init_weights lays out SAGE's W_self / W_neigh pairs.  fp32: round to the fp32
    values the engine trains from."""
    total = sum(int(r) * int(c) for r, c in shapes)
    flat = make_layer_weights(1, max(total, 1), 1, seed)[0].reshape(-1)
    out, off = [], 0
    for r, c in shapes:
        w = flat[off:off + r * c].reshape(r, c)
        if init == "he":      # the engine's ModelConfig.init == 'he' (train.init_scale)
            w = w * (2.0 * np.sqrt(6.0 / c))
        out.append(w.astype(np.float32).astype(np.float64) if fp32 else w.copy())
        off += r * c
    return out


def _flat(ws) -> np.ndarray:
    if not ws:
        return np.zeros(1, np.float64)
    return np.ascontiguousarray(np.concatenate([np.asarray(w, np.float64).reshape(-1) for w in ws]))


def forward_full(g: CSR, x: np.ndarray, ws, layers: int, nthreads: int = 1) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    F = x.shape[1]
    H = ws[0].shape[0] if layers else F
    out = np.zeros(g.n * (H if layers else F), np.float64)
    port().gro_forward_full(g.n, g.row_offsets, g.cols, x, F, _flat(ws), H, layers, out, nthreads)
    return out.reshape(g.n, -1)


def forward_server_local(g: CSR, x: np.ndarray, ws, layers: int, hop: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    F = x.shape[1]
    H = ws[0].shape[0] if layers else F
    n_inner = int((hop == 0).sum())
    out = np.zeros(max(n_inner * (H if layers else F), 1), np.float64)
    port().gro_forward_server_local(g.n, g.row_offsets, g.cols, x, F, _flat(ws), H, layers,
                                    np.ascontiguousarray(hop, np.uint32), out)
    return out[:n_inner * (H if layers else F)].reshape(n_inner, -1)


def extract_full(g: CSR, assignment: np.ndarray, server: int, layers: int):
    hop = np.zeros(g.n, np.uint32)
    ind = port().gro_extract_full(g.n, g.row_offsets, g.cols,
                                  np.ascontiguousarray(assignment, np.uint32), server, layers, hop)
    return hop, int(ind)


def extract_sampled(g: CSR, assignment: np.ndarray, server: int, max_hop: int, fanout: int,
                    seed: int):
    hop = np.zeros(g.n, np.uint32)
    ind = port().gro_extract_sampled(g.n, g.row_offsets, g.cols,
                                     np.ascontiguousarray(assignment, np.uint32), server, max_hop,
                                     fanout, seed, hop)
    return hop, int(ind)


def batch_closure(g: CSR, universe: np.ndarray, targets: np.ndarray, max_hop: int, fanout: int,
                  seed: int) -> np.ndarray:
    out = np.zeros(g.n, np.uint8)
    t = np.ascontiguousarray(targets, np.uint32)
    port().gro_batch_closure(g.n, g.row_offsets, g.cols, np.ascontiguousarray(universe, np.uint8),
                             t, len(t), max_hop, fanout, seed, out)
    return np.nonzero(out)[0].astype(np.uint32)


def peel_mfg(g: CSR, batch_vertices: np.ndarray, targets: np.ndarray, layers: int) -> np.ndarray:
    in_batch = np.zeros(g.n, np.uint8)
    in_batch[batch_vertices] = 1
    t = np.ascontiguousarray(targets, np.uint32)
    counts = np.zeros(layers + 1, np.uint64)
    port().gro_peel_mfg(g.n, g.row_offsets, g.cols, in_batch, t, len(t), layers, counts)
    return counts


def split_batch(batch_vertices, server_assign, gpu_assign, server: int, gpus: int) -> np.ndarray:
    bv = np.ascontiguousarray(batch_vertices, np.uint32)
    out = np.zeros(max(len(bv), 1), np.uint32)
    port().gro_split_batch(bv, len(bv), np.ascontiguousarray(server_assign, np.uint32),
                           np.ascontiguousarray(gpu_assign, np.uint32), server, gpus, out)
    return out[:len(bv)]


# ---- training extension (parity unpinned) ------------------------------------
class Model:
    def __init__(self, kind: int, dims, relu_last: bool = False):
        self.kind = kind
        self.dims = np.ascontiguousarray(dims, np.uint32)
        self.layers = len(dims) - 1
        self.relu_last = int(relu_last)
        self._c = _ModelC(kind, self.layers, self.dims.ctypes.data_as(C.POINTER(C.c_uint32)),
                          self.relu_last)

    def weight_shapes(self):
        shapes = []
        for l in range(self.layers):
            shapes.append((int(self.dims[l + 1]), int(self.dims[l])))
            if self.kind == SAGE:
                shapes.append((int(self.dims[l + 1]), int(self.dims[l])))
        return shapes

    def weight_count(self) -> int:
        return int(port().gro_weight_count(C.byref(self._c)))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def model_forward(g: CSR, x: np.ndarray, model: Model, w: np.ndarray, nthreads: int = 1):
    total = sum(g.n * int(d) for d in model.dims[1:])
    acts = np.zeros(total, np.float64)
    port().gro_model_forward(g.n, g.row_offsets, g.cols, np.ascontiguousarray(x, np.float64),
                             C.byref(model._c), np.ascontiguousarray(w, np.float64), _ptr(acts),
                             nthreads)
    return _split_acts(acts, g.n, model.dims[1:])


def _split_acts(flat, n, dims):
    out, off = [], 0
    for d in dims:
        out.append(flat[off:off + n * int(d)].reshape(n, int(d)))
        off += n * int(d)
    return out


def train_epoch(g: CSR, x: np.ndarray, labels: np.ndarray, model: Model, w: np.ndarray, lr: float,
                want_state: bool = False, row_limit: int | None = None, nthreads: int = 1):
    """One epoch in fp64; updates ``w`` in place.  Returns loss (and state)."""
    C_ = int(model.dims[-1])
    total = sum(g.n * int(d) for d in model.dims[1:])
    grads = np.zeros(model.weight_count(), np.float64) if want_state else None
    acts = np.zeros(total, np.float64) if want_state else None
    dacts = np.zeros(total, np.float64) if want_state else None
    loss = port().gro_train_epoch(g.n, g.row_offsets, g.cols, np.ascontiguousarray(x, np.float64),
                                  np.ascontiguousarray(labels, np.int32), C_, C.byref(model._c), w,
                                  lr, _ptr(grads), _ptr(acts), _ptr(dacts),
                                  g.n if row_limit is None else row_limit, nthreads)
    if not want_state:
        return loss
    return loss, grads, _split_acts(acts, g.n, model.dims[1:]), _split_acts(dacts, g.n, model.dims[1:])


def train_epoch_masked(g: CSR, x: np.ndarray, labels: np.ndarray, model: Model, w: np.ndarray,
                       lr: float, loss_rows: int, loss_count: float, nthreads: int = 1,
                       layer_rows=None):
    """Epoch with the loss over rows < loss_rows / loss_count.  lr == 0 returns the
    gradients without updating (for summing several subgraphs).  Returns (loss, grads)."""
    grads = np.zeros(model.weight_count(), np.float64)
    lr_arr = None if layer_rows is None else np.ascontiguousarray(layer_rows, np.uint32)
    loss = port().gro_train_epoch_masked(g.n, g.row_offsets, g.cols, np.ascontiguousarray(x, np.float64),
                                         np.ascontiguousarray(labels, np.int32), int(model.dims[-1]),
                                         C.byref(model._c), w, lr, _ptr(grads), loss_rows, loss_count,
                                         _ptr(lr_arr), nthreads)
    return loss, grads


def make_labels(n: int, classes: int, seed: int) -> np.ndarray:
    """Builder-defined labels: KeyedRng(seed, v, "labl").next_below(classes)."""
    # vectorised SplitMix64: first draw of stream (seed, v, 0x6c61626c)
    M = (1 << 64) - 1
    g = 0x9e3779b97f4a7c15

    def fin(z):
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)) & np.uint64(M)
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)) & np.uint64(M)
        return z ^ (z >> np.uint64(31))

    with np.errstate(over="ignore"):
        v = np.arange(n, dtype=np.uint64)
        s = np.full(n, mix64(seed), np.uint64)
        s = fin((s ^ (v + np.uint64(g))) + np.uint64(g))
        s = fin((s ^ np.uint64((0x6c61626c + 0xc2b2ae3d27d4eb4f) & M)) + np.uint64(g))
        x = fin(s + np.uint64(g))
    hi = (x >> np.uint64(32)).astype(np.uint64)
    lo = (x & np.uint64(0xFFFFFFFF)).astype(np.uint64)
    c = np.uint64(classes)
    # (x * c) >> 64 computed exactly with 32-bit halves
    return ((hi * c + ((lo * c) >> np.uint64(32))) >> np.uint64(32)).astype(np.int32)


def ref_plan(g_handle, hop: np.ndarray, server: int, hop_limit: int, sampled: bool, layers: int,
             max_hop: int, fanout: int, seed: int, hidden: int, feat: int, r: int = 0,
             budget: int = 0):
    """The compiled reference's plan_cobatch_fixed_r (r > 0) or plan_cobatch (budget):
    a list of (targets, vertices, mfg, bytes) per batch, or the error string."""
    R = ref()
    hop = np.ascontiguousarray(hop, np.uint32)
    if r:
        p = R.grr_plan_cobatch_fixed_r(g_handle, hop, server, hop_limit, int(sampled), layers, max_hop,
                                       fanout, seed, r, hidden, feat)
    else:
        p = R.grr_plan_cobatch(g_handle, hop, server, hop_limit, int(sampled), layers, max_hop,
                               fanout, seed, budget, hidden, feat)
    if not p:
        return R.grr_last_error().decode()
    out = []
    for b in range(R.grr_plan_batches(p)):
        nt, nv, by = C.c_uint64(), C.c_uint64(), C.c_uint64()
        R.grr_plan_batch_sizes(p, b, C.byref(nt), C.byref(nv), C.byref(by))
        t = np.zeros(max(nt.value, 1), np.uint32)
        v = np.zeros(max(nv.value, 1), np.uint32)
        m = np.zeros(layers + 1, np.uint64)
        R.grr_plan_batch_copy(p, b, t, v, m)
        out.append((t[:nt.value], v[:nv.value], [int(x) for x in m], int(by.value)))
    R.grr_plan_free(p)
    return out


def rng_draws(seed: int, k1: int, k2: int, count: int) -> np.ndarray:
    out = np.zeros(count, np.uint64)
    ref().grr_rng_draws(seed, k1, k2, count, out)
    return out
