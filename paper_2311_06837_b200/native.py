"""The C-ABI trainer (gdx_trainer_*, include/gdx.h; csrc/trainer.cu) from Python.

The epoch runs entirely in libgdx's C++: the layer loop, the NVLink row exchange
and the weight-gradient all-reduce over CUDA IPC, the CUDA graph of the epoch.
Python only builds the inputs (host CSR, or a local subgraph's CSR and prefixes)
and, for world > 1, gathers the 64-byte IPC blobs with torch.distributed (any
backend) -- the same handshake a C++ host does with MPI or sockets.  This is the
path bench.py measures; train.FullGraphTrainer is the torch-orchestrated twin
with the experimental exchange knobs.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import call
from .errors import InputError
from .graph import Graph

KIND = {"sum": 0, "gcn": 1, "sage": 2}
LABEL_SEED, FEATURE_SEED = 2, 1


class TrainerConfig(C.Structure):
    _fields_ = [("kind", C.c_int), ("layers", C.c_uint32), ("dims", C.POINTER(C.c_uint32)),
                ("lr", C.c_float), ("rank", C.c_uint32), ("world", C.c_uint32), ("device", C.c_int),
                ("feature_seed", C.c_uint64), ("label_seed", C.c_uint64), ("use_graph", C.c_int),
                ("no_agg_first", C.c_int), ("push_ctas", C.c_uint32), ("peer_timeout_s", C.c_double),
                ("heavy_degree", C.c_uint32), ("fused_exchange", C.c_int), ("packed24", C.c_int)]


class TrainerGraph(C.Structure):
    _fields_ = [("num_vertices", C.c_uint32), ("nnz", C.c_uint64), ("row_offsets", C.c_void_p),
                ("cols", C.c_void_p), ("local_rows", C.c_uint64), ("rows_in", C.c_void_p),
                ("rows_out", C.c_void_p), ("loss_rows", C.c_uint32), ("loss_count", C.c_double),
                ("global_ids", C.c_void_p)]


_SIGS = {
    "gdx_trainer_create": (C.c_int, [C.POINTER(TrainerConfig), C.POINTER(TrainerGraph), C.POINTER(C.c_void_p)]),
    "gdx_trainer_destroy": (C.c_int, [C.c_void_p]),
    "gdx_trainer_weight_count": (C.c_uint64, [C.c_void_p]),
    "gdx_trainer_init_weights": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int]),
    "gdx_trainer_set_weights": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "gdx_trainer_get_weights": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "gdx_trainer_get_grads": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "gdx_trainer_ipc_blob_bytes": (C.c_uint64, [C.c_void_p]),
    "gdx_trainer_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdx_trainer_connect": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdx_trainer_epoch": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "gdx_trainer_stage_inputs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "gdx_trainer_step_staged": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double)]),
    "gdx_trainer_stream": (C.c_void_p, [C.c_void_p]),
    "gdx_trainer_info": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32]),
    "gdx_trainer_profile": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_double)]),
    "gdx_trainer_profile_gemm": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_double)]),
}
_bound = False


def _bind():
    global _bound
    if not _bound:
        L = _lib.lib()
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _bound = True
    return _lib.lib()


def _fused_default() -> bool:
    """GDX_FUSED_EXCHANGE=1|0 selects the one-kernel exchange + aggregation for N > 1."""
    import os
    return os.environ.get("GDX_FUSED_EXCHANGE", "0") != "0"


def weight_shapes(kind: str, dims) -> list:
    out = []
    for l in range(len(dims) - 1):
        out.append((dims[l + 1], dims[l]))
        if kind == "sage":
            out.append((dims[l + 1], dims[l]))
    return out


class NativeTrainer:
    """One gdx_trainer per rank/GPU.  Full graph (row blocks of the whole CSR, per-layer
    NVLink exchange) or, with subgraph=, this rank's preloaded EAS subgraph."""

    def __init__(self, g: Graph, cfg, *, rank: int = 0, world: int = 1, device: int | None = None,
                 weights=None, weight_seed: int = 3, subgraph=None, pg=None, use_graph: bool = True,
                 feature_seed: int = FEATURE_SEED, label_seed: int = LABEL_SEED, push_ctas: int = 0,
                 no_agg_first: bool = False, heavy_degree: int = 0, fused_exchange: bool | None = None,
                 packed24: bool = False):
        import torch
        L = _bind()
        if cfg.kind not in KIND:
            raise InputError(f"unknown model kind {cfg.kind!r}")
        self.cfg, self.rank, self.world, self.pg = cfg, rank, world, pg
        self.device = torch.cuda.current_device() if device is None else device
        self.dims = list(cfg.dims)
        self._dims_c = (C.c_uint32 * len(self.dims))(*self.dims)
        c = TrainerConfig(KIND[cfg.kind], len(self.dims) - 1, self._dims_c, cfg.lr, rank, world, self.device,
                          feature_seed, label_seed, int(use_graph), int(no_agg_first), push_ctas, 0.0,
                          heavy_degree, int(_fused_default() if fused_exchange is None else fused_exchange),
                          int(packed24))
        gr = TrainerGraph()
        gr.num_vertices = g.num_vertices()
        self.subgraph_mode = subgraph is not None
        keep = []
        if subgraph is None:
            ro, ci = g.row_offsets(), g.col_indices()
            gr.nnz = g.num_edges()
            gr.row_offsets, gr.cols = ro.ctypes.data, ci.ctypes.data
            keep += [ro, ci]
        else:
            from .gnn import LocalSubgraph
            loc = LocalSubgraph(subgraph, g, torch.device("cuda", self.device))
            Lc = len(self.dims) - 1
            lptr = loc.lptr.cpu().numpy().astype(np.uint64)
            lcol = loc.lcol.cpu().numpy().view(np.uint32)[:int(lptr[-1])].copy()
            l2g = loc.l2g[:max(loc.n, 1)].cpu().numpy().view(np.uint32)[:loc.n].copy()
            rows_in = np.array([loc.upto(Lc - l) for l in range(Lc)], np.uint32)
            rows_out = np.array([loc.upto(Lc - l - 1) for l in range(Lc)], np.uint32)
            loss_rows = loc.upto(0)
            cnt = float(loss_rows)
            if world > 1:
                import torch.distributed as dist
                t = torch.tensor([cnt], dtype=torch.float64,
                                 device="cpu" if dist.get_backend(pg) == "gloo" else f"cuda:{self.device}")
                dist.all_reduce(t, group=pg)
                cnt = float(t.item())
            gr.nnz = int(lptr[-1])
            gr.row_offsets, gr.cols = lptr.ctypes.data, (lcol if len(lcol) else np.zeros(1, np.uint32)).ctypes.data
            gr.local_rows = loc.n
            gr.rows_in, gr.rows_out = rows_in.ctypes.data, rows_out.ctypes.data
            gr.loss_rows, gr.loss_count = loss_rows, cnt
            gr.global_ids = l2g.ctypes.data
            keep += [lptr, lcol, l2g, rows_in, rows_out]
            self.local_rows = loc.n
            self.l2g, self.rows_in = l2g, rows_in
            del loc
        h = C.c_void_p()
        call("gdx_trainer_create", C.byref(c), C.byref(gr), C.byref(h))
        self._h = h.value
        self.nloc, self.nnz_local, self.lo = self.info()[:3]
        self.F = self.dims[0]
        if weights is not None:
            self.set_weights(weights)
        else:
            call("gdx_trainer_init_weights", self._h, weight_seed, int(getattr(cfg, "init", "uniform") == "he"))
        if world > 1:
            self._connect()

    # ---- plumbing ----
    def _connect(self):
        import torch.distributed as dist
        nb = int(_lib.lib().gdx_trainer_ipc_blob_bytes(self._h))
        blob = C.create_string_buffer(nb)
        call("gdx_trainer_ipc_export", self._h, blob)
        out = [None] * self.world
        dist.all_gather_object(out, blob.raw, group=self.pg)
        allb = C.create_string_buffer(b"".join(out), nb * self.world)
        call("gdx_trainer_connect", self._h, allb)
        dist.barrier(group=self.pg)

    def info(self) -> list:
        out = np.zeros(10, np.uint64)
        call("gdx_trainer_info", self._h, out.ctypes.data, 10)
        return [int(x) for x in out]

    @property
    def graph_captured(self) -> bool:
        return bool(self.info()[6])

    def stream(self):
        """The trainer's stream as a torch ExternalStream (for event timing)."""
        import torch
        return torch.cuda.ExternalStream(_lib.lib().gdx_trainer_stream(self._h), device=self.device)

    # ---- weights ----
    def _count(self) -> int:
        return int(_lib.lib().gdx_trainer_weight_count(self._h))

    def set_weights(self, weights):
        flat = np.ascontiguousarray(np.concatenate([np.asarray(w, np.float64).ravel() for w in weights]))
        call("gdx_trainer_set_weights", self._h, flat.ctypes.data, len(flat))

    def _split(self, flat):
        out, off = [], 0
        for (o, i) in weight_shapes(self.cfg.kind, self.dims):
            out.append(flat[off:off + o * i].reshape(o, i).copy())
            off += o * i
        return out

    def get_weights(self) -> list:
        flat = np.zeros(self._count(), np.float64)
        call("gdx_trainer_get_weights", self._h, flat.ctypes.data, len(flat))
        return self._split(flat)

    def get_grads(self) -> list:
        flat = np.zeros(self._count(), np.float64)
        call("gdx_trainer_get_grads", self._h, flat.ctypes.data, len(flat))
        return self._split(flat)

    # ---- epochs ----
    def train_epoch(self, sync_loss: bool = True):
        if sync_loss:
            loss = C.c_double()
            call("gdx_trainer_epoch", self._h, C.byref(loss))
            return loss.value
        call("gdx_trainer_epoch", self._h, None)
        return None

    def stage_inputs(self, x_host: np.ndarray | None, labels_host=None, x_ptr: int = 0, labels_ptr: int = 0):
        """Enqueue the H2D of the next step's feature block (host fp32 [nloc, F],
        C-contiguous; pinned memory for overlap) and labels."""
        if x_host is not None:
            if x_host.dtype != np.float32 or x_host.shape != (self.nloc, self.F) or not x_host.flags.c_contiguous:
                raise InputError(f"stage_inputs: features must be float32 [{self.nloc}, {self.F}], contiguous")
            x_ptr = x_host.ctypes.data
            if labels_host is not None:
                labels_ptr = np.ascontiguousarray(labels_host, np.int32).ctypes.data
        call("gdx_trainer_stage_inputs", self._h, x_ptr, labels_ptr or None)

    def step_staged(self, with_labels: bool = True, sync_loss: bool = True):
        loss = C.c_double()
        call("gdx_trainer_step_staged", self._h, int(with_labels), C.byref(loss) if sync_loss else None)
        return loss.value if sync_loss else None

    def profile(self, on: bool):
        call("gdx_trainer_profile", self._h, int(on), None, None, None)

    def profile_read_gemm(self):
        """(ms, launches, useful flops) of the profiled epochs' GEMMs (call before profile_read)."""
        ms, n, fl = C.c_double(), C.c_uint64(), C.c_double()
        call("gdx_trainer_profile_gemm", self._h, C.byref(ms), C.byref(n), C.byref(fl))
        return ms.value, int(n.value), fl.value

    def profile_read(self):
        ms, n, by = C.c_double(), C.c_uint64(), C.c_double()
        call("gdx_trainer_profile", self._h, 0, C.byref(ms), C.byref(n), C.byref(by))
        return ms.value, int(n.value), by.value

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().gdx_trainer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
