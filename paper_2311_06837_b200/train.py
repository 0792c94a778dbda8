"""Full-graph GNN training on the B200 engine (the training extension of the
reference's layer model).

One process per GPU.  Rank r owns the contiguous row block [lo, hi) of the
vertex set (the graph's rows, its labels and its input features); every
layer is

  forward   Z_loc = H_loc W^T            (K2 tcgen05 GEMM; GCN row scale fused)
            all-gather Z -> Z_full        (NCCL over NVLink; the a13 exchange)
            H'_loc = act(agg(Z_full))     (K1; self term, degree scale, SAGE self
                                           path, ReLU and the split-bf16 copy fused)
  backward  g = dH * relu'(H') -> split G, gs = scaled g   (elementwise)
            all-gather gs -> gs_full
            dZ_loc = agg^T(gs_full)       (K3 = K1 on the symmetric CSR)
            dH_loc = G W                  (K2)
            dW = G^T H (split-K over rows) (K2) -> all-reduce -> SGD (fused reduce)

Models (no bias; dims[0] = features, dims[-1] = classes, ReLU between layers):
  'sum'  : P = W (H_v + sum_u H_u)                  (reference_gnn.cpp:64-89)
  'gcn'  : P = W s_v (s_v H_v + sum_u s_u H_u), s = (deg+1)^-1/2
  'sage' : P = W_s H_v + W_n mean_u H_u             (GraphSAGE-mean)
Loss: mean softmax cross-entropy over all vertices; SGD.  Parity is against the
fp64 oracle restatement (parity unpinned: no reference implementation exists).
"""
from __future__ import annotations

import math
import os
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call
from .device import DeviceCSR, Split, aggregate, dense, gemm_tn, pad4, pad8, require_cuda, stream_handle
from .errors import InputError, InternalError
from .gnn import FEAT_TAG, WEIG_TAG
from .graph import Graph, partition_contiguous

LABEL_SEED_DEFAULT = 0x6c61626c


@dataclass
class ModelConfig:
    kind: str = "sage"              # 'sage' | 'gcn' | 'sum'
    dims: list = field(default_factory=lambda: [602, 64, 64, 41])
    lr: float = 0.1
    # 'uniform': U(-.5,.5), the reference's make_layer_weights values; 'he': the same
    # draws times 2 sqrt(6 / fan_in) (He-uniform), which keeps a 56-layer stack finite
    # (U(-.5,.5) grows activations ~1.6x per layer and overflows by layer ~40)
    init: str = "uniform"

    @property
    def layers(self) -> int:
        return len(self.dims) - 1

    @property
    def classes(self) -> int:
        return self.dims[-1]

    def weight_shapes(self):
        """Reference-order weight list: per layer W (sum/gcn) or W_self, W_neigh (sage)."""
        out = []
        for l in range(self.layers):
            out.append((self.dims[l + 1], self.dims[l]))
            if self.kind == "sage":
                out.append((self.dims[l + 1], self.dims[l]))
        return out


def init_weights(cfg: ModelConfig, seed: int) -> list:
    """Consecutive U(-.5,.5) draws of stream (seed, "weig") in weight_shapes order
    (the make_layer_weights stream, reference_gnn.cpp:18-32, extended to SAGE)."""
    require_cuda()
    d = torch.device("cuda", torch.cuda.current_device())
    ws, first = [], 0
    for (o, i) in cfg.weight_shapes():
        t = torch.empty(o * i, dtype=torch.float64, device=d)
        call("gdx_init_uniform_f64", seed, WEIG_TAG, 0, first, o, i, -0.5, 0.5, t.data_ptr(), i,
             stream_handle())
        w = t.cpu().numpy().reshape(o, i)
        ws.append(w * init_scale(cfg.init, i))
        first += o * i
    return ws


def init_scale(init: str, fan_in: int) -> float:
    """Multiplier of the U(-.5,.5) weight draws (see ModelConfig.init)."""
    if init == "uniform":
        return 1.0
    if init == "he":
        return 2.0 * math.sqrt(6.0 / fan_in)
    raise InputError(f"unknown weight init {init!r}")


L2_RESIDENT_BYTES = 96 << 20  # gathered matrices up to this size stay in the 126 MB L2
# pin the gathered matrix in L2 with a persisting access-policy window (GDX_L2_WINDOW=1)
L2_WINDOW = os.environ.get("GDX_L2_WINDOW", "0") != "0"


def agg_width(fout: int, rows: int) -> int:
    """Row width of a gathered matrix.  L2-resident matrices pad to 32-byte sectors
    (what the L2 gather pays for); HBM-resident ones pad to whole 128-byte lines,
    since a misaligned row costs an extra DRAM line per gather (measured: 48-wide
    rows are slower than 64-wide ones when gathered from HBM)."""
    w8 = pad8(fout)
    if rows * w8 * 4 <= L2_RESIDENT_BYTES:
        return w8
    return 32 if fout <= 32 else (w8 + 31) // 32 * 32


AGG_ROWS = 1  # gdx.h GDX_AGG_ROWS


class _nullctx:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def source_bounds(row_ptr: torch.Tensor, col: torch.Tensor, rows: int, block: int, world: int,
                  device) -> list:
    """Per-row start of each source rank's column block [q*block, (q+1)*block) in a CSR
    with ascending columns: world+1 int64 arrays (bounds[q][v] .. bounds[q+1][v] are
    row v's sources owned by rank q)."""
    b = [torch.empty(max(rows, 1), dtype=torch.int64, device=device) for _ in range(world + 1)]
    for q in range(world):
        call("gdx_row_split", row_ptr.data_ptr(), col.data_ptr(), rows, q * block, (q + 1) * block,
             b[q].data_ptr(), b[q + 1].data_ptr(), stream_handle())
    return b


AGG_ROWS2 = 2   # half-width lane groups, two chunks per lane (degree ~8-20)
AGG_FLAT = 3    # edge-flat walk over row groups (degree < 6)


def agg_variant(width: int, nnz: int, rows: int) -> int:
    """Aggregation kernel for a CSR.  Low degree (< 20): half-width row groups -- on a
    papers-shape cooperative batch step 20.8 ms vs 21.5 (edge-flat) and 21.6 (row groups),
    tools/profile_target.py; degree 12 alone 3.60 vs 3.96 ms (tools/agg_bench.py; the
    edge-flat walk wins only on isolated degree-2.6 passes, 1.61 vs 1.68 ms).  48-wide
    rows: row groups (5% faster at degree 492).  Warp per row otherwise."""
    deg = nnz / rows if rows else 0.0
    forced = os.environ.get("GDX_AGG_LOWDEG")   # tuning: force the low-degree kernel (1, 2, 3)
    if forced and rows and deg < 20:
        return int(forced)
    if rows and deg < 7:
        return AGG_ROWS   # predicated-tail row groups: degree 3 1.60 ms vs 1.75, 6 2.33 vs 2.36
    if rows and deg < 20:
        return AGG_ROWS2
    return AGG_ROWS if pad4(width) == 48 else 0


def _splitk_eff(split_k: int, k: int) -> int:
    """Split-K count for a K of k rows with no empty split (<= split_k)."""
    kb = -(-k // 64)
    if kb <= 1:
        return 1
    per = -(-kb // min(split_k, kb))
    return -(-kb // per)


class _Layer:
    """Device state of one layer: W_cat (fp32 master + split copies), buffers."""

    def __init__(self, kind, fin, fout, nloc, nfull, d, splitk_target, first, fin_w=None, p2p=None):
        self.kind, self.fin, self.fout = kind, fin, fout
        # GEMM K: the input operand's logical width (the previous layer's row width)
        self.k = fin if first else (fin_w if fin_w is not None else pad8(fin))
        self.w = agg_width(fout, nfull)           # aggregation / row width of this layer
        self.nz = 2 * self.w if kind == "sage" else self.w   # GEMM N (W_cat rows)
        self.fin_ld = pad8(self.k)
        self.upd_cols = fin                       # weight columns the SGD pass updates
        # master weights, row pitch == split pitch so the fused SGD can index both
        self.W = torch.zeros((self.nz, self.fin_ld), dtype=torch.float32, device=d)
        self.Wsp = Split(self.nz, self.k, d, ld=self.fin_ld)  # forward B (nz x k); MN-major B of dH
        self.dW = None  # view into the trainer's flat gradient buffer (set by the trainer)
        kb = max(1, math.ceil(nloc / 64))
        ntiles = max(1, math.ceil(fin / (256 if fin > 128 else (128 if fin > 64 else 64))))
        self.split_k = max(1, min(kb, splitk_target // ntiles))
        self.ws = torch.zeros((self.split_k * self.nz, self.fin_ld), dtype=torch.float32, device=d)
        # activations
        self.S = dense(nloc, self.w, d) if kind == "sage" else None     # SAGE self path
        if p2p is None:
            self.Zfull = dense(nfull, self.w, d)                         # gathered rows
            self.dfull = dense(nfull, self.w, d)                         # gathered grads
            self.z_peers = self.d_peers = None
        else:   # shared with the peers: producers store straight into every rank's copy
            self.Zfull, self.z_peers = p2p.buffer(nfull, self.w)
            self.dfull, self.d_peers = p2p.buffer(nfull, self.w)
        self.Hout = dense(nloc, self.w, d)                               # act output fp32
        self.Hsp = Split(nloc, self.w, d)                                # next layer's A
        self.G = Split(nloc, self.nz, d)                                 # [dP | dZn] or dZ

    def set_weights(self, mats):
        """mats: [W] or [W_self, W_neigh] (fout x fin each), fp64 numpy."""
        self.W.zero_()
        if self.kind == "sage":
            ws, wn = mats
            self.W[:self.fout, :self.fin] = torch.from_numpy(ws.astype(np.float32))
            self.W[self.w:self.w + self.fout, :self.fin] = torch.from_numpy(wn.astype(np.float32))
        else:
            self.W[:self.fout, :self.fin] = torch.from_numpy(mats[0].astype(np.float32))
        self.refresh_splits()

    def refresh_splits(self):
        self.Wsp.fill_from(self.W, self.fin_ld)

    def get_weights(self, M=None):
        W = (self.W if M is None else M).double().cpu().numpy()
        if self.kind == "sage":
            return [W[:self.fout, :self.fin].copy(), W[self.w:self.w + self.fout, :self.fin].copy()]
        return [W[:self.fout, :self.fin].copy()]


class _AggFirstLayer:
    """A widening SAGE output layer run aggregate-first (SURVEY §8a a5's order choice,
    as forward_full does for widening layers): the exchange and the neighbour sum
    run at the INPUT width and only the loss rows are transformed,
        A = mean_{u in N(v)} H(u)          (H rows exchanged, fin_w wide)
        logits = [H | A] [W_s | W_n]^T     (one GEMM, K = 2 fin_w, rows = loss rows)
    backward:  dW = g^T [H | A];  [dH_self | dA] = g [W_s | W_n];
               dH(u) = dH_self(u) + sum_{v in N(u)} dA(v) / deg(v)  (dA rows exchanged).
    Same linear map as the transform-first layer; the transform-first order would
    exchange and gather fout-wide rows of every input row instead."""

    agg_first = True

    def __init__(self, fin, fout, fin_w, nloc, nfull, d, splitk_target, p2p=None):
        self.kind, self.fin, self.fout = "sage", fin, fout
        self.w = fin_w                       # exchange / aggregation width (the input's)
        self.k = 2 * fin_w                   # GEMM K: [H | A]
        self.fin_ld = self.k
        self.upd_cols = self.k               # both halves (padding columns stay zero)
        self.nz = pad8(fout)                 # W' rows (logit columns)
        self.W = torch.zeros((self.nz, self.fin_ld), dtype=torch.float32, device=d)
        self.Wsp = Split(self.nz, self.k, d, ld=self.fin_ld)
        self.dW = None
        kb = max(1, math.ceil(nloc / 64))
        ntiles = max(1, math.ceil(self.k / (256 if self.k > 128 else (128 if self.k > 64 else 64))))
        self.split_k = max(1, min(kb, splitk_target // ntiles))
        self.ws = torch.zeros((self.split_k * self.nz, self.fin_ld), dtype=torch.float32, device=d)
        if p2p is None:
            self.Xin_full = dense(nfull, fin_w, d)     # previous layer's output rows, gathered
            self.dAfull = dense(nfull, fin_w, d)       # dA / deg rows, gathered
            self.x_peers = self.da_peers = None
        else:
            self.Xin_full, self.x_peers = p2p.buffer(nfull, fin_w)
            self.dAfull, self.da_peers = p2p.buffer(nfull, fin_w)
        self.C = Split(nloc, self.k, d)                # [H | A] split operand
        self.Hout = dense(nloc, self.nz, d)            # logits
        self.Gl = Split(nloc, self.nz, d)              # g = dlogits (split)
        self.dself = dense(nloc, fin_w, d)             # g W_s
        self.dtmp = dense(nloc, fin_w, d)              # dH before the ReLU mask

    def set_weights(self, mats):
        ws, wn = mats
        self.W.zero_()
        self.W[:self.fout, :self.fin] = torch.from_numpy(ws.astype(np.float32))
        self.W[:self.fout, self.w:self.w + self.fin] = torch.from_numpy(wn.astype(np.float32))
        self.refresh_splits()

    def refresh_splits(self):
        self.Wsp.fill_from(self.W, self.fin_ld)

    def get_weights(self, M=None):
        W = (self.W if M is None else M).double().cpu().numpy()
        return [W[:self.fout, :self.fin].copy(), W[:self.fout, self.w:self.w + self.fin].copy()]

    def w_cols(self, half: int) -> Split:
        """MN-major B view of W' columns [half*fin_w, (half+1)*fin_w)."""
        v = Split.__new__(Split)
        v.rows, v.cols, v.ld = self.nz, self.w, self.fin_ld
        v.hi = _Ptr(self.Wsp.hi.data_ptr() + 2 * half * self.w)
        v.lo = _Ptr(self.Wsp.lo.data_ptr() + 2 * half * self.w)
        return v


class FullGraphTrainer:
    """Data-parallel-over-rows full-graph trainer (one instance per rank/GPU).

    pg: torch.distributed process group (None for a single GPU).  The graph is
    host-resident on every rank (generation is deterministic); each rank uploads
    only its own rows.
    """

    def __init__(self, g: Graph, cfg: ModelConfig, *, rank: int = 0, world: int = 1,
                 feature_seed: int = 1, label_seed: int = 2, weights=None, weight_seed: int = 3,
                 pg=None, device=None, subgraph=None):
        """subgraph: optional DependencySubgraph of this rank (EAS / shared-preload
        mode): the rank trains on its own preloaded inner + halo
        vertices, the loss covers its inner vertices, and only the weight gradients
        are exchanged (all-reduce over pg).  Without it, ranks own contiguous row
        blocks of the whole graph and all-gather each layer's rows."""
        require_cuda()
        if cfg.kind not in ("sage", "gcn", "sum"):
            raise InputError(f"unknown model kind {cfg.kind!r}")
        if cfg.classes > 256:
            raise InputError("classes must be <= 256")
        self.g, self.cfg, self.rank, self.world, self.pg = g, cfg, rank, world, pg
        self.d = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        d = self.d
        n = g.num_vertices()
        self.n = n
        F = cfg.dims[0]
        self.F = F
        self.subgraph_mode = subgraph is not None
        if not self.subgraph_mode:
            # ceil-sized contiguous row blocks: rank r owns [r*B, min((r+1)*B, n)); the
            # gathered buffers hold world*B rows so every all-gather block is B rows.
            B = -(-n // world)
            self.block = B
            self.offsets = np.minimum(np.arange(world + 1, dtype=np.int64) * B, n)
            self.lo, self.hi = int(self.offsets[rank]), int(self.offsets[rank + 1])
            self.nloc = self.hi - self.lo
            self.nrows_gather = world * B
            self.exchange = RowExchange(np.arange(world + 1, dtype=np.int64) * B, rank, world, pg)
            ro = g.row_offsets()
            base = int(ro[self.lo])
            lro = (ro[self.lo:self.hi + 1] - np.uint64(base)).astype(np.uint64)
            lci = g.col_indices()[base:int(ro[self.hi])]
            self.csr = DeviceCSR.upload(lro, lci, d)
            self.nnz_local = len(lci)
            deg = torch.from_numpy(np.diff(lro).astype(np.float64)).to(d)
            self.loss_rows, self.loss_count = self.nloc, float(n)
            # inputs: rows of the keyed streams (feature row v starts at draw v*F)
            self.X = dense(self.nloc, F, d)
            call("gdx_init_uniform", feature_seed, FEAT_TAG, 0, self.lo * F, self.nloc, F, -0.5, 0.5,
                 self.X.data_ptr(), self.X.shape[1], stream_handle())
            self.labels = torch.empty(max(self.nloc, 1), dtype=torch.int32, device=d)
            call("gdx_init_labels", label_seed, self.lo, self.nloc, cfg.classes,
                 self.labels.data_ptr(), stream_handle())
        else:
            from .gnn import LocalSubgraph
            loc = LocalSubgraph(subgraph, g, d)
            self.local = loc
            self.lo, self.nloc = 0, loc.n
            self.hi = loc.n
            self.nrows_gather = loc.n
            self.exchange = RowExchange(np.array([0, loc.n], np.int64), 0, 1, None)
            self.csr = loc.csr
            self.nnz_local = int(loc.lptr[-1].item())
            deg = (loc.lptr[1:] - loc.lptr[:-1]).double()
            self.loss_rows = loc.upto(0)  # inner vertices come first (hop 0)
            cnt = torch.tensor([float(self.loss_rows)], dtype=torch.float64, device=d)
            if world > 1:
                import torch.distributed as dist
                dist.all_reduce(cnt, group=pg)
            self.loss_count = float(cnt.item())
            # preloaded inputs: the global stream rows of every local vertex
            Xall = dense(n, F, d)
            call("gdx_init_uniform", feature_seed, FEAT_TAG, 0, 0, n, F, -0.5, 0.5, Xall.data_ptr(),
                 Xall.shape[1], stream_handle())
            self.X = dense(self.nloc, F, d)
            call("gdx_gather_rows", Xall.data_ptr(), Xall.shape[1], loc.l2g.data_ptr(), self.nloc, F,
                 self.X.data_ptr(), self.X.shape[1], stream_handle())
            del Xall
            lab = torch.empty(max(n, 1), dtype=torch.int32, device=d)
            call("gdx_init_labels", label_seed, 0, n, cfg.classes, lab.data_ptr(), stream_handle())
            self.labels = lab[loc.l2g[:max(self.nloc, 1)].long()].contiguous()
        # rows produced by each layer: everything in full-graph mode; in subgraph mode the
        # hop masking of forward_server_local (reference_gnn.cpp:119-137): layer l (0-based)
        # reads rows with hop <= L-l and produces rows with hop <= L-l-1, a prefix of the
        # (hop, id)-ordered local ids; rows never produced stay zero.
        Lc = cfg.layers
        if self.subgraph_mode:
            self.rows_in = [self.local.upto(Lc - l) for l in range(Lc)]
            self.rows_out = [self.local.upto(Lc - l - 1) for l in range(Lc)]
            if self.rows_in[0] < self.nloc:  # inputs beyond L hops are unavailable
                self.X[self.rows_in[0]:].zero_()
        else:
            self.rows_in = [self.nloc] * Lc
            self.rows_out = [self.nloc] * Lc
        self.inv_deg = torch.where(deg > 0, 1.0 / deg.clamp(min=1), torch.zeros_like(deg)).float()
        self.gcn_s = (1.0 / torch.sqrt(deg + 1.0)).float()
        # per-row sub-range of locally owned sources: aggregated while the all-gather runs
        xmode = os.environ.get("GDX_EXCHANGE", "p2p")
        use_p2p = (not self.subgraph_mode) and world > 1 and xmode in ("p2p", "p2p-epilogue")
        self.p2p_split = use_p2p and os.environ.get("GDX_P2P_SPLIT", "1") != "0"
        self.overlap = (not self.subgraph_mode) and world > 1 and (
            self.p2p_split or (not use_p2p and os.environ.get("GDX_OVERLAP", "1") != "0"))
        if self.overlap:
            self.seg_lo = torch.empty(max(self.nloc, 1), dtype=torch.int64, device=d)
            self.seg_hi = torch.empty(max(self.nloc, 1), dtype=torch.int64, device=d)
            call("gdx_row_split", self.csr.row_ptr.data_ptr(), self.csr.col.data_ptr(), self.nloc,
                 self.lo, self.hi, self.seg_lo.data_ptr(), self.seg_hi.data_ptr(), stream_handle())
            self.nnz_local_src = int((self.seg_hi - self.seg_lo)[:self.nloc].sum().item())
            # per-source segments for the pipelined (ring-order) exchange
            self.src_bounds = source_bounds(self.csr.row_ptr, self.csr.col, self.nloc, self.block,
                                            world, d)
            self.src_nnz = [int((self.src_bounds[q + 1] - self.src_bounds[q])[:self.nloc].sum().item())
                            for q in range(world)]
        self.Xsp = Split(self.nloc, F, d)
        self._refresh_input_splits()
        self._init_model(xmode, use_p2p, weights, weight_seed)
        torch.cuda.synchronize(d)

    def _init_model(self, xmode, use_p2p, weights, weight_seed):
        """Exchange, per-layer buffers (self.nloc local rows, self.nrows_gather gathered
        rows), the flat gradient buffer and the weights."""
        cfg, d = self.cfg, self.d
        # row exchange: NVLink peer-memory push (default) or NCCL all-gather
        self.p2p = P2PExchange(self.rank, self.world, self.pg, d,
                               "epilogue" if xmode == "p2p-epilogue" else "ce") if use_p2p else None
        sm = torch.cuda.get_device_properties(d).multi_processor_count
        self.layers = []
        for l in range(cfg.layers):
            if l == cfg.layers - 1 and l > 0 and cfg.kind == "sage" and \
                    os.environ.get("GDX_AGG_FIRST", "1") != "0" and \
                    agg_width(cfg.dims[l + 1], self.nrows_gather) > self.layers[-1].w:
                self.layers.append(_AggFirstLayer(cfg.dims[l], cfg.dims[l + 1], self.layers[-1].w,
                                                  self.nloc, self.nrows_gather, d, 2 * sm,
                                                  p2p=self.p2p))
                continue
            self.layers.append(_Layer(cfg.kind, cfg.dims[l], cfg.dims[l + 1], self.nloc,
                                      self.nrows_gather, d, 2 * sm, l == 0,
                                      self.layers[-1].w if l else None, p2p=self.p2p))
        # all weight gradients (+ the loss) in one flat buffer: one all-reduce per epoch
        sizes = [L.nz * L.fin_ld for L in self.layers]
        self.grad_flat = torch.zeros(sum(sizes) + 1, dtype=torch.float32, device=d)
        off = 0
        for L, sz in zip(self.layers, sizes):
            L.dW = self.grad_flat[off:off + sz].view(L.nz, L.fin_ld)
            off += sz
        if weights is None:
            weights = init_weights(cfg, weight_seed)
        self.set_weights(weights)
        self.partial = dense(self.nloc, max(L.w for L in self.layers), d) if self.overlap else None
        self.loss_acc = torch.zeros(1, dtype=torch.float64, device=d)
        if self.p2p is not None:
            # the layers' shared buffers are torch views over memory P2PExchange owns:
            # free it only when the trainer (and so every view) is gone
            self._p2p_finalizer = weakref.finalize(self, _close_quietly, self.p2p)
        self.keep_activations = False
        self.activations = []

    def close(self):
        """Release the captured graph, every buffer view and the peer mappings
        (call on all ranks; the trainer is unusable afterwards)."""
        self.graph = None
        self.layers = []
        self.partial = None
        torch.cuda.synchronize(self.d)
        fin = getattr(self, "_p2p_finalizer", None)
        if fin is not None:
            fin()
        self.p2p = None

    # ---- state ----
    def _refresh_input_splits(self):
        self.Xsp.fill_from(self.X, self.X.shape[1])

    def set_weights(self, weights):
        k = 2 if self.cfg.kind == "sage" else 1
        for l, layer in enumerate(self.layers):
            layer.set_weights(weights[k * l:k * l + k])

    def get_weights(self):
        out = []
        for layer in self.layers:
            out.extend(layer.get_weights())
        return out

    def get_grads(self):
        """The last step's weight gradients (reference order, like get_weights): the
        reduced dW each layer's split-K pass (+ all-reduce) left in the flat buffer."""
        out = []
        for layer in self.layers:
            out.extend(layer.get_weights(layer.dW))
        return out

    def load_features(self, x_host: torch.Tensor, labels_host: torch.Tensor | None = None):
        """H2D of this rank's feature rows (pinned host fp32, nloc x F) and labels."""
        self.X[:self.nloc, :self.F].copy_(x_host, non_blocking=True)
        if labels_host is not None:
            self.labels[:self.nloc].copy_(labels_host, non_blocking=True)
        self._refresh_input_splits()

    # ---- kernel instrumentation (bench roofline) ----
    def enable_kernel_events(self, on: bool):
        self._events = [] if on else None

    def _agg(self, csr, src, width, nnz_hint=None, **kw):
        kw.setdefault("variant", agg_variant(width, self.nnz_local, self.nloc))
        if L2_WINDOW and src.numel() * 4 <= L2_RESIDENT_BYTES:
            call("gdx_set_l2_window", src.data_ptr(), src.numel() * 4, 1.0, stream_handle())
        ev = getattr(self, "_events", None)
        if ev is None:
            return aggregate(csr, src, width, **kw)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        aggregate(csr, src, width, **kw)
        b.record()
        rows = csr.rows
        if nnz_hint is not None:            # one source block of a pipelined exchange
            nnz = nnz_hint
        elif "row_begin" in kw:             # local-source pass of a split aggregation
            nnz = self.nnz_local_src
        elif "skip" in kw:                  # remote-source pass (+ partial read)
            nnz = self.nnz_local - self.nnz_local_src
        else:
            nnz = self.nnz_local
        ev.append((a, b, 4 * nnz + 8 * (rows + 1) + 4 * width * nnz + 4 * width * rows))

    def kernel_event_summary(self):
        """(total ms, launches, algorithmic bytes) of the instrumented aggregations."""
        torch.cuda.synchronize()
        ev = getattr(self, "_events", None) or []
        return (sum(a.elapsed_time(b) for a, b, _ in ev), len(ev), sum(x for _, _, x in ev))

    def _exchange_aggregate(self, full: torch.Tensor, width: int, rows: int | None = None, **epi):
        """All-gather `full` and aggregate the owned rows from it.  With N > 1 the
        locally owned source block is aggregated while NCCL moves the remote blocks,
        then the remote sources finish the rows with the fused epilogue.  rows:
        aggregate only the first `rows` rows (hop masking in subgraph mode)."""
        csr = self.csr if rows is None or rows == self.csr.rows else self.csr.slice_rows(0, rows)
        if self.p2p is not None and not self.p2p_split:
            self.p2p.wait()
            return self._agg(csr, full, width, **epi)
        if self.p2p is not None and self.p2p.ring:
            # pipelined: peers push to us one at a time (ring order), so source block q
            # is aggregated as soon as it landed while the next one is in flight
            P = self.partial[:, :pad4(width)] if self.partial.shape[1] != pad4(width) else self.partial
            b, r, N = self.src_bounds, self.rank, self.world
            self._agg(csr, full, width, nnz_hint=self.src_nnz[r], out=P, row_begin=b[r], row_end=b[r + 1])
            for step in range(1, N):
                q = (r - step) % N
                self.p2p.wait_src(q, first=step == 1)
                if step < N - 1:
                    self._agg(csr, full, width, nnz_hint=self.src_nnz[q], row_begin=b[q],
                              row_end=b[q + 1], partial=P, out=P)
                else:
                    self._agg(csr, full, width, nnz_hint=self.src_nnz[q], row_begin=b[q],
                              row_end=b[q + 1], partial=P, **epi)
            self.p2p.join()
            return None
        if self.p2p is not None:
            # the producer already pushed our rows into every peer and signalled;
            # aggregate the owned sources, wait for the peers' rows, finish the rest
            P = self.partial[:, :pad4(width)] if self.partial.shape[1] != pad4(width) else self.partial
            self._agg(csr, full, width, out=P, row_begin=self.seg_lo, row_end=self.seg_hi)
            self.p2p.wait()
            return self._agg(csr, full, width, skip=(self.seg_lo, self.seg_hi), partial=P, **epi)
        if not self.overlap:
            self.exchange.allgather_rows(full)
            return self._agg(csr, full, width, **epi)
        work = self.exchange.allgather_rows_async(full)
        if work is None:  # gathered synchronously (unequal blocks)
            return self._agg(csr, full, width, **epi)
        P = self.partial[:, :pad4(width)] if self.partial.shape[1] != pad4(width) else self.partial
        self._agg(csr, full, width, out=P, row_begin=self.seg_lo, row_end=self.seg_hi)
        work.wait()
        return self._agg(csr, full, width, skip=(self.seg_lo, self.seg_hi), partial=P, **epi)

    # ---- collectives ----
    def _allreduce(self, t: torch.Tensor):
        """Gradient all-reduce over every rank (both modes)."""
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(t, group=self.pg)

    # ---- one epoch ----
    def _x_operand(self):
        """Layer 0's input rows as a GEMM operand: the local split copy, or (cooperative
        batches with the fused LOAD) the resident store plus the batch's row index, read
        by the GEMMs through TMA gather4 -- (split, gather index or None)."""
        xg = getattr(self, "_xg", None)
        return (self.Xsp, None) if xg is None else (self.Xall, xg)

    def forward(self):
        cfg = self.cfg
        A, xg = self._x_operand()
        acts = []
        for l, L in enumerate(self.layers):
            relu = l + 1 < cfg.layers
            m_in, r_out = self.rows_in[l], self.rows_out[l]
            if getattr(L, "agg_first", False):
                # the previous layer left its rows in L.Xin_full (own block) and their
                # split copy in L.C[:, :w]; exchange them, average the neighbours into
                # L.C[:, w:], then one GEMM over the produced rows
                self._publish(L.Xin_full[self.lo:self.hi], L.x_peers)
                self._exchange_aggregate(L.Xin_full, L.w, rows=r_out, out_split=_SplitView(L.C, L.w),
                                         self_coef=0.0, self_base=self.lo, post_scale=self.inv_deg)
                gemm_tn(L.C, L.Wsp, c0=L.Hout, m=r_out)
                if self.keep_activations:
                    acts.append(L.Hout[:self.nloc, :L.fout].clone())
                continue
            own = L.Zfull[self.lo:self.hi]
            pe = self._peers(L.z_peers, 1 if cfg.kind == "sage" else 0)
            gx = dict(a_rows=xg) if l == 0 and xg is not None else {}
            if cfg.kind == "sage":
                gemm_tn(A, L.Wsp, c0=L.S, c1=own, split=L.w, m=m_in, peers=pe, **gx)
            elif cfg.kind == "gcn":
                gemm_tn(A, L.Wsp, c0=own, row_scale=self.gcn_s, m=m_in, peers=pe, **gx)
            else:
                gemm_tn(A, L.Wsp, c0=own, m=m_in, peers=pe, **gx)
            self._publish(own, L.z_peers, stored=pe is not None)
            nxt = self.layers[l + 1] if l + 1 < cfg.layers else None
            if getattr(nxt, "agg_first", False):   # output rows feed an aggregate-first layer
                out, out_split = nxt.Xin_full[self.lo:self.hi], _SplitView(nxt.C, 0)
            else:
                out, out_split = L.Hout, L.Hsp
            if cfg.kind == "sage":
                self._exchange_aggregate(L.Zfull, L.w, rows=r_out, out=out, out_split=out_split,
                                         self_coef=0.0, self_base=self.lo, post_scale=self.inv_deg,
                                         add=L.S, relu=relu)
            elif cfg.kind == "gcn":
                self._exchange_aggregate(L.Zfull, L.w, rows=r_out, out=out, out_split=out_split,
                                         self_coef=1.0, self_base=self.lo, post_scale=self.gcn_s, relu=relu)
            else:
                self._exchange_aggregate(L.Zfull, L.w, rows=r_out, out=out, out_split=out_split,
                                         self_coef=1.0, self_base=self.lo, relu=relu)
            A = L.Hsp
            if self.keep_activations:
                acts.append(out[:self.nloc, :L.fout].clone())
        self.activations = acts
        return self.layers[-1].Hout

    def _act(self, l: int) -> torch.Tensor:
        """fp32 output rows of layer l (the ReLU mask of its backward)."""
        nxt = self.layers[l + 1] if l + 1 < len(self.layers) else None
        if getattr(nxt, "agg_first", False):
            return nxt.Xin_full[self.lo:self.hi]
        return self.layers[l].Hout

    def _peers(self, deltas, target: int):
        if self.p2p is None or deltas is None or self.p2p.mode != "epilogue":
            return None
        return (target, deltas)

    def _publish(self, own: torch.Tensor, deltas, stored: bool = False):
        """After the producer of an exchanged buffer: make our rows visible to peers.
        stored: the producer was launched with peers= (GDX_EXCHANGE=p2p-epilogue) and
        already wrote the rows into every peer's copy, so only the arrival signal is
        left.  Producers without peer stores (the aggregate kernel writing an
        aggregate-first layer's input rows, the dA GEMM, gdx_grad_prepare) are pushed
        by the SM push kernel in every mode."""
        if self.p2p is None:
            return
        if stored and self.p2p.mode == "epilogue":
            self.p2p.signal()
        else:
            self.p2p.push(own, deltas, rows=getattr(self, "send_rows", None))

    def _grad_targets(self, l: int):
        """Where the prepared gradient of layer l's output goes: gs = g * dst_scale into the
        gathered buffer's own rows, and (SAGE) the unscaled split copy into G[:, :w]."""
        L = self.layers[l]
        own = L.dfull[self.lo:self.hi]
        scale = {"sage": self.inv_deg, "gcn": self.gcn_s}.get(self.cfg.kind)
        split = L.G if self.cfg.kind == "sage" else None
        return own, scale, split

    def backward_and_step(self):
        """Backward of every layer + SGD.  The last layer's g comes fused out of the
        softmax kernel; each lower layer's g = dH * relu' (scaled for the next
        aggregation, split for the weight gradient) comes fused out of the dH GEMM
        epilogue, so there is no separate elementwise pass."""
        cfg = self.cfg
        nL = cfg.layers
        for l in range(nL - 1, -1, -1):
            L = self.layers[l]
            r_in = self.rows_in[l]   # dZ is needed for the rows that fed layer l
            if getattr(L, "agg_first", False):
                self._backward_agg_first(l)
                continue
            # dZ = agg^T(gs): SAGE -> G[:, w:2w]; GCN/SUM -> G (all columns)
            if cfg.kind == "sage":
                Gn = _SplitView(L.G, L.w)
                self._exchange_aggregate(L.dfull, L.w, rows=r_in, out_split=Gn, self_coef=0.0,
                                         self_base=self.lo)
            elif cfg.kind == "gcn":
                self._exchange_aggregate(L.dfull, L.w, rows=r_in, out_split=L.G, self_coef=1.0,
                                         self_base=self.lo, post_scale=self.gcn_s)
            else:
                self._exchange_aggregate(L.dfull, L.w, rows=r_in, out_split=L.G, self_coef=1.0,
                                         self_base=self.lo)
            # dH_{l} = G W_cat (before this layer's update; W_cat read MN-major in place),
            # epilogue: ReLU backward with H_{l} as mask, scale, split -> layer l-1's inputs
            if l > 0:
                own, scale, split = self._grad_targets(l - 1)
                pe = self._peers(self.layers[l - 1].d_peers, 0)
                gemm_tn(L.G, L.Wsp, c0=own, b_mn=True, mask=self._act(l - 1),
                        row_scale=scale, out_split=split, split_unscaled=True, m=self.rows_out[l - 1],
                        peers=pe)
                self._publish(own, self.layers[l - 1].d_peers, stored=pe is not None)
            # dW = G^T H_in, split-K over the local rows; both operands MN-major in place
            # (K = the rows that fed layer l; rows past them carry no gradient)
            A_in = self.Xsp if l == 0 else self.layers[l - 1].Hsp
            Bop, gx = A_in.rows_view(r_in), {}
            if l == 0:
                xs, xg = self._x_operand()
                if xg is not None:
                    Bop, gx = xs, dict(b_rows=xg[:r_in])
            sk = _splitk_eff(L.split_k, r_in)
            ws = self._wstream()
            if ws is not None:  # overlap with the next layer's (L2-bound) aggregation
                ws.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(ws) if ws is not None else _nullctx():
                gemm_tn(L.G.rows_view(r_in), Bop, c0=L.ws, split_k=sk, a_mn=True, b_mn=True, **gx)
                self._sgd_or_reduce(L, sk, L.upd_cols)
        if getattr(self, "_ws", None) is not None:
            torch.cuda.current_stream().wait_stream(self._ws)
        if self.world > 1:
            # one all-reduce for every layer's dW and the loss, then SGD (+ split refresh)
            self.grad_flat[-1:].copy_(self.loss_acc)
            self._allreduce(self.grad_flat)
            self.loss_acc.copy_(self.grad_flat[-1:])
            for L in self.layers:
                call("gdx_splitk_reduce", L.dW.data_ptr(), 1, 0, L.nz, L.upd_cols, L.fin_ld, None,
                     L.W.data_ptr(), cfg.lr, L.Wsp.hi.data_ptr(), L.Wsp.lo.data_ptr(), stream_handle())

    def _wstream(self):
        """Side stream for the weight-gradient GEMMs (GDX_DW_OVERLAP=1), else None."""
        if os.environ.get("GDX_DW_OVERLAP", "0") == "0":
            return None
        if getattr(self, "_ws", None) is None:
            self._ws = torch.cuda.Stream(device=self.d)
        return self._ws

    def _sgd_or_reduce(self, L, sk: int, cols: int):
        """Reduce layer L's split-K partials into dW; on one GPU also apply SGD (and
        refresh the split copy) in the same pass."""
        if self.world == 1:  # reduce split-K partials and apply SGD in one pass
            call("gdx_splitk_reduce", L.ws.data_ptr(), sk, L.nz * L.fin_ld, L.nz, cols, L.fin_ld,
                 L.dW.data_ptr(), L.W.data_ptr(), self.cfg.lr, L.Wsp.hi.data_ptr(), L.Wsp.lo.data_ptr(),
                 stream_handle())
        else:                # reduce partials; SGD after the epoch's single all-reduce
            call("gdx_splitk_reduce", L.ws.data_ptr(), sk, L.nz * L.fin_ld, L.nz, cols, L.fin_ld,
                 L.dW.data_ptr(), None, 0.0, None, None, stream_handle())

    def _backward_agg_first(self, l: int):
        """Backward of an aggregate-first layer (g = dlogits in L.Gl, split)."""
        L = self.layers[l]
        r = self.rows_out[l]
        # [dH_self | dA/deg] = g [W_s | W_n] with the pre-update weights
        gemm_tn(L.Gl, L.w_cols(0), c0=L.dself, b_mn=True, m=r)
        own = L.dAfull[self.lo:self.hi]
        gemm_tn(L.Gl, L.w_cols(1), c0=own, b_mn=True, row_scale=self.inv_deg, m=r)
        self._publish(own, L.da_peers)
        # dW' = g^T [H | A] over the produced rows (runs while the dA rows move)
        sk = _splitk_eff(L.split_k, r)
        gemm_tn(L.Gl.rows_view(r), L.C.rows_view(r), c0=L.ws, split_k=sk, a_mn=True, b_mn=True)
        self._sgd_or_reduce(L, sk, L.upd_cols)
        # dH(u) = dH_self(u) + sum_{v in N(u)} dA(v)/deg(v), over the rows that fed layer l
        self._exchange_aggregate(L.dAfull, L.w, rows=self.rows_in[l], out=L.dtmp, self_coef=0.0,
                                 self_base=self.lo, add=L.dself)
        # ReLU backward + the previous layer's gradient targets (scaled rows to gather,
        # unscaled split copy for its dW), then publish them
        pown, scale, split = self._grad_targets(l - 1)
        act = self._act(l - 1)
        call("gdx_grad_prepare", L.dtmp.data_ptr(), L.dtmp.shape[1], act.data_ptr(), act.stride(0),
             self.rows_out[l - 1], L.w, _lib.ptr(scale), None, 0, pown.data_ptr(), pown.stride(0),
             _lib.ptr(split.hi) if split is not None else None,
             _lib.ptr(split.lo) if split is not None else None, split.ld if split is not None else 0,
             stream_handle())
        self._publish(pown, self.layers[l - 1].d_peers)

    def train_epoch(self, sync_loss: bool = True):
        """Forward, loss, backward, SGD.  Returns the loss (host float) if sync_loss."""
        self.loss_acc.zero_()
        logits = self.forward()
        Llast = self.layers[-1]
        if getattr(Llast, "agg_first", False):
            # g = dlogits, split only (its consumers are the layer's own GEMMs)
            call("gdx_softmax_xent_fused", logits.data_ptr(), logits.shape[1], self.loss_rows,
                 self.cfg.classes, self.labels.data_ptr(), 1.0 / self.loss_count, None, 0, None,
                 None, 0, Llast.Gl.hi.data_ptr(), Llast.Gl.lo.data_ptr(), Llast.Gl.ld,
                 self.loss_acc.data_ptr(), stream_handle())
            self.backward_and_step()
            if sync_loss:
                return float(self.loss_acc.item()) / self.loss_count
            return None
        own, scale, split = self._grad_targets(self.cfg.layers - 1)
        if self._peers(self.layers[-1].d_peers, 0) is not None:   # p2p-epilogue: softmax stores to peers
            Lz = self.layers[-1]
            deltas = (_lib.C.c_int64 * 7)(*Lz.d_peers)
            call("gdx_softmax_xent_fused_peers", logits.data_ptr(), logits.shape[1], self.loss_rows,
                 self.cfg.classes, self.labels.data_ptr(), 1.0 / self.loss_count, _lib.ptr(scale),
                 own.data_ptr(), own.stride(0), _lib.ptr(split.hi) if split is not None else None,
                 _lib.ptr(split.lo) if split is not None else None, split.ld if split is not None else 0,
                 self.loss_acc.data_ptr(), len(Lz.d_peers), deltas, stream_handle())
            self.p2p.signal()
        else:
            call("gdx_softmax_xent_fused", logits.data_ptr(), logits.shape[1], self.loss_rows,
                 self.cfg.classes, self.labels.data_ptr(), 1.0 / self.loss_count, None, 0,
                 _lib.ptr(scale), own.data_ptr(), own.stride(0),
                 _lib.ptr(split.hi) if split is not None else None,
                 _lib.ptr(split.lo) if split is not None else None,
                 split.ld if split is not None else 0, self.loss_acc.data_ptr(), stream_handle())
            if self.p2p is not None:
                self._publish(own, self.layers[-1].d_peers)
        self.backward_and_step()  # (multi-GPU: the loss rides on the gradient all-reduce)
        if sync_loss:
            return float(self.loss_acc.item()) / self.loss_count
        return None

    # ---- CUDA graph of one epoch (removes host launch overhead) ----
    def capture(self, warmup: int = 2):
        """Capture one epoch (forward, loss, backward, collectives, SGD) as a CUDA
        graph.  All buffers are static (allocated in __init__ / first epochs), TMA
        descriptors travel by value in the kernel nodes, NCCL collectives are
        captured on the same stream."""
        for _ in range(warmup):
            self.train_epoch(sync_loss=False)
        torch.cuda.synchronize(self.d)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.train_epoch(sync_loss=False)
        torch.cuda.synchronize(self.d)
        return self.graph

    def replay(self, sync_loss: bool = False):
        self.graph.replay()
        if sync_loss:
            return float(self.loss_acc.item()) / self.loss_count
        return None


class FeatureStream:
    """Double-buffered host->device feature loading for the end-to-end path: the
    next step's feature block is copied (own stream, pinned source) while the
    current epoch computes; consume() orders the compute stream after the copy,
    converts it to the split-bf16 GEMM operand and frees the staging buffer."""

    def __init__(self, tr: "FullGraphTrainer"):
        self.tr = tr
        d = tr.d
        self.stage = [torch.empty((tr.nloc, tr.F), dtype=torch.float32, device=d) for _ in range(2)]
        self.labels = [torch.empty_like(tr.labels) for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(device=d)
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]
        self.issued = 0
        self.consumed = 0
        # per-copy timing events on the copy stream (H2D duration under overlap)
        self.copy_events: list[tuple[torch.cuda.Event, torch.cuda.Event]] = []

    def copy_ms(self) -> float:
        """Mean duration of the issued copies (call after they completed)."""
        if not self.copy_events:
            return 0.0
        return sum(a.elapsed_time(b) for a, b in self.copy_events) / len(self.copy_events)

    def prefetch(self, x_host: torch.Tensor, labels_host: torch.Tensor | None = None):
        i = self.issued % 2
        cs = self.copy_stream
        if self.issued >= 2:
            cs.wait_event(self.free[i])
        cs.wait_stream(torch.cuda.current_stream()) if self.issued == 0 else None
        with torch.cuda.stream(cs):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            # the stage is contiguous [nloc, F] (the host layout), so this is ONE DMA at
            # the PCIe rate; consume() splits it with ld = F.  (Copying into the 16-byte
            # padded view instead makes torch stage a temporary and repack it with a
            # kernel that competes with the running epoch for SMs: 10.1 ms alone ->
            # 14-16 ms; a pitched cudaMemcpy2DAsync with 2408-byte rows ran at 17 GB/s.)
            if x_host.shape != (self.tr.nloc, self.tr.F) or x_host.dtype != torch.float32:
                raise InputError(f"FeatureStream: features must be float32 [{self.tr.nloc}, {self.tr.F}]")
            if not x_host.is_pinned() or not x_host.is_contiguous():
                raise InputError("FeatureStream: features must be pinned, contiguous host memory")
            self.stage[i].copy_(x_host, non_blocking=True)
            if labels_host is not None:
                self.labels[i][:self.tr.nloc].copy_(labels_host, non_blocking=True)
            e1.record(cs)
            self.copy_events.append((e0, e1))
            self.ready[i].record(cs)
        self.issued += 1

    def consume(self, with_labels: bool = True):
        i = self.consumed % 2
        cur = torch.cuda.current_stream()
        cur.wait_event(self.ready[i])
        tr = self.tr
        tr.Xsp.fill_from(self.stage[i], tr.F)
        if with_labels:
            tr.labels.copy_(self.labels[i])
        self.free[i].record(cur)
        self.consumed += 1


class _RawCUDA:
    """CUDA Array Interface wrapper so torch can view memory libgdx allocated."""

    def __init__(self, ptr: int, shape, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def _close_quietly(p2p: "P2PExchange"):
    try:
        p2p.close()
    except Exception:  # interpreter teardown: the CUDA context may already be gone
        pass


class P2PExchange:
    """Row exchange over NVLink peer memory, no NCCL on the data path.

    Each gathered buffer is a separate cudaMalloc allocation whose CUDA IPC handle is
    shared with every rank (or, for 'mc', a torch symmetric-memory allocation with an
    NVSwitch multicast mapping).  After the producer (GEMM / softmax) has written this
    rank's rows into its own buffer, the rows are pushed to the same offset in every
    peer's buffer and each peer's arrival slot for this rank is bumped:
      'sm' (default): one push kernel, 16-byte NVLink stores to every peer, the last
            CTA releases the stores and signals (680 GB/s received per GPU at N=4,
            tools/xch_bench.py; NCCL all-gather 546, copy engines 366);
      'ce': copy engines, one stream per peer, then a signal kernel;
      'mc': multimem.st through the multicast mapping (one store, the switch
            replicates; not faster: an all-gather is bound by each GPU's ingress);
      'epilogue': the producing GEMM / softmax epilogue stores into the peers itself.
    `wait()` (before the remote-source aggregation) spins until every peer's slot
    reached the round."""

    # A wedged peer makes gdx_peer_wait trap after this long instead of hanging forever
    # (GDX_PEER_TIMEOUT_S, default 20 s).  A trap is a sticky device fault: it poisons
    # this process's CUDA context, so the process must exit -- there is no recovery.
    TIMEOUT_NS = int(float(os.environ.get("GDX_PEER_TIMEOUT_S", "20")) * 1e9)

    def __init__(self, rank: int, world: int, pg, device, mode: str = "ce"):
        """mode 'ce': the producer writes locally; copy engines push the owned rows to
        every peer on a side stream, overlapping the local-source aggregation (no SMs
        spent on the transfer).  mode 'epilogue': the GEMM / softmax epilogue itself
        stores into the peers (bulk async copies of each finished tile)."""
        import torch.distributed as dist
        self.rank, self.world, self.pg, self.d = rank, world, pg, device
        self.mode = mode
        # copy-engine streams: `ce_split` per peer (one copy engine sustains ~200 GB/s of
        # NVLink writes; several in parallel approach the link rate)
        self.ce_split = max(1, int(os.environ.get("GDX_CE_SPLIT", "1")))
        # 'sm': one SM-driven push kernel (all peers, fused signal) on a side stream
        # 'mc': buffers in torch symmetric memory with an NVSwitch multicast mapping; the
        # push stores each vector once and the switch replicates it to every GPU
        self.push_kind = os.environ.get("GDX_PUSH", "sm")
        self._mc_bufs = []   # (local base, bytes, multicast base, handle)
        if self.push_kind == "mc":
            import torch.distributed._symmetric_memory as symm
            self._symm = symm
            try:
                symm.enable_symm_mem_for_group(pg.group_name)
            except Exception:  # newer torch enables it implicitly
                pass
        self.push_ctas = int(os.environ.get("GDX_PUSH_CTAS", "32"))
        # ring order (GDX_P2P_RING=1): push to rank+1, rank+2, ... one peer at a time and
        # aggregate each source block as it lands.  Measured slower at N=4 (Reddit 3.41 vs
        # 3.09 ms, products 10.96 vs 10.25 ms): one GPU pair gets well under the GPU's
        # NVLink ingress, so the all-peer push wins; kept as an option.
        self.ring = self.push_kind == "sm" and world > 2 and os.environ.get("GDX_P2P_RING", "0") != "0"
        self.push_done = torch.zeros(1, dtype=torch.int32, device=device)
        self.sides = [torch.cuda.Stream(device=device) for _ in range((world - 1) * self.ce_split)]
        self.pushed = None
        self._owned, self._opened = [], []
        self.slots = self._alloc(8 * world)            # arrival slot per source rank
        self.expected = self._alloc(8)                 # rounds this rank has waited for
        handles = self._gather_handle(self.slots)
        peer_slot_ptrs = []
        for r in range(world):
            if r == rank:
                continue
            base = self._open(handles[r])
            peer_slot_ptrs.append(base + 8 * rank)      # our slot in peer r's array
        self.peer_slots_dev = torch.tensor(peer_slot_ptrs, dtype=torch.int64, device=device)
        dist.barrier(group=pg)

    def _alloc(self, nbytes: int) -> int:
        p = _lib.C.c_void_p()
        call("gdx_device_alloc", nbytes, _lib.C.byref(p))
        self._owned.append(p.value)
        return p.value

    def _open(self, handle: bytes) -> int:
        buf = _lib.C.create_string_buffer(handle, 64)
        p = _lib.C.c_void_p()
        call("gdx_ipc_open", buf, _lib.C.byref(p))
        self._opened.append(p.value)
        return p.value

    def _gather_handle(self, ptr: int) -> list:
        import torch.distributed as dist
        h = _lib.C.create_string_buffer(64)
        call("gdx_ipc_get_handle", ptr, h)
        out = [None] * self.world
        dist.all_gather_object(out, h.raw, group=self.pg)
        return out

    def buffer(self, rows: int, cols: int):
        """Zeroed [rows, cols] fp32 buffer shared with every peer; returns
        (tensor, byte deltas to the same address in each peer's buffer)."""
        if self.push_kind == "mc":
            t = self._symm.empty((max(rows, 1), cols), dtype=torch.float32, device=self.d)
            t.zero_()
            hdl = self._symm.rendezvous(t, self.pg.group_name)
            if not hdl.multicast_ptr:
                raise InternalError("GDX_PUSH=mc: no NVSwitch multicast support on this system")
            base = t.data_ptr()
            # symmetric allocations may sit at an offset inside the mapped buffer
            mc = hdl.multicast_ptr + (base - hdl.buffer_ptrs[self.rank])
            self._mc_bufs.append((base, t.numel() * 4, mc, hdl, t))
            deltas = [hdl.buffer_ptrs[r] - hdl.buffer_ptrs[self.rank] for r in range(self.world) if r != self.rank]
            return t[:rows], deltas
        ptr = self._alloc(rows * cols * 4)
        t = torch.as_tensor(_RawCUDA(ptr, (rows, cols)), device=self.d)
        handles = self._gather_handle(ptr)
        deltas = [self._open(handles[r]) - ptr for r in range(self.world) if r != self.rank]
        return t, deltas

    def signal(self):
        call("gdx_peer_signal", self.peer_slots_dev.data_ptr(), self.world - 1, stream_handle())

    def push(self, own: torch.Tensor, deltas, rows=None):
        """'ce' mode: after the producer, copy the owned (contiguous) rows into each
        peer's buffer with copy engines (ce_split streams per peer, 256-byte aligned
        pieces), then signal that peer once all its pieces landed."""
        main = torch.cuda.current_stream()
        nbytes = own.numel() * own.element_size()
        if rows is not None and self.push_kind in ("sm", "mc"):
            # sparse: only the rows each peer reads (row lists from the batch geometry)
            idx, off = rows
            st = self.sides[0]
            st.wait_stream(main)
            d = (_lib.C.c_int64 * 7)(*deltas)
            o = (_lib.C.c_uint64 * 8)(*off)
            with torch.cuda.stream(st):
                call("gdx_push_rows", own.data_ptr(), own.stride(0) * own.element_size(), idx.data_ptr(), o, d,
                     len(deltas), self.peer_slots_dev.data_ptr(), self.push_done.data_ptr(),
                     max(self.push_ctas, 64), stream_handle())
            self.pushed = [st]
            return
        if self.push_kind == "mc":
            st = self.sides[0]
            st.wait_stream(main)
            p = own.data_ptr()
            mc = next(m + (p - b) for b, n, m, _, _ in self._mc_bufs if b <= p < b + n)
            with torch.cuda.stream(st):
                call("gdx_push_multicast", p, nbytes, mc, len(deltas), self.peer_slots_dev.data_ptr(),
                     self.push_done.data_ptr(), self.push_ctas, stream_handle())
            self.pushed = [st]
            return
        if self.push_kind == "sm" and self.ring:
            st = self.sides[0]
            st.wait_stream(main)
            slot0 = self.peer_slots_dev.data_ptr()
            with torch.cuda.stream(st):
                for step in range(1, self.world):
                    q = (self.rank + step) % self.world
                    i = q if q < self.rank else q - 1
                    d = (_lib.C.c_int64 * 7)(deltas[i])
                    call("gdx_push_peers", own.data_ptr(), nbytes, d, 1, slot0 + 8 * i,
                         self.push_done.data_ptr(), self.push_ctas, stream_handle())
            self.pushed = [st]
            return
        if self.push_kind == "sm":
            st = self.sides[0]
            st.wait_stream(main)
            d = (_lib.C.c_int64 * 7)(*deltas)
            with torch.cuda.stream(st):
                call("gdx_push_peers", own.data_ptr(), nbytes, d, len(deltas), self.peer_slots_dev.data_ptr(),
                     self.push_done.data_ptr(), self.push_ctas, stream_handle())
            self.pushed = [st]
            return
        K = self.ce_split
        piece = ((nbytes + K - 1) // K + 255) // 256 * 256
        slot0 = self.peer_slots_dev.data_ptr()
        base = own.data_ptr()
        for i, dl in enumerate(deltas):
            sts = self.sides[i * K:(i + 1) * K]
            for j, st in enumerate(sts):
                st.wait_stream(main)
                lo = min(nbytes, j * piece)
                hi = min(nbytes, lo + piece)
                if hi > lo:
                    with torch.cuda.stream(st):
                        call("gdx_memcpy_async", base + lo + dl, base + lo, hi - lo, stream_handle())
            for st in sts[1:]:
                sts[0].wait_stream(st)
            with torch.cuda.stream(sts[0]):
                call("gdx_peer_signal", slot0 + 8 * i, 1, stream_handle())
        self.pushed = self.sides[:len(deltas) * K]

    def wait_src(self, src: int, first: bool):
        """Pipelined wait: block the stream until source rank `src`'s rows of this round
        landed (first=True starts the round)."""
        call("gdx_peer_wait_src", self.slots, self.expected, src, int(first), self.TIMEOUT_NS,
             stream_handle())

    def join(self):
        """Order the stream after our own pushes (before the pushed rows are rewritten)."""
        if self.pushed:
            main = torch.cuda.current_stream()
            for st in self.pushed:
                main.wait_stream(st)
            self.pushed = None

    def wait(self):
        if self.pushed:  # our pushes finished (the push streams join the main stream)
            main = torch.cuda.current_stream()
            for st in self.pushed:
                main.wait_stream(st)
            self.pushed = None
        call("gdx_peer_wait", self.slots, self.expected, self.world, self.rank, self.TIMEOUT_NS,
             stream_handle())

    def close(self):
        """Unmap the peers' buffers and free ours.  Only valid once nothing views the
        memory any more: FullGraphTrainer.close() drops its views first, and a
        weakref finalizer runs this when the trainer is collected."""
        for p in self._opened:
            _lib.lib().gdx_ipc_close(p)
        self._opened = []
        for p in self._owned:
            _lib.lib().gdx_device_free(p)
        self._owned = []


class RowExchange:
    """The per-layer exchange of a row-partitioned full graph:
    every rank owns the contiguous row block offsets[r]:offsets[r+1] of a
    [n, w] matrix and receives everybody else's block (all-gather); weight
    gradients are summed (all-reduce).  NCCL on GPUs; any torch.distributed
    backend works, which is how the CPU tests drive it with gloo."""

    def __init__(self, offsets, rank: int, world: int, pg=None):
        self.offsets = np.asarray(offsets, np.int64)
        self.rank, self.world, self.pg = rank, world, pg
        sizes = np.diff(self.offsets)
        self.equal_blocks = bool(np.all(sizes == sizes[0]))

    def allgather_rows_async(self, full: torch.Tensor):
        """Start the all-gather on NCCL's stream (equal blocks); returns a handle whose
        wait() orders the current stream after it, or None when nothing to do."""
        if self.world == 1 or not self.equal_blocks:
            self.allgather_rows(full)
            return None
        import torch.distributed as dist
        n = int(self.offsets[-1])
        lo, hi = int(self.offsets[self.rank]), int(self.offsets[self.rank + 1])
        return dist.all_gather_into_tensor(full[:n], full[lo:hi], group=self.pg, async_op=True)

    def allgather_rows(self, full: torch.Tensor):
        if self.world == 1:
            return
        import torch.distributed as dist
        n = int(self.offsets[-1])
        lo, hi = int(self.offsets[self.rank]), int(self.offsets[self.rank + 1])
        if self.equal_blocks:
            dist.all_gather_into_tensor(full[:n], full[lo:hi].clone() if full.device.type == "cpu"
                                        else full[lo:hi], group=self.pg)
        else:
            # unequal blocks: gather padded blocks, then scatter them into place
            sizes = np.diff(self.offsets)
            mb = int(sizes.max())
            send = torch.zeros((mb,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
            send[:hi - lo] = full[lo:hi]
            recv = torch.empty((self.world * mb,) + tuple(full.shape[1:]), dtype=full.dtype,
                               device=full.device)
            dist.all_gather_into_tensor(recv, send, group=self.pg)
            for r in range(self.world):
                if r != self.rank:
                    a, b = int(self.offsets[r]), int(self.offsets[r + 1])
                    full[a:b].copy_(recv[r * mb:r * mb + (b - a)])

    def allreduce(self, t: torch.Tensor):
        if self.world == 1:
            return
        import torch.distributed as dist
        dist.all_reduce(t, group=self.pg)


class _SplitView:
    """Column-offset view of a Split (writes into columns [off, ...))."""

    def __init__(self, s: Split, off: int):
        self.ld = s.ld
        self.hi = _Ptr(s.hi.data_ptr() + 2 * off)
        self.lo = _Ptr(s.lo.data_ptr() + 2 * off)


class _Ptr:
    def __init__(self, p):
        self.p = p

    def data_ptr(self):
        return self.p
