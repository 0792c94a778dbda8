"""Cooperative-batching training: the batches of a
``plan_cobatch[_fixed_r]`` plan (batch_plan.cpp:103-153) trained one after
another, each split across the server's GPUs by ``split_batch``
(sim.cpp:81-102) with a per-layer row exchange inside the batch.

Semantics (builder-defined: the reference prices batches in ``simulate_epoch``,
sim.cpp:223-266, but has no training code, so parity here is against the fp64
oracle, unpinned against the reference):

* a batch is the reference ``Batch``: sorted targets and the sampled closure
  ``vertices`` (batch_closure, batch_plan.cpp:28-70);
* vertex v of the batch gets its peel distance d(v) from the targets over the
  batch's induced adjacency -- exactly the levels ``peel_mfg`` counts
  (batch_plan.cpp:75-101), so ``mfg_vertices_per_layer[l] == |{d <= L-l}|``;
* layer l (1-based) computes the rows with d <= L-l from their in-batch
  neighbours (forward_server_local's hop masking, reference_gnn.cpp:119-137,
  with hop := d); the loss is the mean softmax cross-entropy over the targets;
  one SGD step per batch (Alg. 1 of the paper: R updates per epoch);
* GPU w of the server owns the rows ``split_batch`` gives it; local row ids are
  ordered (owner, d, id) and padded to a common block, so every rank's rows valid
  at layer l are a prefix of its block and the exchange is the same equal-block
  push / all-gather as full-graph training.

The per-batch geometry (local CSR in padded ids, degrees, hop prefixes) is built
once on the device and stays resident; each epoch then LOADs the batch's input
rows from the resident split-bf16 feature store (``gdx_gather_split_rows``) and
runs forward / loss / backward / SGD for every batch.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call
from .batch_plan import BatchPlan
from .device import DeviceCSR, Split, dense, require_cuda, stream_handle
from .errors import InputError
from .extract import kUnlimitedFanout, sampled_growth_device
from .graph import Graph, Partition
from .train import FEAT_TAG, FullGraphTrainer, ModelConfig, RowExchange, source_bounds


@dataclass
class BatchGeometry:
    """One rank's view of one batch."""
    csr: DeviceCSR          # rows = this rank's block, columns = padded batch ids
    l2g: torch.Tensor       # int32 [nloc] global id of each local row, (d, id) order
    nloc: int
    block: int              # padded block size (every rank's rows start at rank*block)
    rows_in: list           # per layer: rows read (d <= L-l)
    rows_out: list          # per layer: rows produced (d <= L-l-1)
    loss_rows: int          # targets of this rank (d == 0, a prefix)
    loss_count: int         # targets of the batch (all ranks)
    nnz: int
    nnz_src: int            # entries whose source this rank owns
    inv_deg: torch.Tensor
    gcn_s: torch.Tensor
    seg_lo: torch.Tensor | None
    seg_hi: torch.Tensor | None
    mfg: list               # |{d <= L-l}| over the whole batch, l = 0..L (== peel_mfg)
    edges_per_step: int     # CSR entries aggregated by this rank per step (fwd + bwd passes)
    src_bounds: list = None  # per-source column segments (pipelined exchange)
    src_nnz: list = None
    send_rows: tuple = None  # (u32 row indices of this block, per-peer offsets) for sparse pushes


def split_batch_share(vb: torch.Tensor, sp: torch.Tensor, gp: torch.Tensor, server: int,
                      gpus: int) -> torch.Tensor:
    """split_batch (sim.cpp:81-102) on the device: GPU of each batch vertex (int32)."""
    nb = vb.numel()
    share = torch.empty(max(nb, 1), dtype=torch.int32, device=vb.device)
    if nb:
        work = torch.empty(5 * nb + 2 * gpus + 8, dtype=torch.int32, device=vb.device)
        call("gdx_split_batch", vb.data_ptr(), nb, sp.data_ptr(), gp.data_ptr(), server, gpus,
             share.data_ptr(), work.data_ptr(), stream_handle())
    return share[:nb]


def exchange_row_needs(cols: torch.Tensor, block: int, rank: int, world: int, pg):
    """Which rows of this rank's block each peer's CSR references -- the reference
    simulator's per-GPU 'deps' (sim.cpp:241-250).  Every rank lists the rows it reads
    from each source block (cols: its CSR columns in padded ids), one all_to_all hands
    each list to its source.  Returns (row indices within this rank's block, int32,
    concatenated over the peers r != rank in ascending order; offsets, len world)."""
    import torch.distributed as dist
    d = cols.device
    c = cols.long()
    need = []
    for q in range(world):
        if q == rank:
            need.append(torch.zeros(0, dtype=torch.int32, device=d))
            continue
        sel = c[(c >= q * block) & (c < (q + 1) * block)]
        need.append((torch.unique(sel) - q * block).to(torch.int32))
    counts = torch.tensor([t.numel() for t in need], dtype=torch.int64, device=d)
    got = torch.empty_like(counts)
    dist.all_to_all_single(got, counts, group=pg)
    ns, nr = int(counts.sum()), int(got.sum())
    send = torch.cat(need) if ns else torch.zeros(1, dtype=torch.int32, device=d)
    recv = torch.empty(max(nr, 1), dtype=torch.int32, device=d)
    dist.all_to_all_single(recv[:nr], send[:ns], output_split_sizes=got.tolist(),
                           input_split_sizes=counts.tolist(), group=pg)
    g = got.tolist()
    off = [0]
    for q in range(world):
        if q != rank:
            off.append(off[-1] + g[q])
    return recv, off


def _dev_assign(p, device) -> torch.Tensor:
    """Device int32 copy of a Partition's assignment (tensors pass through)."""
    if isinstance(p, torch.Tensor):
        return p
    return torch.from_numpy(np.ascontiguousarray(p.assignment, np.uint32).view(np.int32)).to(device)


def batch_geometry(g: Graph, targets: np.ndarray, vertices: np.ndarray, sp: Partition,
                   gp: Partition, server: int, rank: int, world: int, layers: int,
                   device, sort_sources: bool) -> BatchGeometry:
    """Peel levels, owner split, (owner, d, id) numbering and the rank's local CSR."""
    n = g.num_vertices()
    dg = g.device(device)
    vb = torch.from_numpy(np.ascontiguousarray(vertices, np.uint32).view(np.int32)).to(device)
    tb = torch.from_numpy(np.ascontiguousarray(targets, np.uint32).view(np.int32)).to(device)
    in_batch = torch.zeros(max(n, 1), dtype=torch.uint8, device=device)
    in_batch[vb.long()] = 1
    tmask = torch.zeros(max(n, 1), dtype=torch.uint8, device=device)
    tmask[tb.long()] = 1
    # peel levels = BFS distance from the targets inside the batch (unlimited fanout growth)
    mark = sampled_growth_device(g, tmask, in_batch, layers, kUnlimitedFanout, 0)
    d_b = mark[vb.long()]
    owner = split_batch_share(vb, _dev_assign(sp, device), _dev_assign(gp, device), server, world)
    keep = d_b >= 0
    v_k, d_k, o_k = vb[keep].long(), d_b[keep].long(), owner[keep].long()
    mfg = [int((d_k <= layers - l).sum().item()) for l in range(layers + 1)]
    key = (o_k << 40) | (d_k << 32) | v_k
    key, _ = torch.sort(key)
    o_s = key >> 40
    d_s = (key >> 32) & 0xFF
    v_s = key & 0xFFFFFFFF
    counts = torch.bincount(o_s, minlength=world).cpu().numpy().astype(np.int64)
    block = int(max(1, counts.max())) if len(counts) else 1
    starts = np.concatenate([[0], np.cumsum(counts)])
    pos = torch.arange(len(key), device=device) - torch.from_numpy(starts[:-1]).to(device)[o_s]
    local_of = torch.full((max(n, 1),), -1, dtype=torch.int32, device=device)
    local_of[v_s] = (o_s * block + pos).to(torch.int32)
    a, b = int(starts[rank]), int(starts[rank + 1])
    l2g = v_s[a:b].to(torch.int32).contiguous()
    d_my = d_s[a:b].cpu().numpy()
    nloc = b - a
    rows_in = [int(np.sum(d_my <= layers - l)) for l in range(layers)]
    rows_out = [int(np.sum(d_my <= layers - l - 1)) for l in range(layers)]
    # this rank's rows: in-batch neighbours (d <= L) in padded ids
    cnt = torch.zeros(max(nloc, 1), dtype=torch.int64, device=device)
    call("gdx_local_csr", dg.row_ptr.data_ptr(), dg.col.data_ptr(), l2g.data_ptr(), nloc,
         local_of.data_ptr(), cnt.data_ptr(), None, None, stream_handle())
    lptr = torch.zeros(nloc + 1, dtype=torch.int64, device=device)
    total = _lib.u64(0)
    call("gdx_exclusive_scan_u64", cnt.data_ptr(), nloc, lptr.data_ptr(), _lib.C.byref(total),
         stream_handle())
    nnz = int(total.value)
    lcol = torch.empty(max(nnz, 1), dtype=torch.int32, device=device)
    call("gdx_local_csr", dg.row_ptr.data_ptr(), dg.col.data_ptr(), l2g.data_ptr(), nloc,
         local_of.data_ptr(), None, lptr.data_ptr(), lcol.data_ptr(), stream_handle())
    if sort_sources and nnz:
        # ascending padded ids per row, so the locally owned sources are one segment
        rid = torch.repeat_interleave(torch.arange(nloc, device=device), (lptr[1:] - lptr[:-1]))
        k2, _ = torch.sort((rid << 32) | lcol[:nnz].long())
        lcol[:nnz] = (k2 & 0xFFFFFFFF).to(torch.int32)
        del rid, k2
    csr = DeviceCSR(lptr, lcol, nloc)
    deg = (lptr[1:] - lptr[:-1]).double()
    inv_deg = torch.where(deg > 0, 1.0 / deg.clamp(min=1), torch.zeros_like(deg)).float()
    gcn_s = (1.0 / torch.sqrt(deg + 1.0)).float()
    seg_lo = seg_hi = None
    nnz_src = nnz
    if sort_sources:
        seg_lo = torch.empty(max(nloc, 1), dtype=torch.int64, device=device)
        seg_hi = torch.empty(max(nloc, 1), dtype=torch.int64, device=device)
        call("gdx_row_split", lptr.data_ptr(), lcol.data_ptr(), nloc, rank * block,
             rank * block + nloc, seg_lo.data_ptr(), seg_hi.data_ptr(), stream_handle())
        nnz_src = int((seg_hi - seg_lo)[:nloc].sum().item()) if nloc else 0
    src_bounds = src_nnz = None
    if sort_sources:
        src_bounds = source_bounds(lptr, lcol, nloc, block, world, device)
        src_nnz = [int((src_bounds[q + 1] - src_bounds[q])[:nloc].sum().item()) if nloc else 0
                   for q in range(world)]
    del local_of, in_batch, tmask, mark
    lp = lptr.cpu().numpy()
    edges = int(sum(lp[r] for r in rows_out) + sum(lp[r] for r in rows_in))
    return BatchGeometry(csr, l2g, nloc, block, rows_in, rows_out, rows_out[-1] if layers else nloc,
                         len(targets), nnz, nnz_src, inv_deg, gcn_s, seg_lo, seg_hi, mfg, edges,
                         src_bounds, src_nnz)


class CobatchTrainer(FullGraphTrainer):
    """Cooperative-batch trainer (one instance per rank/GPU of the server).

    plan: the server's BatchPlan; server_partition / gpu_partition as in the
    reference simulator (gpu ids of server s are s*gpus .. s*gpus+gpus-1)."""

    def __init__(self, g: Graph, cfg: ModelConfig, plan: BatchPlan, server_partition: Partition,
                 gpu_partition: Partition, server: int = 0, *, rank: int = 0, world: int = 1,
                 feature_seed: int = 1, label_seed: int = 2, weights=None, weight_seed: int = 3,
                 pg=None, device=None):
        require_cuda()
        if cfg.kind not in ("sage", "gcn", "sum"):
            raise InputError(f"unknown model kind {cfg.kind!r}")
        if cfg.classes > 256:
            raise InputError("classes must be <= 256")
        if plan.layers != cfg.layers:
            raise InputError(f"plan has {plan.layers} layers, model has {cfg.layers}")
        self.g, self.cfg, self.rank, self.world, self.pg = g, cfg, rank, world, pg
        self.d = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        d = self.d
        n = g.num_vertices()
        self.n, self.F = n, cfg.dims[0]
        F = self.F
        self.subgraph_mode = False
        self.is_cobatch = True
        self.plan = plan
        # the resident feature store (every vertex, split bf16) and labels: the
        # preloaded inputs each batch LOADs its rows from
        self.Xall = Split(n, F, d)
        chunk = max(1, min(n, (256 << 20) // (4 * max(F, 1))))
        tmp = dense(chunk, F, d)
        for r0 in range(0, n, chunk):
            r1 = min(n, r0 + chunk)
            call("gdx_init_uniform", feature_seed, FEAT_TAG, 0, r0 * F, r1 - r0, F, -0.5, 0.5,
                 tmp.data_ptr(), tmp.shape[1], stream_handle())
            call("gdx_split_bf16", tmp.data_ptr(), tmp.shape[1], r1 - r0, F,
                 self.Xall.hi.data_ptr() + 2 * r0 * self.Xall.ld,
                 self.Xall.lo.data_ptr() + 2 * r0 * self.Xall.ld, self.Xall.ld, 0, stream_handle())
        del tmp
        self.labels_all = torch.empty(max(n, 1), dtype=torch.int32, device=d)
        call("gdx_init_labels", label_seed, 0, n, cfg.classes, self.labels_all.data_ptr(),
             stream_handle())
        xmode = os.environ.get("GDX_EXCHANGE", "p2p")
        use_p2p = world > 1 and xmode in ("p2p", "p2p-epilogue")
        self.p2p_split = use_p2p and os.environ.get("GDX_P2P_SPLIT", "1") != "0"
        self.overlap = world > 1 and (
            self.p2p_split or (not use_p2p and os.environ.get("GDX_OVERLAP", "1") != "0"))
        spd, gpd = _dev_assign(server_partition, d), _dev_assign(gpu_partition, d)
        self.geoms = [batch_geometry(g, b.target_vertices, b.vertices, spd, gpd, server, rank,
                                     world, cfg.layers, d, self.overlap)
                      for b in plan.batches]
        del spd, gpd
        if world > 1 and os.environ.get("GDX_SPARSE_PUSH", "1") != "0":
            for geo in self.geoms:
                self._exchange_needs(geo)
        # buffers sized for the largest batch
        self.nloc = max([geo.nloc for geo in self.geoms] + [1])
        self.cap_rows = self.nloc
        self.nrows_gather = world * max([geo.block for geo in self.geoms] + [1])
        self.Xsp = Split(self.nloc, F, d)
        self.labels = torch.zeros(self.nloc, dtype=torch.int32, device=d)
        self._init_model(xmode, use_p2p, weights, weight_seed)
        # fused LOAD (GDX_FUSED_LOAD=1): measured slower on a papers-shape epoch (4.27 s vs
        # 4.17 s with the separate 6 TB/s gather pass; the gathered 128-byte half-rows cost
        # the two layer-0 GEMMs more than the pass), so off by default
        self._fused_load = (os.environ.get("GDX_FUSED_LOAD", "0") == "1"
                            and not getattr(self.layers[0], "agg_first", False))
        self.epoch_loss = torch.zeros(1, dtype=torch.float64, device=d)
        self.total_targets = sum(len(b.target_vertices) for b in plan.batches)
        self.current = None
        torch.cuda.synchronize(d)

    def _exchange_needs(self, geo: BatchGeometry):
        """Sparse-push row lists of one batch (see exchange_row_needs); kept only when
        they save at least 10% of the full-block push."""
        recv, off = exchange_row_needs(geo.csr.col[:geo.nnz], geo.block, self.rank, self.world, self.pg)
        if off[-1] <= 0.9 * (self.world - 1) * geo.nloc:
            geo.send_rows = (recv, off)

    def _peers(self, deltas, target: int):
        """No producer-side peer stores for cooperative batches: a producer writes only the
        batch's produced row prefix, while the peers must also see the zeroed rows past it
        (bind() clears them locally; a stale row from the previous batch would leak into the
        peers' aggregation), so every exchange is a push of the whole block."""
        return None

    def _refresh_input_splits(self):  # inputs arrive split (LOAD); nothing to refresh
        pass

    def bind(self, i: int):
        """Point the trainer at batch i and LOAD its input rows and labels."""
        geo = self.geoms[i]
        self.current = i
        self.csr = geo.csr
        self.nloc = geo.nloc
        self.lo = self.rank * geo.block
        self.hi = self.lo + geo.nloc
        self.nnz_local, self.nnz_local_src = geo.nnz, geo.nnz_src
        self.rows_in, self.rows_out = geo.rows_in, geo.rows_out
        self.loss_rows, self.loss_count = geo.loss_rows, float(geo.loss_count)
        self.inv_deg, self.gcn_s = geo.inv_deg, geo.gcn_s
        self.seg_lo, self.seg_hi = geo.seg_lo, geo.seg_hi
        self.src_bounds, self.src_nnz = geo.src_bounds, geo.src_nnz
        self.send_rows = geo.send_rows
        self.exchange = RowExchange(np.arange(self.world + 1, dtype=np.int64) * geo.block,
                                    self.rank, self.world, self.pg)
        # LOAD: input rows of this rank's block from the resident store (gdx_gather_split_rows),
        # or, with GDX_FUSED_LOAD=1, read by the layer-0 forward and dW GEMMs themselves
        # (TMA gather4 through geo.l2g)
        if self._fused_load and geo.nloc:
            self._xg = geo.l2g[:geo.nloc]
        else:
            self._xg = None
            call("gdx_gather_split_rows", self.Xall.hi.data_ptr(), self.Xall.lo.data_ptr(), self.Xall.ld,
                 geo.l2g.data_ptr(), geo.nloc, self.F, self.Xsp.hi.data_ptr(), self.Xsp.lo.data_ptr(),
                 self.Xsp.ld, stream_handle())
        if geo.nloc:   # labels of the batch rows: 4-byte rows moved bit for bit
            call("gdx_gather_rows", self.labels_all.data_ptr(), 1, geo.l2g.data_ptr(), geo.nloc, 1,
                 self.labels.data_ptr(), 1, stream_handle())
        # rows this batch does not produce must hold no gradient (buffers are reused
        # across batches): own gradient rows past each layer's produced prefix and, for
        # SAGE, the dP half of G on rows read but not produced (the dW GEMM's K covers
        # rows_in; the aggregation rewrites the other half there every step)
        s = stream_handle()

        def clear(t2d, r0, r1, cols=None):
            if r1 > r0:
                pitch = t2d.stride(0) * t2d.element_size()
                width = (t2d.shape[1] if cols is None else cols) * t2d.element_size()
                call("gdx_memset2d_async", t2d.data_ptr() + r0 * pitch, pitch, 0, width, r1 - r0, s)

        for l, L in enumerate(self.layers):
            r_out, r_in = geo.rows_out[l], geo.rows_in[l]
            if getattr(L, "agg_first", False):   # dA rows past the produced ones, dH_self
                clear(L.dAfull, self.lo + r_out, self.hi)
                clear(L.dself, r_out, r_in)
                continue
            clear(L.dfull, self.lo + r_out, self.hi)
            if self.cfg.kind == "sage":
                clear(L.G.hi.view(-1, L.G.ld), r_out, r_in, L.w)
                clear(L.G.lo.view(-1, L.G.ld), r_out, r_in, L.w)

    def train_batch(self, i: int):
        self.bind(i)
        FullGraphTrainer.train_epoch(self, sync_loss=False)
        self.epoch_loss += self.loss_acc

    def train_epoch(self, sync_loss: bool = True):
        """One pass over every batch of the plan (one SGD step per batch).  Returns the
        mean loss over all targets (host float) if sync_loss."""
        self.epoch_loss.zero_()
        for i in range(len(self.geoms)):
            self.train_batch(i)
        if sync_loss:
            return float(self.epoch_loss.item()) / max(self.total_targets, 1)
        return None

    def capture(self, warmup: int = 1):
        """One CUDA graph per batch (LOAD, clears, forward, loss, backward, exchanges, SGD:
        every step of the batch is a library kernel or a stream-ordered copy/memset with
        the batch's geometry baked in), sharing one memory pool."""
        for _ in range(warmup):
            self.train_epoch(sync_loss=False)
        torch.cuda.synchronize(self.d)
        self.graphs, pool = [], None
        for i in range(len(self.geoms)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=pool):
                self.train_batch(i)
            pool = g.pool()
            self.graphs.append(g)
        torch.cuda.synchronize(self.d)

    def replay_epoch(self, sync_loss: bool = False):
        """One epoch as R graph replays (capture() first)."""
        self.epoch_loss.zero_()
        for g in self.graphs:
            g.replay()
        if sync_loss:
            return float(self.epoch_loss.item()) / max(self.total_targets, 1)
        return None
