"""Cooperative batching on the device -- the reference's batch_plan.hpp API and
the simulator's split_batch (sim.cpp:81-102), re-exported.

batch_closure (batch_plan.cpp:28-70) is the same device hop loop as EAS with
the batch universe as the candidate mask; peel_mfg (:75-101) is a
level-synchronous device BFS; split_batch is a closed-form device kernel.
Target splitting (split_targets_mincut, :114-126) is host min-cut (C++).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call
from .device import require_cuda, stream_handle
from .errors import CapacityError, InputError
from .extract import DependencySubgraph, SamplingConfig, sampled_growth_device, _Work
from .graph import Graph, Partition

kBytesPerScalar = 4
kUnlimitedMemory = (1 << 64) - 1


@dataclass
class ModelSpec:
    """cost_model.hpp ModelSpec."""
    layers: int = 1
    hidden_dim: int = 64
    feature_dim: int = 64
    expansion_factor: float = 1.5


@dataclass
class Batch:
    """batch_plan.hpp:20-25."""
    target_vertices: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    vertices: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    mfg_vertices_per_layer: list = field(default_factory=list)
    est_memory_bytes: int = 0


@dataclass
class BatchPlan:
    worker_id: int = 0
    strategy: str = "fetch_then_split"
    layers: int = 0
    batches: list = field(default_factory=list)

    def batch_count(self) -> int:
        return len(self.batches)


def estimate_batch_memory(b: Batch, model: ModelSpec) -> int:
    """batch_plan.cpp:13-20."""
    total = 0
    for l, cnt in enumerate(b.mfg_vertices_per_layer):
        width = model.feature_dim if l == 0 else model.hidden_dim
        total += int(cnt) * width * kBytesPerScalar
    return total


def _mask(n: int, vertices, dev) -> torch.Tensor:
    m = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
    if len(vertices):
        m[torch.from_numpy(np.asarray(vertices, np.int64)).to(dev)] = 1
    return m


def batch_closure(g: Graph, universe: np.ndarray, targets: np.ndarray, cfg: SamplingConfig) -> np.ndarray:
    """Sampled closure of ``targets`` inside ``universe`` (u8 mask over all vertices)."""
    require_cuda()
    dev = g.device().row_ptr.device
    tmask = _mask(g.num_vertices(), targets, dev)
    allowed = torch.from_numpy(np.ascontiguousarray(universe, np.uint8)).to(dev)
    mark = sampled_growth_device(g, tmask, allowed, cfg.max_hop, cfg.fanout, cfg.seed)
    # ascending ids of the claimed vertices (compacted on the device)
    return torch.nonzero(mark != -1).flatten().to(torch.int32).cpu().numpy().view(np.uint32)


def peel_mfg(g: Graph, batch_vertices: np.ndarray, targets: np.ndarray, layers: int) -> list:
    require_cuda()
    dg = g.device()
    dev = dg.row_ptr.device
    n = g.num_vertices()
    in_batch = _mask(n, batch_vertices, dev)
    t = torch.from_numpy(np.ascontiguousarray(targets, np.uint32).view(np.int32)).to(dev)
    work = _Work.get(n, dev)
    counts = np.zeros(layers + 1, np.uint64)
    call("gdx_peel_mfg", dg.row_ptr.data_ptr(), dg.col.data_ptr(), n, in_batch.data_ptr(),
         t.data_ptr(), len(targets), layers, work.data_ptr(), counts.ctypes.data, stream_handle())
    return [int(c) for c in counts]


def make_batch(g: Graph, universe: np.ndarray, targets: np.ndarray, layers: int,
               cfg: SamplingConfig, model: ModelSpec) -> Batch:
    """batch_plan.cpp:103-112."""
    b = Batch(np.asarray(targets, np.uint32))
    b.vertices = batch_closure(g, universe, b.target_vertices, cfg)
    b.mfg_vertices_per_layer = peel_mfg(g, b.vertices, b.target_vertices, layers)
    b.est_memory_bytes = estimate_batch_memory(b, model)
    return b


def split_targets_mincut(g: Graph, targets: np.ndarray, r: int, seed: int) -> list:
    """batch_plan.cpp:114-126: min-cut split of the targets' induced subgraph (host C++)."""
    if r <= 1 or len(targets) <= 1:
        return [np.asarray(targets, np.uint32)]
    from .partition_host import induced_subgraph, partition_mincut
    sub, gids = induced_subgraph(g, targets)
    p = partition_mincut(sub, r, seed)
    return [np.sort(gids[p.assignment == k]).astype(np.uint32) for k in range(r)]


def split_targets_random(targets: np.ndarray, r: int, seed: int) -> list:
    """Scale variant of split_targets_mincut: partition_random (partition.cpp:51-61)
    of the targets' induced subgraph -- the assignment depends only on the target
    count, so the subgraph is never built.  For graphs whose host min-cut is too slow
    (papers shape: 111 M vertices) and structure-free graphs, where min-cut finds no
    locality anyway."""
    t = np.asarray(targets, np.uint32)
    if r <= 1 or len(t) <= 1:
        return [t]
    a = np.zeros(len(t), np.uint32)
    call("gdx_host_partition_random", len(t), r, int(seed), a.ctypes.data)
    return [t[a == k] for k in range(r)]


def _workspace_bytes(dev) -> int:
    """Device workspace for one gdx_cobatch_eval call (groups evaluated together)."""
    free, _ = torch.cuda.mem_get_info(dev)
    return int(max(1 << 26, min(free // 4, 32 << 30)))


def cobatch_eval(g: Graph, universe: torch.Tensor, groups: list, layers: int, cfg: SamplingConfig,
                 emit: bool = False):
    """Every group's batch closure + MFG counts in batched device launches
    (gdx_cobatch_eval; batch_plan.cpp:28-112 for all groups of one R).  Returns
    (sizes, mfg[groups][layers+1], vertex lists or None)."""
    dg = g.device()
    dev = dg.row_ptr.device
    n = g.num_vertices()
    G = len(groups)
    off = np.zeros(G + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in groups])
    flat = (np.concatenate([np.asarray(x, np.uint32) for x in groups]) if int(off[-1])
            else np.zeros(1, np.uint32))
    t = torch.from_numpy(flat.view(np.int32)).to(dev)
    sizes = np.zeros(G, np.uint64)
    mfg = np.zeros(G * (layers + 1), np.uint64)
    ws = _workspace_bytes(dev)
    args = (dg.row_ptr.data_ptr(), dg.col.data_ptr(), n, universe.data_ptr(), t.data_ptr(),
            off.ctypes.data, G, cfg.max_hop, cfg.fanout & 0xFFFFFFFF, cfg.seed, layers, ws,
            sizes.ctypes.data, mfg.ctypes.data)
    call("gdx_cobatch_eval", *args, None, None, stream_handle())
    verts = None
    if emit:
        voff = np.zeros(G + 1, np.uint64)
        voff[1:] = np.cumsum(sizes)
        out = torch.empty(max(int(voff[-1]), 1), dtype=torch.int32, device=dev)
        call("gdx_cobatch_eval", *args, out.data_ptr(), voff.ctypes.data, stream_handle())
        h = out.cpu().numpy().view(np.uint32)
        verts = [h[int(voff[i]):int(voff[i + 1])].copy() for i in range(G)]
    return sizes, mfg.reshape(G, layers + 1), verts


def _target_groups(sub: DependencySubgraph, g: Graph, r: int, cfg: SamplingConfig,
                   target_split: str) -> list:
    if target_split == "random":
        return split_targets_random(sub.inner_vertices, r, cfg.seed)
    if target_split == "mincut":
        return split_targets_mincut(g, sub.inner_vertices, r, cfg.seed)
    raise InputError(f"plan_cobatch: unknown target split {target_split!r}")


def _universe(sub: DependencySubgraph, g: Graph) -> torch.Tensor:
    dev = g.device().row_ptr.device
    m = _mask(g.num_vertices(), np.concatenate([sub.inner_vertices, sub.halo_vertices]), dev)
    return m


def _plan_from(sub, layers, groups, sizes, mfg, verts, model) -> BatchPlan:
    plan = BatchPlan(sub.server_id, "fetch_then_split", layers)
    for i, grp in enumerate(groups):
        b = Batch(np.asarray(grp, np.uint32), verts[i], [int(c) for c in mfg[i]])
        b.est_memory_bytes = estimate_batch_memory(b, model)
        plan.batches.append(b)
    return plan


def _build_cobatch(sub: DependencySubgraph, g: Graph, layers: int, cfg: SamplingConfig, r: int,
                   model: ModelSpec, target_split: str = "mincut") -> BatchPlan:
    groups = _target_groups(sub, g, r, cfg, target_split)
    sizes, mfg, verts = cobatch_eval(g, _universe(sub, g), groups, layers, cfg, emit=True)
    return _plan_from(sub, layers, groups, sizes, mfg, verts, model)


def plan_cobatch_fixed_r(sub: DependencySubgraph, g: Graph, layers: int, cfg: SamplingConfig,
                         r: int, model: ModelSpec, target_split: str = "mincut") -> BatchPlan:
    """batch_plan.cpp:146-153.  target_split="random" swaps the host min-cut target
    split for split_targets_random (papers-scale plans)."""
    if r == 0:
        raise InputError("plan_cobatch: batch count must be >= 1")
    require_cuda()
    capped = min(r, max(1, len(sub.inner_vertices)))
    return _build_cobatch(sub, g, layers, cfg, capped, model, target_split)


def _est_bytes(mfg_row, model: ModelSpec) -> int:
    return sum(int(c) * (model.feature_dim if l == 0 else model.hidden_dim) * kBytesPerScalar
               for l, c in enumerate(mfg_row))


def plan_cobatch(sub: DependencySubgraph, g: Graph, layers: int, cfg: SamplingConfig,
                 mem_budget: int, model: ModelSpec, target_split: str = "mincut") -> BatchPlan:
    """batch_plan.cpp:155-180: the smallest R whose batches all fit the budget, by the
    reference's linear scan (max batch memory is not monotone in R, :162-163).  Each R
    is one batched device evaluation of all its groups (no per-hop host syncs); only
    the winning R's vertex lists are materialised."""
    if mem_budget == 0:
        raise InputError("plan_cobatch: mem_budget must be > 0")
    require_cuda()
    universe = _universe(sub, g)
    max_r = max(1, len(sub.inner_vertices))
    for r in range(1, max_r + 1):
        groups = _target_groups(sub, g, r, cfg, target_split)
        sizes, mfg, _ = cobatch_eval(g, universe, groups, layers, cfg)
        est = [_est_bytes(row, model) for row in mfg]
        if max(est) <= mem_budget:
            sizes, mfg, verts = cobatch_eval(g, universe, groups, layers, cfg, emit=True)
            return _plan_from(sub, layers, groups, sizes, mfg, verts, model)
    w = int(np.argmax(est))
    first = int(groups[w][0]) if len(groups[w]) else 0
    raise CapacityError(f"single-target batch for vertex {first} needs {est[w]} "
                        f"bytes, budget is {mem_budget}")


def split_batch(batch_vertices: np.ndarray, server_partition: Partition, gpu_partition: Partition,
                server: int, gpus: int) -> list:
    """sim.cpp:81-102 on the device: inner vertices to their home GPU, halo vertices
    (ascending) to the least-loaded GPU (ties -> lowest).  Returns sorted shares."""
    require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    bv = np.ascontiguousarray(batch_vertices, np.uint32)
    nb = len(bv)
    if nb == 0:
        return [np.zeros(0, np.uint32) for _ in range(gpus)]
    tb = torch.from_numpy(bv.view(np.int32)).to(dev)
    sp = torch.from_numpy(server_partition.assignment.view(np.int32)).to(dev)
    gp = torch.from_numpy(gpu_partition.assignment.view(np.int32)).to(dev)
    share = torch.empty(nb, dtype=torch.int32, device=dev)
    work = torch.empty(5 * nb + 2 * gpus + 8, dtype=torch.int32, device=dev)
    call("gdx_split_batch", tb.data_ptr(), nb, sp.data_ptr(), gp.data_ptr(), server, gpus,
         share.data_ptr(), work.data_ptr(), stream_handle())
    s = share.cpu().numpy()
    return [bv[s == w] for w in range(gpus)]


def split_batch_owner(batch_vertices, server_partition, gpu_partition, server, gpus) -> np.ndarray:
    """Per-vertex local GPU of split_batch (same kernel, un-grouped)."""
    shares = split_batch(batch_vertices, server_partition, gpu_partition, server, gpus)
    bv = np.asarray(batch_vertices, np.uint32)
    out = np.zeros(len(bv), np.uint32)
    for w, s in enumerate(shares):
        out[np.searchsorted(bv, s)] = w
    return out
