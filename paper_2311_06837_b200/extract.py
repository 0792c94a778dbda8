"""Dependency-subgraph extraction on the GPU -- the reference's extract.hpp API.

``extract_full`` (extract.cpp:87-113) and ``extract_sampled`` (extract.cpp:135-182,
expansion-aware sampling) both run as the device hop loop ``gdx_sampled_growth``
(K4/K5); ``induced_edges`` is counted on device (extract.cpp:49-58).  Index
sets are bit-exact with the reference for every (graph, partition, config).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call
from .device import require_cuda, stream_handle
from .errors import InputError
from .graph import Graph, Partition

UNSEEN = 0xFFFFFFFF
kUnlimitedFanout = 0xFFFFFFFF


@dataclass
class SamplingConfig:
    """extract.hpp:15-21 (defaults m=1, k=15)."""
    max_hop: int = 1
    fanout: int = 15
    seed: int = 0

    def unlimited(self) -> bool:
        return self.fanout == kUnlimitedFanout


@dataclass
class DependencySubgraph:
    """extract.hpp:27-42."""
    server_id: int = 0
    inner_vertices: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    halo_vertices: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    halo_hops: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    induced_edges: int = 0
    hop_limit: int = 0
    sampled: bool = False

    def is_inner(self, v: int) -> bool:
        i = np.searchsorted(self.inner_vertices, v)
        return bool(i < len(self.inner_vertices) and self.inner_vertices[i] == v)

    def is_halo(self, v: int) -> bool:
        i = np.searchsorted(self.halo_vertices, v)
        return bool(i < len(self.halo_vertices) and self.halo_vertices[i] == v)

    def contains(self, v: int) -> bool:
        return self.is_inner(v) or self.is_halo(v)

    def hop_of(self, v: int) -> int:
        if self.is_inner(v):
            return 0
        i = np.searchsorted(self.halo_vertices, v)
        if i == len(self.halo_vertices) or self.halo_vertices[i] != v:
            raise InputError(f"hop_of: vertex {v} not in subgraph")
        return int(self.halo_hops[i])

    def all_vertices(self) -> np.ndarray:
        return np.union1d(self.inner_vertices, self.halo_vertices).astype(np.uint32)

    def hop_array(self, n: int) -> np.ndarray:
        """Per-vertex hop label (0 inner, h halo, UNSEEN outside)."""
        hop = np.full(n, UNSEEN, np.uint32)
        hop[self.inner_vertices] = 0
        hop[self.halo_vertices] = self.halo_hops
        return hop


def _check_server(g: Graph, p: Partition, server_id: int):
    if len(p.assignment) != g.num_vertices():
        raise InputError("extract: partition size does not match graph")
    if server_id >= p.num_parts:
        raise InputError(f"extract: server id {server_id} out of range ({p.num_parts} parts)")


class _Work:
    """Per-device scratch for the hop loop (grown on demand)."""
    _cache: dict = {}

    @classmethod
    def get(cls, n: int, device) -> torch.Tensor:
        key = str(device)
        t = cls._cache.get(key)
        if t is None or t.numel() < 3 * n + 64:
            t = torch.empty(3 * n + 64, dtype=torch.int32, device=device)
            cls._cache[key] = t
        return t


def sampled_growth_device(g: Graph, excluded: torch.Tensor, allowed, max_hop: int, fanout: int,
                          seed: int) -> torch.Tensor:
    """Runs the device hop loop; returns the int32 mark tensor (UNSEEN = -1)."""
    dg = g.device()
    dev = dg.row_ptr.device
    n = g.num_vertices()
    mark = torch.where(excluded.bool(), torch.zeros((), dtype=torch.int32, device=dev),
                       torch.full((), -1, dtype=torch.int32, device=dev)).contiguous()
    work = _Work.get(n, dev)
    call("gdx_sampled_growth", dg.row_ptr.data_ptr(), dg.col.data_ptr(), n, excluded.data_ptr(),
         None if allowed is None else allowed.data_ptr(), max_hop, fanout & 0xFFFFFFFF, seed,
         mark.data_ptr(), work.data_ptr(), stream_handle())
    return mark


def induced_count_device(g: Graph, mark: torch.Tensor) -> int:
    dg = g.device()
    work = _Work.get(g.num_vertices(), dg.row_ptr.device)
    out = _lib.u64(0)
    call("gdx_induced_count", dg.row_ptr.data_ptr(), dg.col.data_ptr(), g.num_vertices(),
         mark.data_ptr(), work.data_ptr(), _lib.C.byref(out), stream_handle())
    return int(out.value)


def _finish(g: Graph, server_id: int, mark: torch.Tensor, hop_limit: int, sampled: bool) -> DependencySubgraph:
    hop = mark.cpu().numpy().view(np.uint32)
    inner = np.nonzero(hop == 0)[0].astype(np.uint32)
    halo = np.nonzero((hop != 0) & (hop != UNSEEN))[0].astype(np.uint32)
    return DependencySubgraph(server_id, inner, halo, hop[halo].copy(), induced_count_device(g, mark),
                              hop_limit, sampled)


def _inner_mask(g: Graph, p: Partition, server_id: int) -> torch.Tensor:
    dev = g.device().row_ptr.device
    a = torch.from_numpy(p.assignment.view(np.int32)).to(dev)
    return (a == server_id).to(torch.uint8).contiguous()


def extract_full(g: Graph, server_partition: Partition, server_id: int, layers: int) -> DependencySubgraph:
    """Full L-hop closure (extract.cpp:87-113): unlimited-fanout growth == BFS distances."""
    require_cuda()
    _check_server(g, server_partition, server_id)
    inner = _inner_mask(g, server_partition, server_id)
    mark = sampled_growth_device(g, inner, None, layers, kUnlimitedFanout, 0)
    return _finish(g, server_id, mark, layers, False)


@dataclass
class SampleTraceStep:
    """extract.hpp:49-53."""
    frontier_vertex: int
    hop: int
    taken: list


def sample_trace(g: Graph, inner_mask: np.ndarray, cfg: SamplingConfig) -> list:
    """The reference's SampleTrace (which frontier vertex took which halo vertex, in the
    sequential order of extract.cpp:158-178), from the host attribution replay
    (gdx_host_sample_trace)."""
    ro, ci = g.row_offsets(), g.col_indices()
    im = np.ascontiguousarray(inner_mask, np.uint8)
    ns, nt = _lib.u64(0), _lib.u64(0)
    args = (g.num_vertices(), ro.ctypes.data, ci.ctypes.data if len(ci) else None, im.ctypes.data, cfg.max_hop,
            cfg.fanout & 0xFFFFFFFF, cfg.seed)
    call("gdx_host_sample_trace", *args, 0, 0, _lib.C.byref(ns), _lib.C.byref(nt), None, None, None, None)
    S, T = int(ns.value), int(nt.value)
    sv = np.zeros(max(S, 1), np.uint32)
    sh = np.zeros(max(S, 1), np.uint32)
    so = np.zeros(S + 1, np.uint64)
    tk = np.zeros(max(T, 1), np.uint32)
    call("gdx_host_sample_trace", *args, S, T, _lib.C.byref(ns), _lib.C.byref(nt), sv.ctypes.data, sh.ctypes.data,
         so.ctypes.data, tk.ctypes.data)
    return [SampleTraceStep(int(sv[i]), int(sh[i]), [int(x) for x in tk[int(so[i]):int(so[i + 1])]])
            for i in range(S)]


def extract_sampled(g: Graph, server_partition: Partition, server_id: int, cfg: SamplingConfig,
                    trace=None) -> DependencySubgraph:
    """Expansion-aware sampling (extract.cpp:135-182), bit-exact on device.  ``trace``: a
    list that receives the SampleTrace steps (extract.hpp:49-64) -- the order-dependent
    attribution, replayed on the host."""
    require_cuda()
    _check_server(g, server_partition, server_id)
    inner = _inner_mask(g, server_partition, server_id)
    mark = sampled_growth_device(g, inner, None, cfg.max_hop, cfg.fanout, cfg.seed)
    sub = _finish(g, server_id, mark, cfg.max_hop, not cfg.unlimited())
    if trace is not None:
        trace.extend(sample_trace(g, inner.cpu().numpy(), cfg))
    return sub


def neighbor_explosion_profile(g: Graph, server_partition: Partition, server_id: int,
                               max_layers: int):
    """extract.cpp:184-202: closure sizes for hop limits 1..max_layers (one BFS)."""
    if max_layers == 0:
        raise InputError("neighbor_explosion_profile: max_layers must be >= 1")
    _check_server(g, server_partition, server_id)
    deep = extract_full(g, server_partition, server_id, max_layers)
    added = np.bincount(deep.halo_hops, minlength=max_layers + 1) if len(deep.halo_hops) else \
        np.zeros(max_layers + 1, np.int64)
    size = len(deep.inner_vertices)
    out = []
    for layer in range(1, max_layers + 1):
        size += int(added[layer])
        out.append((layer, size))
    return out
