"""Graph and Partition host types -- the reference's API surface (graph.hpp,
partition.hpp) over the CSR layout the kernels consume.

``Graph`` keeps the reference's CSR exactly: ``row_offsets`` u64[V+1],
``col_indices`` u32[nnz], rows sorted ascending, deduplicated, no self loops,
undirected => symmetric (graph.hpp:11-60).  Generation and partitioning are
host preprocessing and run in libgdx's C++ (OpenMP), bit-identical to the
reference.  ``Graph.device()`` uploads the CSR once per device and caches it.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import InputError

VertexId = np.uint32


class Graph:
    def __init__(self, num_vertices: int, row_offsets: np.ndarray, col_indices: np.ndarray,
                 undirected: bool = True):
        self._n = int(num_vertices)
        self._ro = np.ascontiguousarray(row_offsets, np.uint64)
        self._ci = np.ascontiguousarray(col_indices, np.uint32)
        self._undirected = undirected
        self._dev = {}
        if self._ro.shape != (self._n + 1,):
            raise InputError("graph: row_offsets must have num_vertices + 1 entries")
        if int(self._ro[-1]) != len(self._ci):
            raise InputError("graph: row_offsets[-1] must equal len(col_indices)")

    # ---- reference accessors (graph.hpp:30-50) ----
    def num_vertices(self) -> int:
        return self._n

    def num_edges(self) -> int:
        return len(self._ci)

    def undirected(self) -> bool:
        return self._undirected

    def neighbors(self, v: int) -> np.ndarray:
        return self._ci[int(self._ro[v]):int(self._ro[v + 1])]

    def degree(self, v: int) -> int:
        return int(self._ro[v + 1] - self._ro[v])

    def row_offsets(self) -> np.ndarray:
        return self._ro

    def col_indices(self) -> np.ndarray:
        return self._ci

    def degrees(self) -> np.ndarray:
        return np.diff(self._ro).astype(np.int64)

    def __eq__(self, other) -> bool:
        return (isinstance(other, Graph) and self._n == other._n
                and np.array_equal(self._ro, other._ro) and np.array_equal(self._ci, other._ci))

    # ---- construction ----
    @staticmethod
    def from_edges(edges, num_vertices: int, undirected: bool = True) -> "Graph":
        """Graph::from_edges (graph.cpp:25-67): drops self loops, sorts and dedups rows."""
        if num_vertices == 0:
            raise InputError("graph must have at least one vertex")
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        if len(e) and (e.min() < 0 or e.max() >= num_vertices):
            bad = int(e.max())
            raise InputError(f"edge endpoint {bad} out of range for {num_vertices} vertices")
        e = e[e[:, 0] != e[:, 1]]
        src = e[:, 0] if not undirected else np.concatenate([e[:, 0], e[:, 1]])
        dst = e[:, 1] if not undirected else np.concatenate([e[:, 1], e[:, 0]])
        key = np.unique(src.astype(np.uint64) * np.uint64(num_vertices) + dst.astype(np.uint64))
        rows = (key // np.uint64(num_vertices)).astype(np.int64)
        cols = (key % np.uint64(num_vertices)).astype(np.uint32)
        ro = np.zeros(num_vertices + 1, np.uint64)
        np.add.at(ro, rows + 1, 1)
        return Graph(num_vertices, np.cumsum(ro, dtype=np.uint64), cols, undirected)

    def device(self, device=None):
        """Device CSR (cached per device)."""
        import torch

        from .device import DeviceCSR
        d = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        key = str(d)
        if key not in self._dev:
            self._dev[key] = DeviceCSR.upload(self._ro, self._ci, d)
        return self._dev[key]


def gen_random_graph(n: int, avg_degree: float, seed: int) -> Graph:
    """gen_random_graph (graph.cpp:137-154): undirected G(n, p), p = d/(n-1),
    per-vertex streams keyed (seed, u) -- generated in parallel by libgdx."""
    if n == 0:
        raise InputError("gen_random_graph: n must be >= 1")
    if avg_degree < 0.0:
        raise InputError("gen_random_graph: avg_degree must be >= 0")
    if avg_degree >= float(n):
        raise InputError(f"gen_random_graph: avg_degree {avg_degree:.6f} >= n, simple graph impossible")
    L = _lib.lib()
    ro = np.zeros(n + 1, np.uint64)
    nnz = int(L.gdx_host_gen_random_graph_count(n, float(avg_degree), int(seed), ro.ctypes.data))
    cols = np.empty(max(nnz, 1), np.uint32)
    _lib.call("gdx_host_gen_random_graph_fill", n, float(avg_degree), int(seed), ro.ctypes.data,
              cols.ctypes.data)
    return Graph(n, ro, cols[:nnz], True)


@dataclass
class Partition:
    """partition.hpp:15-23."""
    assignment: np.ndarray
    num_parts: int
    part_sizes: np.ndarray = field(default=None)

    def __post_init__(self):
        self.assignment = np.ascontiguousarray(self.assignment, np.uint32)
        if self.part_sizes is None:
            self.part_sizes = np.bincount(self.assignment, minlength=self.num_parts).astype(np.uint32)

    def part_of(self, v: int) -> int:
        return int(self.assignment[v])

    def members(self, part: int) -> np.ndarray:
        return np.nonzero(self.assignment == part)[0].astype(np.uint32)


def partition_random(g: Graph, parts: int, seed: int) -> Partition:
    """partition_random (partition.cpp:51-61), in libgdx host C++."""
    n = g.num_vertices()
    out = np.zeros(n, np.uint32)
    _lib.call("gdx_host_partition_random", n, parts, int(seed), out.ctypes.data)
    return Partition(out, parts)


def partition_contiguous(n: int, parts: int) -> Partition:
    """Contiguous row blocks (first n % parts blocks one larger) -- the full-graph
    row ownership used for multi-GPU training on structure-free graphs."""
    base, rem = divmod(n, parts)
    sizes = np.array([base + (1 if p < rem else 0) for p in range(parts)], np.int64)
    return Partition(np.repeat(np.arange(parts, dtype=np.uint32), sizes), parts)
