"""Host partitioning (stays on the CPU): partition_mincut,
induced_subgraph and hierarchical_partition with the reference's semantics
(partition.cpp:63-259).  The min-cut itself runs in libgdx's C++."""
from __future__ import annotations

import numpy as np

from . import _lib
from .errors import InputError
from .graph import Graph, Partition, partition_random
from .rng import mix64

kDefaultBalanceEps = 0.05


def partition_mincut(g: Graph, parts: int, seed: int, epsilon: float = kDefaultBalanceEps) -> Partition:
    """partition.cpp:63-170, bit-identical (libgdx host C++)."""
    n = g.num_vertices()
    out = np.zeros(max(n, 1), np.uint32)
    _lib.call("gdx_host_partition_mincut", n, g.row_offsets().ctypes.data, g.col_indices().ctypes.data,
              parts, int(seed), float(epsilon), out.ctypes.data)
    return Partition(out[:n], parts)


def induced_subgraph(g: Graph, vertices_sorted) -> tuple[Graph, np.ndarray]:
    """partition.cpp:204-224: subgraph induced by a sorted vertex set, local ids in
    the order of the set; returns (graph, local -> global ids)."""
    gids = np.asarray(vertices_sorted, np.uint32)
    n = g.num_vertices()
    local = np.full(n, -1, np.int64)
    local[gids] = np.arange(len(gids))
    ro, ci = g.row_offsets(), g.col_indices()
    starts, ends = ro[gids].astype(np.int64), ro[gids + 1].astype(np.int64)
    lens = ends - starts
    idx = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + np.arange(lens.sum())
    nb = local[ci[idx]] if len(idx) else np.zeros(0, np.int64)
    row = np.repeat(np.arange(len(gids)), lens)
    keep = nb >= 0
    cnt = np.bincount(row[keep], minlength=len(gids))
    lro = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint64)
    # global rows are sorted and the map is monotone, so local rows stay sorted
    return Graph(len(gids), lro, nb[keep].astype(np.uint32)), gids


class HierarchicalPartition:
    def __init__(self, server: Partition, gpu: Partition, gpus_per_server: int):
        self.server, self.gpu, self.gpus_per_server = server, gpu, gpus_per_server


def hierarchical_partition(g: Graph, servers: int, gpus_per_server: int, mode: str, seed: int,
                           epsilon: float = kDefaultBalanceEps) -> HierarchicalPartition:
    """partition.cpp:226-259: server split, then per-server GPU split with seed
    mix64(seed ^ (s + 1))."""
    if servers == 0 or gpus_per_server == 0:
        raise InputError("hierarchical_partition: servers and gpus_per_server must be >= 1")
    if servers * gpus_per_server > g.num_vertices():
        raise InputError("hierarchical_partition: more workers than vertices")

    def run(graph, parts, s):
        return partition_random(graph, parts, s) if mode == "random" else partition_mincut(graph, parts, s, epsilon)

    sp = run(g, servers, seed)
    gpu = np.zeros(g.num_vertices(), np.uint32)
    for s in range(servers):
        sub, gids = induced_subgraph(g, sp.members(s))
        local = run(sub, gpus_per_server, mix64(seed ^ (s + 1)))
        gpu[gids] = s * gpus_per_server + local.assignment
    return HierarchicalPartition(sp, Partition(gpu, servers * gpus_per_server), gpus_per_server)
