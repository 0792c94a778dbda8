"""B200-native GraNNDis hot path (arXiv 2311.06837).

Drop-in for the reference's per-layer hot path: the graph /
partition / layer API of /root/reference/proj/include re-implemented over
hand-written sm_100a kernels in ``libgdx.so`` (C ABI: include/gdx.h).

    from paper_2311_06837_b200 import gen_random_graph, partition_random, \
        make_features, make_layer_weights, forward_full, extract_sampled, SamplingConfig

There is no CPU fallback: every compute entry point runs a libgdx kernel and
raises InternalError when the library or the GPU is missing.
"""
from .errors import (CapacityError, ContractError, GranndisError, InputError, InternalError,
                     ParseError)
from .graph import Graph, Partition, gen_random_graph, partition_contiguous, partition_random
from .extract import (DependencySubgraph, SamplingConfig, extract_full, extract_sampled,
                      kUnlimitedFanout, neighbor_explosion_profile)
from .gnn import (EquivalenceReport, equivalence_check, forward_full, forward_server_local,
                  make_features, make_layer_weights)
from .batch_plan import (Batch, BatchPlan, ModelSpec, batch_closure, estimate_batch_memory,
                         make_batch, peel_mfg, plan_cobatch, plan_cobatch_fixed_r, split_batch)
from .rng import KeyedRng, mix64

__all__ = [
    "CapacityError", "ContractError", "GranndisError", "InputError", "InternalError", "ParseError",
    "Graph", "Partition", "gen_random_graph", "partition_contiguous", "partition_random",
    "DependencySubgraph", "SamplingConfig", "extract_full", "extract_sampled", "kUnlimitedFanout",
    "neighbor_explosion_profile", "EquivalenceReport", "equivalence_check", "forward_full",
    "forward_server_local", "make_features", "make_layer_weights", "Batch", "BatchPlan",
    "ModelSpec", "batch_closure", "estimate_batch_memory", "make_batch", "peel_mfg",
    "plan_cobatch", "plan_cobatch_fixed_r", "split_batch", "KeyedRng", "mix64",
]
