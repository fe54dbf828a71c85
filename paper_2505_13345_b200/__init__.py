"""B200-native Occult expert-parallel MoE layer (arXiv 2505.13345).

Drop-in for the reference's C++ API surface (moesim): router config,
expert-placement table, dispatch/compute/combine entry points, pruning knob.
The compute path is hand-written sm_100a CUDA behind the C-ABI in
include/occult.h (libocc.so); this package is the host-side mirror.
"""
from .api import (  # noqa: F401
    CapacityError, CommReport, ConfigError, DataError, DeviceError, ExpertParallelLayer, MoEConfig, MoesimError, Placement,
    PlacementError, PruneSpec, RoutingError, ShapeError, StateError, UsageError, accumulate_collab,
    build_collab_graph, build_similarity_table, collaboration_aware_placement, exchange_layout,
    gate_logits_f64, gate_scores_f64, launch_count, lib, normalize_graph, reschedule_placement, round_robin_sources,
    topk_route, trivial_placement,
)
