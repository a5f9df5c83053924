"""g2: a B200-native (sm_100a) GOTHIC-style octree gravity step.

Drop-in for the gravitree hot path (Morton keys + radix sort, makeTree,
calcNode, walkTree, block-step predict/correct) behind the C-ABI in
include/g2/capi.h; ``gravitree`` is the Python mirror of the reference API.
"""
from .gravitree import (DataError, Diagnostics, EngineConfig, GravityEngine, GravParams, InternalError, ParticleSystem,
                        ResourceError, Simulation, SingularityError, StepResult, StepScheme, TraversalEvents,
                        TunerConfig, block_level, compute_diagnostics, count_walk_ops, direct_sum, flops_estimate,
                        force_error, read_snapshot, write_snapshot, Snapshot,
                        nccl_unique_id, predict, predict_speedup, walk_flops)

__all__ = ["DataError", "Diagnostics", "EngineConfig", "GravityEngine", "GravParams", "InternalError", "ParticleSystem",
           "ResourceError", "Simulation", "SingularityError", "StepResult", "StepScheme", "TraversalEvents",
           "TunerConfig", "block_level", "compute_diagnostics", "count_walk_ops", "direct_sum", "flops_estimate", "force_error",
           "nccl_unique_id", "predict", "predict_speedup", "walk_flops", "read_snapshot", "write_snapshot", "Snapshot"]
