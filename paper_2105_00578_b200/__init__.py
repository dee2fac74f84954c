"""B200-native spectral graph partitioning (Sphynx / specpart hot path).

The product is the CUDA library libspecpart_b200.so (C ABI in
include/specpart_b200.h); this package is its host-side mirror of the
reference's C++ API (specpart::partition_graph and its seams).
"""
from . import abi
from .abi import (BreakdownError, DegenerateDegreeError, DimensionError, InfeasibleError, InvalidArgument,
                  SpecpartError, load_library)
from .api import (Context, EigenResult, Graph, Partition, RunConfig, RunReport, RunResult, default_context,
                  eigenvector_count, partition_graph, select_defaults, select_initial_vectors,
                  select_precond_auto)

__all__ = [
    "abi", "BreakdownError", "DegenerateDegreeError", "DimensionError", "InfeasibleError", "InvalidArgument",
    "SpecpartError", "load_library", "Context", "EigenResult", "Graph", "Partition", "RunConfig", "RunReport",
    "RunResult", "default_context", "eigenvector_count", "partition_graph", "select_defaults",
    "select_initial_vectors", "select_precond_auto",
]
