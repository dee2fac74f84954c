"""ctypes mirror of include/specpart_b200.h.

The structs below are the C-ABI layout; keep them in lockstep with the header
(tests/test_abi.py checks every declared symbol and the struct sizes).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

SP_OK, SP_ERROR, SP_PARSE, SP_BREAKDOWN, SP_INFEASIBLE, SP_DEGENERATE, SP_DIMENSION, SP_INVALID, SP_CUDA, SP_NCCL = range(10)
PROBLEM = {"auto": 0, "combinatorial": 1, "generalized": 2, "normalized": 3}
PRECOND = {"auto": 0, "jacobi": 1, "polynomial": 2, "amg": 3, "none": 4}
INIT = {"auto": 0, "random": 1, "piecewise": 2}
LAP = {"combinatorial": 0, "normalized": 1, "degree": 2}
SP_MAX_EIG = 64
SP_MAX_AMG_LEVELS = 20
WARN_BREAKDOWN_RECOVERED, WARN_UNCONVERGED, WARN_IMBALANCE, WARN_AMG_STAGNATED = 1, 2, 4, 8


# ---- the reference's exception types (include/specpart/errors.hpp) ----------
class SpecpartError(RuntimeError):
    code = SP_ERROR


class ParseError(SpecpartError):
    code = SP_PARSE


class BreakdownError(SpecpartError):
    """errors.hpp:23-36 — basis lost rank even after the steepest-descent retry."""
    code = SP_BREAKDOWN

    @property
    def retried(self) -> bool:
        return "after retry" in str(self)


class InfeasibleError(SpecpartError):
    code = SP_INFEASIBLE


class DegenerateDegreeError(SpecpartError):
    code = SP_DEGENERATE


class DimensionError(SpecpartError):
    code = SP_DIMENSION


class InvalidArgument(SpecpartError, ValueError):
    code = SP_INVALID


class CudaError(SpecpartError):
    code = SP_CUDA


class NcclError(SpecpartError):
    code = SP_NCCL


_BY_CODE = {c.code: c for c in (SpecpartError, ParseError, BreakdownError, InfeasibleError,
                                DegenerateDegreeError, DimensionError, InvalidArgument, CudaError, NcclError)}


def raise_for(status: int, message: str) -> None:
    if status != SP_OK:
        raise _BY_CODE.get(status, SpecpartError)(message)


# ---- structs ----------------------------------------------------------------
class SpGraph(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_offsets", C.c_void_p), ("col_indices", C.c_void_p),
                ("values", C.c_void_p), ("vertex_weights", C.c_void_p)]


class SpConfig(C.Structure):
    _fields_ = [("num_parts", C.c_int64), ("problem", C.c_int32), ("precond", C.c_int32),
                ("tol", C.c_double), ("max_iters", C.c_int32), ("init", C.c_int32),
                ("seed", C.c_uint64), ("epsilon", C.c_double), ("doubled_cut", C.c_int32),
                ("record_trace", C.c_int32)]


class SpTraceRecord(C.Structure):
    _fields_ = [("iter", C.c_int32), ("ntheta", C.c_int32), ("min_residual", C.c_double),
                ("max_residual", C.c_double), ("theta", C.c_double * SP_MAX_EIG)]


class SpReport(C.Structure):
    _fields_ = [("n", C.c_int64), ("edges", C.c_int64), ("graph_regular", C.c_int32), ("pad0", C.c_int32),
                ("max_degree", C.c_int64), ("avg_degree", C.c_double), ("degree_ratio", C.c_double),
                ("num_parts", C.c_int64), ("problem", C.c_int32), ("precond", C.c_int32),
                ("tol", C.c_double), ("init", C.c_int32), ("eigenvectors", C.c_int32),
                ("seed", C.c_uint64), ("max_iters", C.c_int32), ("doubled_cut", C.c_int32),
                ("epsilon", C.c_double), ("iterations", C.c_int32), ("breakdown_retries", C.c_int32),
                ("theta", C.c_double * SP_MAX_EIG), ("residual_norms", C.c_double * SP_MAX_EIG),
                ("converged", C.c_uint8 * SP_MAX_EIG), ("poly_degree", C.c_int32), ("warnings", C.c_int32),
                ("laplacian_s", C.c_double), ("eigensolve_s", C.c_double), ("partition_s", C.c_double),
                ("total_s", C.c_double), ("cutsize", C.c_double), ("imbalance", C.c_double),
                ("spmm_launches", C.c_int64), ("spmm_bytes", C.c_double), ("spmm_ms", C.c_double),
                ("kernel_launches", C.c_int32), ("n_gpus", C.c_int32),
                ("poly_launches", C.c_int64), ("poly_bytes", C.c_double), ("poly_ms", C.c_double),
                ("halo_launches", C.c_int64), ("halo_bytes", C.c_double), ("halo_ms", C.c_double),
                ("spmm_eff_bytes", C.c_double), ("poly_eff_bytes", C.c_double),
                ("part_weights", C.POINTER(C.c_double)), ("trace", C.POINTER(SpTraceRecord)),
                ("trace_capacity", C.c_int32), ("trace_len", C.c_int32),
                ("eigenvectors_out", C.POINTER(C.c_double)),
                ("amg_levels", C.c_int32), ("pad1", C.c_int32),
                ("amg_n", C.c_int64 * SP_MAX_AMG_LEVELS), ("amg_nnz", C.c_int64 * SP_MAX_AMG_LEVELS),
                ("mesh_launches", C.c_int64)]


class SpGraphInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("n_symmetrized", C.c_int64),
                ("nnz_symmetrized", C.c_int64), ("max_degree", C.c_int64), ("avg_degree", C.c_double),
                ("degree_ratio", C.c_double), ("regular", C.c_int32), ("pad", C.c_int32)]


P = C.c_void_p
I32, I64, U64, F64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double

# name -> (restype, argtypes); the ref_* twins in oracle/_ref share these minus the context
SIGNATURES = {
    "sp_version": (C.c_int, []),
    "sp_context_create": (I32, [C.c_int, C.POINTER(P)]),
    "sp_nccl_unique_id": (I32, [P]),
    "sp_context_create_dist": (I32, [C.c_int, C.c_int, C.c_int, P, C.POINTER(P)]),
    "sp_context_destroy": (None, [P]),
    "sp_last_error": (C.c_char_p, [P]),
    "sp_debug_guard_check": (I32, [P, P]),
    "sp_context_set_timing": (I32, [P, C.c_int]),
    "sp_context_set_recurrence": (I32, [P, C.c_int]),
    "sp_context_set_relabel": (I32, [P, C.c_int]),
    "sp_partition": (I32, [P, C.POINTER(SpGraph), C.POINTER(SpConfig), P, C.POINTER(SpReport), P]),
    "sp_graph_upload": (I32, [P, C.POINTER(SpGraph), C.POINTER(P)]),
    "sp_graph_free": (None, [P]),
    "sp_partition_resident": (I32, [P, P, C.POINTER(SpConfig), P, C.POINTER(SpReport), P]),
    "sp_build_laplacian": (I32, [P, I32, C.POINTER(SpGraph), P, P, P, P, C.POINTER(F64), C.POINTER(I32)]),
    "sp_spmm": (I32, [P, I32, C.POINTER(SpGraph), P, I32, P]),
    "sp_spmm_solver": (I32, [P, I32, C.POINTER(SpGraph), P, I32, P]),
    "sp_spmm_csr": (I32, [P, I64, I64, P, P, P, P, I32, P]),
    "sp_gram": (I32, [P, I64, P, I32, P, I32, P, P]),
    "sp_block_combine": (I32, [P, I64, P, I32, P, I32, I32, P]),
    "sp_bench_blockop": (I32, [P, I64, I32, I32, I32, I32, I32, I32, C.POINTER(F64)]),
    "sp_initial_guess": (I32, [P, I32, I64, I32, U64, P]),
    "sp_initial_guess_rows": (I32, [P, I32, I64, I32, U64, I64, I64, P]),
    "sp_lobpcg": (I32, [P, C.POINTER(SpGraph), I32, I32, U64, I32, P, I32, F64, I32, I32, P, P, P, P,
                        C.POINTER(I32), C.POINTER(I32)]),
    "sp_poly_apply": (I32, [P, I32, C.POINTER(SpGraph), U64, I32, P, I32, P, P, C.POINTER(I32)]),
    "sp_precond_apply_csr": (I32, [P, I64, P, P, P, I32, U64, I32, P, I32, P, P, C.POINTER(I32)]),
    "sp_precond_apply": (I32, [P, I32, C.POINTER(SpGraph), I32, U64, I32, P, I32, P]),
    "sp_mj_partition": (I32, [P, I64, I32, P, P, I64, P, P, C.POINTER(F64)]),
    "sp_cutsize": (I32, [P, C.POINTER(SpGraph), P, I32, C.POINTER(F64)]),
    "sp_cut_imbalance": (I32, [P, C.POINTER(SpGraph), P, I64, I32, C.POINTER(F64), C.POINTER(F64), P]),
    "sp_ingest": (I32, [P, I64, P, P, I32, C.POINTER(P)]),
    "sp_device_graph_info": (I32, [P, P, C.POINTER(SpGraphInfo)]),
    "sp_device_graph_download": (I32, [P, P, P, P, P]),
    "sp_classify": (I32, [P, C.POINTER(SpGraph), C.POINTER(SpGraphInfo)]),
}

# SPECPART_B200_LIB: load another build of the library (A/B of two builds on one box)
LIB_PATH = Path(os.environ.get("SPECPART_B200_LIB") or Path(__file__).resolve().parent / "libspecpart_b200.so")
_lib = None


def load_library(path: Path | str | None = None) -> C.CDLL:
    """Loads the in-tree CUDA library. Fails loudly: there is no CPU fallback."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the B200 path has no CPU fallback)")
    lib = C.CDLL(str(p), mode=C.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("SPECPART_B200_LIB") and not hasattr(lib, name):
            continue  # an older build under A/B: entry points it predates stay unbound
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    if path is None:
        _lib = lib
    return lib
