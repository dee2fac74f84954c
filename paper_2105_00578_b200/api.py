"""Host-side mirror of the reference's C++ API (include/specpart/*.hpp) over the C-ABI.

Names, argument meaning and error behaviour follow the reference:
    partition_graph(Graph, RunConfig) -> RunResult       pipeline.hpp:106
    build_combinatorial / build_normalized / build_degree laplacian.hpp:24-33
    kernels.spmv_block / kernels.gram                    kernels.hpp:16-24
    initial_guess_random / initial_guess_piecewise       eigensolver.hpp:44-50
    lobpcg                                               eigensolver.hpp:61-64
    polynomial_build(...).apply                          preconditioners.hpp:45-46
    mj_partition                                         partitioner.hpp:39-42
    make_partition / cutsize / imbalance                 graph.hpp:63-75
    symmetrize / largest_connected_component / classify  graph.hpp:53-65
Every call runs the CUDA library (libspecpart_b200.so); a missing library raises
ImportError — there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import abi


# ---- data types -------------------------------------------------------------
@dataclass
class Graph:
    """Graph (graph.hpp:17-32): symmetric CSR adjacency, no self-loops.

    values=None means unit edge costs (SparseMatrix without values,
    sparse.hpp:29); vertex_weights=None means unit weights."""
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray | None = None
    vertex_weights: np.ndarray | None = None

    def __post_init__(self):
        self.row_offsets = np.ascontiguousarray(self.row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(self.col_indices, dtype=np.int32)
        if self.values is not None:
            self.values = np.ascontiguousarray(self.values, dtype=np.float64)
        if self.vertex_weights is not None:
            self.vertex_weights = np.ascontiguousarray(self.vertex_weights, dtype=np.float64)

    @property
    def n(self) -> int:
        return int(self.row_offsets.shape[0] - 1)

    def edge_count(self) -> int:
        return int(self.row_offsets[-1]) // 2

    def as_c(self) -> abi.SpGraph:
        g = abi.SpGraph()
        g.n = self.n
        g.row_offsets = self.row_offsets.ctypes.data
        g.col_indices = self.col_indices.ctypes.data
        g.values = self.values.ctypes.data if self.values is not None else None
        g.vertex_weights = self.vertex_weights.ctypes.data if self.vertex_weights is not None else None
        return g


@dataclass
class RunConfig:
    """RunConfig (pipeline.hpp:20-31). tol=None picks by graph kind."""
    num_parts: int = 2
    problem: str = "auto"
    precond: str = "auto"
    tol: float | None = None
    max_iters: int = 1000
    seed: int = 42
    epsilon: float = 0.01
    doubled_cut: bool = False
    init: str = "auto"
    record_trace: bool = False

    def as_c(self) -> abi.SpConfig:
        c = abi.SpConfig()
        c.num_parts = int(self.num_parts)
        c.problem = abi.PROBLEM[self.problem]
        c.precond = abi.PRECOND[self.precond]
        c.tol = float(self.tol) if self.tol is not None else -1.0
        c.max_iters = int(self.max_iters)
        c.init = abi.INIT[self.init]
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        c.epsilon = float(self.epsilon)
        c.doubled_cut = int(bool(self.doubled_cut))
        c.record_trace = int(bool(self.record_trace))
        return c


@dataclass
class GraphKind:
    """GraphKind (graph.hpp:35-41) plus the sizes sp_graph_info carries."""
    regular: bool
    max_degree: int
    avg_degree: float
    ratio: float
    n: int = 0
    nnz: int = 0
    n_symmetrized: int = 0
    nnz_symmetrized: int = 0

    @property
    def kind(self) -> str:
        return "regular" if self.regular else "irregular"


def _kind_from_c(i: abi.SpGraphInfo) -> GraphKind:
    return GraphKind(bool(i.regular), int(i.max_degree), float(i.avg_degree), float(i.degree_ratio),
                     int(i.n), int(i.nnz), int(i.n_symmetrized), int(i.nnz_symmetrized))


@dataclass
class Partition:
    assignment: np.ndarray
    num_parts: int
    part_weights: np.ndarray
    cutsize: float = 0.0
    imbalance: float = 0.0


@dataclass
class TraceRecord:
    iter: int
    min_residual: float
    max_residual: float
    theta: list


@dataclass
class RunReport:
    n: int = 0
    edges: int = 0
    regular: bool = True
    max_degree: int = 0
    avg_degree: float = 0.0
    degree_ratio: float = 0.0
    num_parts: int = 0
    problem: str = ""
    precond: str = ""
    tol: float = 0.0
    init: str = ""
    eigenvectors: int = 0
    seed: int = 0
    max_iters: int = 0
    epsilon: float = 0.0
    doubled_cut: bool = False
    iterations: int = 0
    breakdown_retries: int = 0
    theta: list = field(default_factory=list)
    residual_norms: list = field(default_factory=list)
    converged: list = field(default_factory=list)
    poly_degree: int = 0
    warnings: list = field(default_factory=list)
    times: dict = field(default_factory=dict)
    cutsize: float = 0.0
    imbalance: float = 0.0
    part_weights: list = field(default_factory=list)
    trace: list = field(default_factory=list)
    amg_levels: list = field(default_factory=list)  # [(n, nnz)] per level (pipeline.hpp:48-51)
    device: dict = field(default_factory=dict)


@dataclass
class RunResult:
    partition: Partition
    report: RunReport
    eigenvectors: np.ndarray | None = None  # n x d (EigenResult::X), when asked for


@dataclass
class EigenResult:
    theta: np.ndarray
    X: np.ndarray
    iterations: int
    residual_norms: np.ndarray
    converged: np.ndarray
    breakdown_retries: int

    def all_converged(self) -> bool:
        return bool(len(self.converged)) and bool(np.all(self.converged))


_NAMES_PROBLEM = {v: k for k, v in abi.PROBLEM.items()}
_NAMES_PRECOND = {v: k for k, v in abi.PRECOND.items()}
_NAMES_INIT = {v: k for k, v in abi.INIT.items()}


def report_from_c(r: abi.SpReport, part_weights: np.ndarray, trace_buf=None) -> RunReport:
    d = r.eigenvectors
    warnings = []
    if r.warnings & abi.WARN_BREAKDOWN_RECOVERED:
        warnings.append("eigensolver recovered from a basis breakdown by clearing the search directions")
    if r.warnings & abi.WARN_UNCONVERGED:
        warnings.append("eigensolver reached max_iters with unconverged columns; "
                        "partitioning on partially converged eigenvectors")
    if r.warnings & abi.WARN_AMG_STAGNATED:
        warnings.append("amg coarsening stagnated; hierarchy stopped early")
    if r.warnings & abi.WARN_IMBALANCE:
        warnings.append(f"imbalance {r.imbalance:.6f} exceeds 1+epsilon = {1.0 + r.epsilon:.6f}")
    trace = []
    if trace_buf is not None:
        for k in range(r.trace_len):
            t = trace_buf[k]
            trace.append(TraceRecord(t.iter, t.min_residual, t.max_residual, list(t.theta[: t.ntheta])))
    return RunReport(
        n=r.n, edges=r.edges, regular=bool(r.graph_regular), max_degree=r.max_degree,
        avg_degree=r.avg_degree, degree_ratio=r.degree_ratio, num_parts=r.num_parts,
        problem=_NAMES_PROBLEM.get(r.problem, "?"), precond=_NAMES_PRECOND.get(r.precond, "?"),
        tol=r.tol, init=_NAMES_INIT.get(r.init, "?"), eigenvectors=d, seed=r.seed,
        max_iters=r.max_iters, epsilon=r.epsilon, doubled_cut=bool(r.doubled_cut),
        iterations=r.iterations, breakdown_retries=r.breakdown_retries,
        theta=list(r.theta[:d]), residual_norms=list(r.residual_norms[:d]),
        converged=[bool(x) for x in r.converged[:d]], poly_degree=r.poly_degree, warnings=warnings,
        times={"laplacian_s": r.laplacian_s, "eigensolve_s": r.eigensolve_s,
               "partition_s": r.partition_s, "total_s": r.total_s},
        cutsize=r.cutsize, imbalance=r.imbalance, part_weights=list(part_weights), trace=trace,
        amg_levels=[(int(r.amg_n[i]), int(r.amg_nnz[i])) for i in range(r.amg_levels)],
        device={"mesh_launches": r.mesh_launches, "spmm_launches": r.spmm_launches, "spmm_bytes": r.spmm_bytes, "spmm_ms": r.spmm_ms,
                "kernel_launches": r.kernel_launches, "n_gpus": r.n_gpus,
                "poly_launches": r.poly_launches, "poly_bytes": r.poly_bytes, "poly_ms": r.poly_ms,
                "halo_launches": r.halo_launches, "halo_bytes": r.halo_bytes, "halo_ms": r.halo_ms,
                "spmm_eff_bytes": r.spmm_eff_bytes, "poly_eff_bytes": r.poly_eff_bytes})


def _ptr(a):
    return a.ctypes.data if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _colmajor(X):
    """(n, m) array -> column-major contiguous buffer (the reference Dense layout)."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    return np.asfortranarray(X)


def _check_x0(x0, n: int, cfg: RunConfig):
    """The C-ABI reads n*d doubles of x0 (d = eigenvector_count(K)): anything else is a
    DimensionError (errors.hpp:51-54), never an out-of-bounds host read."""
    if x0 is None:
        return None
    d = eigenvector_count(int(cfg.num_parts))
    X = np.asarray(x0, dtype=np.float64)
    if X.ndim != 2 or X.shape != (n, d):
        raise abi.DimensionError(f"partition_graph: x0 must have shape (n, d) = ({n}, {d}), got {X.shape}")
    return np.asfortranarray(X)


def _want_vectors(rep, n: int, cfg: RunConfig, on: bool):
    if not on:
        return None
    d = eigenvector_count(int(cfg.num_parts))
    ev = np.empty((n, d), dtype=np.float64, order="F")
    rep.eigenvectors_out = ev.ctypes.data_as(C.POINTER(C.c_double))
    return ev


# ---- context ------------------------------------------------------------------
class Context:
    """One B200 (one rank). world > 1 needs the same nccl_id on every rank."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        self.lib = abi.load_library()
        self._h = C.c_void_p()
        self._graphs = weakref.WeakSet()  # device graphs: released before the context
        if world > 1:
            buf = C.create_string_buffer(nccl_id, 128)
            st = self.lib.sp_context_create_dist(device, rank, world, buf, C.byref(self._h))
        else:
            st = self.lib.sp_context_create(device, C.byref(self._h))
        if st != abi.SP_OK:
            abi.raise_for(st, f"sp_context_create failed ({st}) on device {device}")
        self.device, self.rank, self.world = device, rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = abi.load_library()
        buf = C.create_string_buffer(128)
        abi.raise_for(lib.sp_nccl_unique_id(buf), "ncclGetUniqueId failed")
        return buf.raw

    def close(self):
        for dg in list(getattr(self, "_graphs", ())):
            dg.free()
        if self._h:
            self.lib.sp_context_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st != abi.SP_OK:
            abi.raise_for(st, self.lib.sp_last_error(self._h).decode(errors="replace"))

    def set_timing(self, on: bool):
        self._check(self.lib.sp_context_set_timing(self._h, int(on)))

    def set_relabel(self, on: bool):
        """Irregular graphs: degree-descending relabel inside the solver (on by default)."""
        self._check(self.lib.sp_context_set_relabel(self._h, int(on)))

    def set_recurrence(self, on: bool):
        """LOBPCG AX/AH/AP recurrence (one SpMM per iteration); off = the reference's algorithm."""
        self._check(self.lib.sp_context_set_recurrence(self._h, int(on)))

    # pipeline.cpp:47-167
    def partition_graph(self, g: Graph, cfg: RunConfig, x0=None, out=None,
                        return_eigenvectors: bool = False) -> RunResult:
        """out: optional caller-owned int32[n] array (e.g. pinned) receiving the assignment.
        x0: optional n x d initial block, d = eigenvector_count(K) (the CLI's --init-file)."""
        n = g.n
        if out is not None:
            if out.dtype != np.int32 or out.shape != (n,) or not out.flags.c_contiguous:
                raise ValueError("partition_graph: out must be a contiguous int32 array of length n")
            assignment = out
        else:
            assignment = np.empty(n, dtype=np.int32)
        pw = np.zeros(max(int(cfg.num_parts), 1), dtype=np.float64)
        rep = abi.SpReport()
        rep.part_weights = pw.ctypes.data_as(C.POINTER(C.c_double))
        trace_buf = None
        if cfg.record_trace:
            cap = int(cfg.max_iters) + 1
            trace_buf = (abi.SpTraceRecord * cap)()
            rep.trace = C.cast(trace_buf, C.POINTER(abi.SpTraceRecord))
            rep.trace_capacity = cap
        x0b = _check_x0(x0, n, cfg)
        ev = _want_vectors(rep, n, cfg, return_eigenvectors)
        gc, cc = g.as_c(), cfg.as_c()
        self._check(self.lib.sp_partition(self._h, C.byref(gc), C.byref(cc), assignment.ctypes.data,
                                          C.byref(rep), _ptr(x0b)))
        report = report_from_c(rep, pw, trace_buf)
        part = Partition(assignment, int(cfg.num_parts), pw, rep.cutsize, rep.imbalance)
        return RunResult(part, report, ev)

    def upload(self, g: Graph) -> "DeviceGraph":
        """Copies the graph arrays into HBM (sp_graph_upload)."""
        h = C.c_void_p()
        gc = g.as_c()
        self._check(self.lib.sp_graph_upload(self._h, C.byref(gc), C.byref(h)))
        dg = DeviceGraph(self, h, g.n)
        self._graphs.add(dg)
        return dg

    def partition_resident(self, dg: "DeviceGraph", cfg: RunConfig, copy_assignment: bool = True,
                           x0=None, return_eigenvectors: bool = False) -> RunResult:
        """partition_graph on an HBM-resident graph (sp_partition_resident)."""
        assignment = np.empty(dg.n, dtype=np.int32) if copy_assignment else None
        pw = np.zeros(max(int(cfg.num_parts), 1), dtype=np.float64)
        rep = abi.SpReport()
        rep.part_weights = pw.ctypes.data_as(C.POINTER(C.c_double))
        x0b = _check_x0(x0, dg.n, cfg)
        ev = _want_vectors(rep, dg.n, cfg, return_eigenvectors)
        cc = cfg.as_c()
        self._check(self.lib.sp_partition_resident(self._h, dg.handle, C.byref(cc), _ptr(assignment),
                                                   C.byref(rep), _ptr(x0b)))
        report = report_from_c(rep, pw, None)
        return RunResult(Partition(assignment, int(cfg.num_parts), pw, rep.cutsize, rep.imbalance), report, ev)

    # laplacian.cpp:53-144 (explicit CSR, bit-exact)
    def build_laplacian(self, kind: str, g: Graph):
        k = abi.LAP[kind]
        n, nnz = g.n, int(g.row_offsets[-1])
        nnz_l = n if k == 2 else nnz + n
        offs = np.empty(n + 1, dtype=np.int64)
        cols = np.empty(max(nnz_l, 1), dtype=np.int32)
        vals = np.empty(max(nnz_l, 1), dtype=np.float64)
        diag = np.empty(max(n, 1), dtype=np.float64)
        bound, isdiag = C.c_double(), C.c_int32()
        gc = g.as_c()
        self._check(self.lib.sp_build_laplacian(self._h, k, C.byref(gc), offs.ctypes.data, cols.ctypes.data,
                                                vals.ctypes.data, diag.ctypes.data, C.byref(bound),
                                                C.byref(isdiag)))
        return dict(row_offsets=offs, col_indices=cols[:nnz_l], values=vals[:nnz_l], diag=diag[:n],
                    spectral_bound=bound.value, is_diagonal=bool(isdiag.value))

    def spmm(self, kind: str, g: Graph, X) -> np.ndarray:
        Xc = _colmajor(X)
        n, m = Xc.shape
        Y = np.empty((n, m), dtype=np.float64, order="F")
        gc = g.as_c()
        self._check(self.lib.sp_spmm(self._h, abi.LAP[kind], C.byref(gc), Xc.ctypes.data, m, Y.ctypes.data))
        return Y

    def spmm_solver(self, kind: str, g: Graph, X) -> np.ndarray:
        """Y = L X through the eigensolver's own kernel dispatch (sp_spmm_solver)."""
        Xc = _colmajor(X)
        n, m = Xc.shape
        Y = np.empty((n, m), dtype=np.float64, order="F")
        gc = g.as_c()
        self._check(self.lib.sp_spmm_solver(self._h, abi.LAP[kind], C.byref(gc), Xc.ctypes.data, m,
                                            Y.ctypes.data))
        return Y

    def spmm_csr(self, row_offsets, col_indices, values, X, ncols=None) -> np.ndarray:
        offs = np.ascontiguousarray(row_offsets, dtype=np.int64)
        cols = np.ascontiguousarray(col_indices, dtype=np.int32)
        vals = _f64(values) if values is not None else None
        Xc = _colmajor(X)
        nrows = offs.shape[0] - 1
        ncols = Xc.shape[0] if ncols is None else ncols
        m = Xc.shape[1]
        Y = np.empty((nrows, m), dtype=np.float64, order="F")
        self._check(self.lib.sp_spmm_csr(self._h, nrows, ncols, offs.ctypes.data, cols.ctypes.data,
                                         _ptr(vals), Xc.ctypes.data, m, Y.ctypes.data))
        return Y

    def gram(self, U, V, b=None) -> np.ndarray:
        Uc, Vc = _colmajor(U), _colmajor(V)
        bb = _f64(b) if b is not None else None
        G = np.empty((Uc.shape[1], Vc.shape[1]), dtype=np.float64, order="F")
        self._check(self.lib.sp_gram(self._h, Uc.shape[0], Uc.ctypes.data, Uc.shape[1], Vc.ctypes.data,
                                     Vc.shape[1], _ptr(bb), G.ctypes.data))
        return G

    def mult(self, X, C, Y=None) -> np.ndarray:
        """kernels::mult (Y = X C) or, given Y, kernels::mult_sub (returns Y - X C)."""
        Xc, Cc = _colmajor(X), _colmajor(C)
        if Xc.shape[1] != Cc.shape[0]:
            raise abi.DimensionError("mult: inner dimension mismatch")
        out = np.empty((Xc.shape[0], Cc.shape[1]), dtype=np.float64, order="F")
        if Y is not None:
            out[...] = _colmajor(Y)
        self._check(self.lib.sp_block_combine(self._h, Xc.shape[0], Xc.ctypes.data, Xc.shape[1], Cc.ctypes.data,
                                              Cc.shape[1], 0 if Y is None else 1, out.ctypes.data))
        return out

    def initial_guess(self, init: str, n: int, d: int, seed: int = 0) -> np.ndarray:
        X = np.empty((n, d), dtype=np.float64, order="F")
        self._check(self.lib.sp_initial_guess(self._h, abi.INIT[init], n, d, seed, X.ctypes.data))
        return X

    def initial_guess_rows(self, init: str, n: int, d: int, seed: int, row0: int, nloc: int) -> np.ndarray:
        """Rows [row0, row0+nloc) of initial_guess(init, n, d, seed) (sp_initial_guess_rows)."""
        X = np.empty((nloc, d), dtype=np.float64, order="F")
        self._check(self.lib.sp_initial_guess_rows(self._h, abi.INIT[init], n, d, seed, row0, nloc, X.ctypes.data))
        return X

    def lobpcg(self, g: Graph, problem: str, precond: str, X0, tol: float, max_iters: int = 1000,
               locking: bool = True, poly_seed: int = 0, poly_degree: int = 25) -> EigenResult:
        X0c = _colmajor(X0)
        n, nev = X0c.shape
        theta = np.empty(nev)
        X = np.empty((n, nev), dtype=np.float64, order="F")
        res = np.empty(nev)
        conv = np.empty(nev, dtype=np.uint8)
        it, rt = C.c_int32(), C.c_int32()
        gc = g.as_c()
        self._check(self.lib.sp_lobpcg(self._h, C.byref(gc), abi.PROBLEM[problem], abi.PRECOND[precond],
                                       poly_seed, poly_degree, X0c.ctypes.data, nev, tol, max_iters,
                                       int(locking), theta.ctypes.data, X.ctypes.data, res.ctypes.data,
                                       conv.ctypes.data, C.byref(it), C.byref(rt)))
        return EigenResult(theta, X, it.value, res, conv.astype(bool), rt.value)

    def poly_apply(self, kind: str, g: Graph, seed: int, degree: int, R):
        Rc = _colmajor(R)
        n, m = Rc.shape
        H = np.empty((n, m), dtype=np.float64, order="F")
        roots = np.empty(max(degree, 1))
        ach = C.c_int32()
        gc = g.as_c()
        self._check(self.lib.sp_poly_apply(self._h, abi.LAP[kind], C.byref(gc), seed, degree, Rc.ctypes.data,
                                           m, H.ctypes.data, roots.ctypes.data, C.byref(ach)))
        return H, roots[: ach.value]

    def precond_apply_csr(self, row_offsets, col_indices, values, precond: str, R, seed: int = 0, degree: int = 25):
        """jacobi / polynomial / none built on an explicit CSR operator and applied to R
        (sp_precond_apply_csr). Returns (H, Leja-ordered roots) — roots empty unless polynomial."""
        offs = np.ascontiguousarray(row_offsets, dtype=np.int64)
        cols = np.ascontiguousarray(col_indices, dtype=np.int32)
        vals = _f64(values)
        Rc = _colmajor(R)
        n, m = Rc.shape
        H = np.empty((n, m), dtype=np.float64, order="F")
        roots = np.empty(max(degree, 25))
        ach = C.c_int32()
        self._check(self.lib.sp_precond_apply_csr(self._h, n, offs.ctypes.data, cols.ctypes.data, vals.ctypes.data,
                                                  abi.PRECOND[precond], seed, degree, Rc.ctypes.data, m,
                                                  H.ctypes.data, roots.ctypes.data, C.byref(ach)))
        return H, roots[: ach.value]

    def precond_apply(self, kind: str, g: Graph, precond: str, R, seed: int = 0, degree: int = 25):
        """H = M R (Preconditioner::apply) for precond in jacobi / polynomial / amg / none."""
        Rc = _colmajor(R)
        n, m = Rc.shape
        H = np.empty((n, m), dtype=np.float64, order="F")
        gc = g.as_c()
        self._check(self.lib.sp_precond_apply(self._h, abi.LAP[kind], C.byref(gc), abi.PRECOND[precond], seed, degree,
                                              Rc.ctypes.data, m, H.ctypes.data))
        return H

    def mj_partition(self, coords, weights, num_parts: int) -> Partition:
        Cc = _colmajor(coords)
        n, dims = Cc.shape
        w = _f64(weights) if weights is not None else None
        a = np.empty(n, dtype=np.int32)
        pw = np.empty(num_parts)
        imb = C.c_double()
        self._check(self.lib.sp_mj_partition(self._h, n, dims, Cc.ctypes.data, _ptr(w), num_parts,
                                             a.ctypes.data, pw.ctypes.data, C.byref(imb)))
        return Partition(a, num_parts, pw, 0.0, imb.value)

    def make_partition(self, g: Graph, assignment, num_parts: int, doubled_cut: bool = False) -> Partition:
        a = np.ascontiguousarray(assignment, dtype=np.int32)
        if a.shape[0] != g.n:
            raise abi.InvalidArgument("make_partition: assignment length mismatch")
        pw = np.empty(num_parts)
        cut, imb = C.c_double(), C.c_double()
        gc = g.as_c()
        self._check(self.lib.sp_cut_imbalance(self._h, C.byref(gc), a.ctypes.data, num_parts,
                                              int(doubled_cut), C.byref(cut), C.byref(imb), pw.ctypes.data))
        return Partition(a, num_parts, pw, cut.value, imb.value)


    # graph.cpp:44-182 on the device (ingest.cu)
    def ingest(self, row_offsets, col_indices, lcc: bool = True) -> "DeviceGraph":
        """symmetrize(A) and, with lcc, largest_connected_component of it, left in HBM
        (sp_ingest). A is the square pattern (row_offsets, col_indices); values are
        ignored as in the reference (graph.cpp:44-64)."""
        offs = np.ascontiguousarray(row_offsets, dtype=np.int64)
        cols = np.ascontiguousarray(col_indices, dtype=np.int32)
        h = C.c_void_p()
        self._check(self.lib.sp_ingest(self._h, offs.shape[0] - 1, offs.ctypes.data, cols.ctypes.data,
                                       int(lcc), C.byref(h)))
        dg = DeviceGraph(self, h, 0, ingested=True)
        self._graphs.add(dg)
        dg.n = dg.info().n
        return dg

    def symmetrize(self, row_offsets, col_indices) -> Graph:
        """symmetrize (graph.hpp:53, graph.cpp:44-64), values=None = unit costs."""
        dg = self.ingest(row_offsets, col_indices, lcc=False)
        try:
            return dg.download()[0]
        finally:
            dg.free()

    def largest_connected_component(self, g: Graph):
        """largest_connected_component (graph.hpp:62, graph.cpp:118-171) of a symmetric
        unit-cost graph: (Graph, old_ids)."""
        dg = self.ingest(g.row_offsets, g.col_indices, lcc=True)
        try:
            return dg.download()
        finally:
            dg.free()

    def classify(self, g: Graph) -> GraphKind:
        """classify (graph.hpp:65, graph.cpp:173-182)."""
        i = abi.SpGraphInfo()
        gc = g.as_c()
        self._check(self.lib.sp_classify(self._h, C.byref(gc), C.byref(i)))
        return _kind_from_c(i)


class DeviceGraph:
    def __init__(self, ctx: Context, handle: C.c_void_p, n: int, ingested: bool = False):
        self.ctx, self.handle, self.n, self.ingested = ctx, handle, n, ingested

    def info(self) -> GraphKind:
        """Sizes and classify (graph.cpp:173-182) on the device (sp_device_graph_info)."""
        i = abi.SpGraphInfo()
        self.ctx._check(self.ctx.lib.sp_device_graph_info(self.ctx._h, self.handle, C.byref(i)))
        return _kind_from_c(i)

    def download(self):
        """(Graph, old_ids) for an ingested graph, (Graph, None) otherwise."""
        i = self.info()
        offs = np.empty(i.n + 1, dtype=np.int64)
        cols = np.empty(max(i.nnz, 1), dtype=np.int32)
        old = np.empty(max(i.n, 1), dtype=np.int64) if self.ingested else None
        self.ctx._check(self.ctx.lib.sp_device_graph_download(self.ctx._h, self.handle, offs.ctypes.data,
                                                              cols.ctypes.data, _ptr(old)))
        return Graph(offs, cols[: i.nnz]), (old[: i.n] if old is not None else None)

    def free(self):
        if self.handle:
            self.ctx.lib.sp_graph_free(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


_default: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def partition_graph(g: Graph, cfg: RunConfig, device: int = 0, x0=None) -> RunResult:
    return default_context(device).partition_graph(g, cfg, x0)


# Reference-side pure helpers (no device work)
def eigenvector_count(num_parts: int) -> int:
    """partitioner.cpp:13-17: floor(log2 K) + 1."""
    if num_parts < 2:
        raise abi.InfeasibleError("eigenvector_count: K must be >= 2")
    return int(num_parts).bit_length()


def select_defaults(regular: bool, precond: str):
    """pipeline.cpp:20-37."""
    table = {
        ("jacobi", True): ("combinatorial", 1e-3), ("jacobi", False): ("generalized", 1e-2),
        ("none", True): ("combinatorial", 1e-3), ("none", False): ("generalized", 1e-2),
        ("polynomial", True): ("combinatorial", 1e-3), ("polynomial", False): ("normalized", 1e-2),
        ("amg", True): ("combinatorial", 1e-2), ("amg", False): ("generalized", 1e-2),
    }
    if (precond, regular) not in table:
        raise abi.InvalidArgument("select_defaults: preconditioner must be resolved")
    return table[(precond, regular)]


def select_precond_auto(regular: bool) -> str:
    return "amg" if regular else "polynomial"


def select_initial_vectors(regular: bool) -> str:
    return "random" if regular else "piecewise"
