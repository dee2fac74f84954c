"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracles.

  oracle/_ref/libspecpart_ref.so     the unmodified reference (/root/reference/proj/src)
                                     compiled by oracle/Makefile (see ref_driver.cpp)
  oracle/_ref/libspecpart_oracle.so  the repo's own plain-C restatement (specpart_oracle.c)

Both export ref_* functions with the argument lists of the sp_* C-ABI minus the
context, so tests call the CUDA path and the oracle identically. Only tests/,
__graft_entry__.smoke() and bench.py (reference / cpu_baseline legs) may use this.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2105_00578_b200 import abi
from paper_2105_00578_b200.api import (EigenResult, Graph, Partition, RunConfig, RunResult, _colmajor, _f64,
                                       _ptr, report_from_c)

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libspecpart_ref.so"
PORT_LIB = HERE / "_ref" / "libspecpart_oracle.so"

P, I32, I64, U64, F64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
_SIG = {
    "ref_last_error": (C.c_char_p, []),
    "ref_partition": (I32, [C.POINTER(abi.SpGraph), C.POINTER(abi.SpConfig), P, C.POINTER(abi.SpReport), P]),
    "ref_build_laplacian": (I32, [I32, C.POINTER(abi.SpGraph), P, P, P, P, C.POINTER(F64), C.POINTER(I32)]),
    "ref_spmm": (I32, [I32, C.POINTER(abi.SpGraph), P, I32, P]),
    "ref_spmm_csr": (I32, [I64, I64, P, P, P, P, I32, P]),
    "ref_gram": (I32, [I64, P, I32, P, I32, P, P]),
    "ref_mult": (I32, [I64, P, I32, P, I32, I32, P]),
    "ref_initial_guess": (I32, [I32, I64, I32, U64, P]),
    "ref_lobpcg": (I32, [C.POINTER(abi.SpGraph), I32, I32, U64, I32, P, I32, F64, I32, I32, P, P, P, P,
                         C.POINTER(I32), C.POINTER(I32)]),
    "ref_poly_apply": (I32, [I32, C.POINTER(abi.SpGraph), U64, I32, P, I32, P, P, C.POINTER(I32)]),
    "ref_poly_apply_csr": (I32, [I64, P, P, P, U64, I32, P, I32, P, C.POINTER(I32)]),
    "ref_precond_apply": (I32, [I32, C.POINTER(abi.SpGraph), I32, U64, I32, P, I32, P]),
    "ref_mj_partition": (I32, [I64, I32, P, P, I64, P, P, C.POINTER(F64)]),
    "ref_cut_imbalance": (I32, [C.POINTER(abi.SpGraph), P, I64, I32, C.POINTER(F64), C.POINTER(F64), P]),
    "ref_sym_eig": (I32, [I32, P, P, P]),
    "ref_generate": (I32, [C.c_char_p, C.POINTER(I64), C.POINTER(I64), P, P]),
    "ref_symmetrize_lcc": (I32, [I64, P, P, C.POINTER(I64), C.POINTER(I64), P, P, P]),
}


class RefLib:
    """The CPU oracle with the same method names as paper_2105_00578_b200.Context."""

    def __init__(self, path: Path | str | None = None):
        p = Path(path) if path else (REF_LIB if REF_LIB.exists() else PORT_LIB)
        if not p.exists():
            raise FileNotFoundError(f"oracle library {p} not built (run `make -C oracle`)")
        self.path = p
        self.kind = "reference" if p.name == REF_LIB.name else "port"
        self.lib = C.CDLL(str(p))
        for name, (res, args) in _SIG.items():
            f = getattr(self.lib, name, None)
            if f is None:
                continue
            f.restype, f.argtypes = res, args

    def has(self, name: str) -> bool:
        return getattr(self.lib, name, None) is not None

    def _check(self, st):
        if st != abi.SP_OK:
            abi.raise_for(st, self.lib.ref_last_error().decode(errors="replace"))

    def partition_graph(self, g: Graph, cfg: RunConfig) -> RunResult:
        a = np.empty(g.n, dtype=np.int32)
        pw = np.zeros(max(cfg.num_parts, 1))
        rep = abi.SpReport()
        rep.part_weights = pw.ctypes.data_as(C.POINTER(C.c_double))
        trace_buf = None
        if cfg.record_trace:
            cap = cfg.max_iters + 1
            trace_buf = (abi.SpTraceRecord * cap)()
            rep.trace = C.cast(trace_buf, C.POINTER(abi.SpTraceRecord))
            rep.trace_capacity = cap
        gc, cc = g.as_c(), cfg.as_c()
        self._check(self.lib.ref_partition(C.byref(gc), C.byref(cc), a.ctypes.data, C.byref(rep), None))
        r = report_from_c(rep, pw, trace_buf)
        return RunResult(Partition(a, cfg.num_parts, pw, rep.cutsize, rep.imbalance), r)

    def build_laplacian(self, kind: str, g: Graph):
        k = abi.LAP[kind]
        n, nnz = g.n, int(g.row_offsets[-1])
        nnz_l = n if k == 2 else nnz + n
        offs = np.empty(n + 1, dtype=np.int64)
        cols = np.empty(max(nnz_l, 1), dtype=np.int32)
        vals = np.empty(max(nnz_l, 1))
        diag = np.empty(max(n, 1))
        bound, isdiag = C.c_double(), C.c_int32()
        gc = g.as_c()
        self._check(self.lib.ref_build_laplacian(k, C.byref(gc), offs.ctypes.data, cols.ctypes.data,
                                                 vals.ctypes.data, diag.ctypes.data, C.byref(bound),
                                                 C.byref(isdiag)))
        return dict(row_offsets=offs, col_indices=cols[:nnz_l], values=vals[:nnz_l], diag=diag[:n],
                    spectral_bound=bound.value, is_diagonal=bool(isdiag.value))

    def spmm(self, kind: str, g: Graph, X):
        Xc = _colmajor(X)
        Y = np.empty(Xc.shape, order="F")
        gc = g.as_c()
        self._check(self.lib.ref_spmm(abi.LAP[kind], C.byref(gc), Xc.ctypes.data, Xc.shape[1], Y.ctypes.data))
        return Y

    def spmm_csr(self, row_offsets, col_indices, values, X, ncols=None):
        offs = np.ascontiguousarray(row_offsets, dtype=np.int64)
        cols = np.ascontiguousarray(col_indices, dtype=np.int32)
        vals = _f64(values) if values is not None else None
        Xc = _colmajor(X)
        nrows = offs.shape[0] - 1
        Y = np.empty((nrows, Xc.shape[1]), order="F")
        self._check(self.lib.ref_spmm_csr(nrows, Xc.shape[0] if ncols is None else ncols, offs.ctypes.data,
                                          cols.ctypes.data, _ptr(vals), Xc.ctypes.data, Xc.shape[1],
                                          Y.ctypes.data))
        return Y

    def gram(self, U, V, b=None):
        Uc, Vc = _colmajor(U), _colmajor(V)
        bb = _f64(b) if b is not None else None
        G = np.empty((Uc.shape[1], Vc.shape[1]), order="F")
        self._check(self.lib.ref_gram(Uc.shape[0], Uc.ctypes.data, Uc.shape[1], Vc.ctypes.data, Vc.shape[1],
                                      _ptr(bb), G.ctypes.data))
        return G

    def mult(self, X, C, Y=None):
        Xc, Cc = _colmajor(X), _colmajor(C)
        out = np.empty((Xc.shape[0], Cc.shape[1]), order="F")
        if Y is not None:
            out[...] = _colmajor(Y)
        self._check(self.lib.ref_mult(Xc.shape[0], Xc.ctypes.data, Xc.shape[1], Cc.ctypes.data, Cc.shape[1],
                                      0 if Y is None else 1, out.ctypes.data))
        return out

    def initial_guess(self, init: str, n: int, d: int, seed: int = 0):
        X = np.empty((n, d), order="F")
        self._check(self.lib.ref_initial_guess(abi.INIT[init], n, d, seed, X.ctypes.data))
        return X

    def lobpcg(self, g: Graph, problem: str, precond: str, X0, tol: float, max_iters: int = 1000,
               locking: bool = True, poly_seed: int = 0, poly_degree: int = 25) -> EigenResult:
        X0c = _colmajor(X0)
        n, nev = X0c.shape
        theta, res = np.empty(nev), np.empty(nev)
        X = np.empty((n, nev), order="F")
        conv = np.empty(nev, dtype=np.uint8)
        it, rt = C.c_int32(), C.c_int32()
        gc = g.as_c()
        self._check(self.lib.ref_lobpcg(C.byref(gc), abi.PROBLEM[problem], abi.PRECOND[precond], poly_seed,
                                        poly_degree, X0c.ctypes.data, nev, tol, max_iters, int(locking),
                                        theta.ctypes.data, X.ctypes.data, res.ctypes.data, conv.ctypes.data,
                                        C.byref(it), C.byref(rt)))
        return EigenResult(theta, X, it.value, res, conv.astype(bool), rt.value)

    def poly_apply(self, kind: str, g: Graph, seed: int, degree: int, R):
        Rc = _colmajor(R)
        H = np.empty(Rc.shape, order="F")
        ach = C.c_int32()
        gc = g.as_c()
        self._check(self.lib.ref_poly_apply(abi.LAP[kind], C.byref(gc), seed, degree, Rc.ctypes.data,
                                            Rc.shape[1], H.ctypes.data, None, C.byref(ach)))
        return H, ach.value

    def poly_apply_csr(self, row_offsets, col_indices, values, seed, degree, R):
        offs = np.ascontiguousarray(row_offsets, dtype=np.int64)
        cols = np.ascontiguousarray(col_indices, dtype=np.int32)
        vals = _f64(values)
        Rc = _colmajor(R)
        H = np.empty(Rc.shape, order="F")
        ach = C.c_int32()
        self._check(self.lib.ref_poly_apply_csr(offs.shape[0] - 1, offs.ctypes.data, cols.ctypes.data,
                                                vals.ctypes.data, seed, degree, Rc.ctypes.data, Rc.shape[1],
                                                H.ctypes.data, C.byref(ach)))
        return H, ach.value

    def precond_apply(self, kind: str, g: Graph, precond: str, R, seed: int = 0, degree: int = 25):
        Rc = _colmajor(R)
        n, m = Rc.shape
        H = np.empty((n, m), order="F")
        gc = g.as_c()
        self._check(self.lib.ref_precond_apply(abi.LAP[kind], C.byref(gc), abi.PRECOND[precond], seed, degree,
                                               Rc.ctypes.data, m, H.ctypes.data))
        return H

    def mj_partition(self, coords, weights, num_parts: int) -> Partition:
        Cc = _colmajor(coords)
        n, dims = Cc.shape
        w = _f64(weights) if weights is not None else None
        a = np.empty(n, dtype=np.int32)
        pw = np.empty(num_parts)
        imb = C.c_double()
        self._check(self.lib.ref_mj_partition(n, dims, Cc.ctypes.data, _ptr(w), num_parts, a.ctypes.data,
                                              pw.ctypes.data, C.byref(imb)))
        return Partition(a, num_parts, pw, 0.0, imb.value)

    def make_partition(self, g: Graph, assignment, num_parts: int, doubled_cut: bool = False) -> Partition:
        a = np.ascontiguousarray(assignment, dtype=np.int32)
        pw = np.empty(num_parts)
        cut, imb = C.c_double(), C.c_double()
        gc = g.as_c()
        self._check(self.lib.ref_cut_imbalance(C.byref(gc), a.ctypes.data, num_parts, int(doubled_cut),
                                               C.byref(cut), C.byref(imb), pw.ctypes.data))
        return Partition(a, num_parts, pw, cut.value, imb.value)

    def sym_eig(self, A):
        A = np.asfortranarray(A, dtype=np.float64)
        m = A.shape[0]
        vals = np.empty(m)
        vecs = np.empty((m, m), order="F")
        self._check(self.lib.ref_sym_eig(m, A.ctypes.data, vals.ctypes.data, vecs.ctypes.data))
        return vals, vecs

    def generate(self, spec: str) -> Graph:
        n, nnz = C.c_int64(), C.c_int64()
        self._check(self.lib.ref_generate(spec.encode(), C.byref(n), C.byref(nnz), None, None))
        offs = np.empty(n.value + 1, dtype=np.int64)
        cols = np.empty(max(nnz.value, 1), dtype=np.int32)
        self._check(self.lib.ref_generate(spec.encode(), C.byref(n), C.byref(nnz), offs.ctypes.data,
                                          cols.ctypes.data))
        return Graph(offs, cols[: nnz.value])

    def symmetrize_lcc(self, n: int, row_offsets, col_indices):
        offs = np.ascontiguousarray(row_offsets, dtype=np.int64)
        cols = np.ascontiguousarray(col_indices, dtype=np.int32)
        nn, nz = C.c_int64(), C.c_int64()
        # size query: the component is at most the whole graph
        o = np.empty(n + 1, dtype=np.int64)
        c = np.empty(max(2 * int(offs[-1]), 1), dtype=np.int32)
        old = np.empty(max(n, 1), dtype=np.int64)
        self._check(self.lib.ref_symmetrize_lcc(n, offs.ctypes.data, cols.ctypes.data, C.byref(nn), C.byref(nz),
                                                o.ctypes.data, c.ctypes.data, old.ctypes.data))
        return Graph(o[: nn.value + 1], c[: nz.value]), old[: nn.value]
