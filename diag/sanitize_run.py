"""Diagnostic workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
one small run of every kernel family of libspecpart_b200.so on cuda:0.

  compute-sanitizer --tool memcheck --error-exitcode 9 python diag/sanitize_run.py

Covers: Laplacian assembly (all kinds), ELL / pattern-ELL / structured-mesh / CSR / binned
irregular SpMMs with every epilogue (through LOBPCG with Jacobi, polynomial and AMG), the
bulk-copy tall-skinny kernels (mbarrier rings), mt19937_64 jump-ahead fill, MJ (CUB sorts),
cut/imbalance, device ingestion (lock-free union-find), AMG setup (expand-sort-reduce).
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_00578_b200 import Context, RunConfig  # noqa: E402
from paper_2105_00578_b200 import generators as gen  # noqa: E402


def main():
    ctx = Context(0)
    mesh7 = gen.stencil3d(34, 32, 12, 7)
    mesh27 = gen.stencil3d(16, 12, 10, 27)
    grid = gen.grid2d(40, 36)
    rm, _ = gen.rmat(12, 16, seed=3)
    for kind in ("combinatorial", "normalized", "degree"):
        ctx.build_laplacian(kind, rm)
        ctx.build_laplacian(kind, mesh27)
    X = np.random.default_rng(0).uniform(-1, 1, (mesh7.n, 7))
    ctx.spmm("combinatorial", mesh7, X)
    ctx.spmm_solver("normalized", rm, np.random.default_rng(1).uniform(-1, 1, (rm.n, 9)))
    runs = [(grid, RunConfig(num_parts=4, precond="jacobi", seed=1)),
            (mesh7, RunConfig(num_parts=8, precond="polynomial", seed=2)),
            (mesh27, RunConfig(num_parts=16, problem="generalized", precond="polynomial", seed=3)),
            (mesh7, RunConfig(num_parts=4, seed=4)),  # auto -> AMG (smoothed, direct coarse)
            (rm, RunConfig(num_parts=8, precond="amg", seed=5)),  # irregular AMG (plain, Chebyshev)
            (rm, RunConfig(num_parts=16, problem="normalized", precond="jacobi", seed=6))]
    for g, cfg in runs:
        r = ctx.partition_graph(g, cfg)
        print(cfg.precond, g.n, r.report.iterations, r.report.cutsize, flush=True)
    n, s, d = gen.rmat_edges(11, 8, seed=9)
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(s, minlength=n), out=offs[1:])
    cols = d[np.argsort(s, kind="stable")].astype(np.int32)
    sub, old = ctx.largest_connected_component(ctx.symmetrize(offs, cols))
    print("ingest", sub.n, flush=True)
    ctx.close()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
