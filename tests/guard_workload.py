"""Run in a SPECPART_B200_GUARD=1 process by tests/test_gpu_guard.py (not collected by pytest):
small cases of every kernel family of the library, then the guard-band verdict as one JSON line."""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_00578_b200 import Context, RunConfig  # noqa: E402
from paper_2105_00578_b200 import generators as gen  # noqa: E402


def star_plus_ring(n, hubs=2):
    """rows of n-1 entries (chunked hub rows, ordered finish) on top of a ring"""
    e = [(i, (i + 1) % n) for i in range(n)]
    for h in range(hubs):
        e += [(h, j) for j in range(n) if j != h and abs(j - h) > 1]
    return gen.graph_from_edges(n, e)


def main():
    ctx = Context(0)
    rng = np.random.default_rng(0)
    done = []
    meshes = [gen.grid2d(40, 33), gen.stencil3d(20, 17, 9, 7), gen.stencil3d(12, 11, 10, 27)]
    irregular = [gen.rmat(11, 8, seed=3)[0], star_plus_ring(9000)]
    for g in meshes + irregular:
        for m in (1, 3, 7, 9):
            X = rng.uniform(-1, 1, (g.n, m))
            for kind in ("combinatorial", "normalized"):
                ctx.spmm(kind, g, X)
                ctx.spmm_solver(kind, g, X)
            ctx.spmm_csr(g.row_offsets, g.col_indices, np.ones(int(g.row_offsets[-1])), X)
        for pre in ("jacobi", "polynomial", "amg"):
            ctx.precond_apply("combinatorial", g, pre, rng.uniform(-1, 1, (g.n, 4)), seed=1, degree=10)
        done.append(f"spmm+precond n={g.n}")
    for n, k, m in ((10000, 9, 9), (3000, 27, 4), (7, 3, 2)):
        X, Cm = rng.uniform(-1, 1, (n, k)), rng.uniform(-1, 1, (k, m))
        ctx.mult(X, Cm)
        ctx.mult(X, Cm, rng.uniform(-1, 1, (n, m)))
        ctx.gram(X, X)
        ctx.gram(X, rng.uniform(-1, 1, (n, m)), rng.uniform(1, 2, n))
    ctx.initial_guess("random", 300000, 4, 7)
    ctx.initial_guess_rows("random", 300000, 4, 7, 12345, 99999)
    ctx.mj_partition(rng.uniform(-1, 1, (5000, 3)), None, 37)
    done.append("blockops/rng/mj")
    cases = [(meshes[0], RunConfig(num_parts=8, precond="jacobi", seed=1)),
             (meshes[1], RunConfig(num_parts=16, precond="polynomial", seed=1)),
             (meshes[2], RunConfig(num_parts=8, problem="generalized", precond="polynomial", seed=2)),
             (meshes[1], RunConfig(num_parts=8, seed=3)),
             (irregular[0], RunConfig(num_parts=16, problem="normalized", precond="jacobi", seed=4)),
             (irregular[0], RunConfig(num_parts=8, precond="amg", seed=5))]
    for rec in (False, True):
        ctx.set_recurrence(rec)
        for g, cfg in cases:
            ctx.partition_graph(g, cfg)
    ctx.set_recurrence(False)
    g = irregular[0]
    dg = ctx.ingest(g.row_offsets, g.col_indices)
    ctx.partition_resident(dg, RunConfig(num_parts=4, seed=1))
    dg.free()
    done.append("partition (jacobi/poly/amg, recurrence on/off, ingest+resident)")
    v, b = C.c_int64(), C.c_int64()
    st = ctx.lib.sp_debug_guard_check(C.byref(v), C.byref(b))
    ctx.close()
    v2, b2 = C.c_int64(), C.c_int64()
    ctx.lib.sp_debug_guard_check(C.byref(v2), C.byref(b2))
    print(json.dumps({"status": st, "violations": v2.value, "buffers": b2.value, "stages": done}))


if __name__ == "__main__":
    main()
