"""GPU: the AX/AH/AP recurrence (sp_context_set_recurrence) against the
reference's recompute-every-iteration LOBPCG (eigensolver.cpp:138-155, 210-222).

With the recurrence the solver applies A only to the new preconditioned block each
iteration and carries A*S, A*X, A*P through the same small transforms; the reported
residuals are true residuals (A*X is recomputed before convergence is accepted). Both
settings must meet the reference's contract: converged, residual <= tol in the
reference's norm (recomputed here with the reference's spmv_block), iterations within
10 %, cut within 2 % and imbalance no worse than the reference's.
"""
import numpy as np
import pytest

from paper_2105_00578_b200 import RunConfig
from paper_2105_00578_b200 import generators as gen

pytestmark = pytest.mark.gpu

CASES = [
    ("grid48_jacobi", gen.grid2d(48, 48), RunConfig(num_parts=4, precond="jacobi", seed=42)),
    ("st7_24_poly", gen.stencil3d(24, 24, 24, 7), RunConfig(num_parts=16, precond="polynomial", seed=42)),
    ("st27_14_gen_poly", gen.stencil3d(14, 14, 14, 27),
     RunConfig(num_parts=8, problem="generalized", precond="polynomial", seed=3)),
    ("rmat13_norm_jacobi", gen.rmat(13, 16, seed=5)[0],
     RunConfig(num_parts=16, problem="normalized", precond="jacobi", seed=42)),
    ("rmat13_gen_jacobi", gen.rmat(13, 16, seed=6)[0], RunConfig(num_parts=8, precond="jacobi", seed=7)),
    ("st7_20_amg", gen.stencil3d(20, 20, 20, 7), RunConfig(num_parts=8, seed=42)),
]


@pytest.mark.parametrize("name,g,cfg", CASES, ids=[c[0] for c in CASES])
def test_recurrence_meets_the_reference_contract(ctx, ref, name, g, cfg):
    b = ref.partition_graph(g, cfg)
    ctx.set_recurrence(True)
    try:
        a = ctx.partition_graph(g, cfg, return_eigenvectors=True)
    finally:
        ctx.set_recurrence(False)
    r = a.report
    assert all(r.converged), (name, r.residual_norms)
    assert abs(r.iterations - b.report.iterations) <= max(2, 0.10 * b.report.iterations), \
        (name, r.iterations, b.report.iterations)
    assert r.cutsize <= 1.02 * b.report.cutsize or abs(r.cutsize - b.report.cutsize) <= 0.02 * b.report.cutsize, \
        (name, r.cutsize, b.report.cutsize)
    assert r.imbalance <= b.report.imbalance + 1e-12
    # true residuals in the reference's norm
    X = a.eigenvectors
    kind = "normalized" if r.problem == "normalized" else "combinatorial"
    LX = ref.spmm(kind, g, X)
    BX = np.diff(g.row_offsets).astype(float)[:, None] * X if r.problem == "generalized" else X
    resid = np.linalg.norm(LX - BX * np.asarray(r.theta)[None, :], axis=0)
    assert np.all(resid <= r.tol * (1 + 1e-6)), (name, resid)
    np.testing.assert_allclose(resid, r.residual_norms, rtol=1e-6, atol=1e-12)


def test_recurrence_saves_spmm_work(ctx):
    g = gen.rmat(13, 16, seed=5)[0]
    cfg = RunConfig(num_parts=16, problem="normalized", precond="jacobi", seed=42)
    off = ctx.partition_graph(g, cfg).report
    ctx.set_recurrence(True)
    try:
        on = ctx.partition_graph(g, cfg).report
    finally:
        ctx.set_recurrence(False)
    per_it_off = off.device["spmm_bytes"] / max(off.iterations, 1)
    per_it_on = on.device["spmm_bytes"] / max(on.iterations, 1)
    assert per_it_on < 0.6 * per_it_off, (per_it_on, per_it_off)
