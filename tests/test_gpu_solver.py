"""GPU parity: LOBPCG, GMRES polynomial preconditioner, end-to-end pipeline.

Mirrors eigensolver_test.cpp:118-306, preconditioner_test.cpp:38-186,
pipeline_test.cpp:66-199 and acceptance c1/c5/c12, with the compiled reference
(oracle/_ref) as the oracle. The solver's data path (block Gram-Schmidt,
reduction order) differs from the reference's at rounding level, so
eigenpairs are compared within the solve tolerance and partitions by cut.
"""
import numpy as np
import pytest

from paper_2105_00578_b200 import BreakdownError, InfeasibleError, RunConfig
from paper_2105_00578_b200 import generators as gen
from paper_2105_00578_b200.api import Graph

pytestmark = pytest.mark.gpu


def _dense(L, n):
    D = np.zeros((n, n))
    for i in range(n):
        for k in range(L["row_offsets"][i], L["row_offsets"][i + 1]):
            D[i, L["col_indices"][k]] += L["values"][k]
    return D


def test_lobpcg_four_cycle_spectrum(ctx):
    # eigensolver_test.cpp:137-150: L_C spectrum {0,2,2,4}; generalized with D=2I halves it
    g = gen.ring(4)
    X0 = ctx.initial_guess("random", 4, 3, 0)
    r = ctx.lobpcg(g, "combinatorial", "none", X0, 1e-9, 500)
    np.testing.assert_allclose(r.theta, [0, 2, 2], atol=1e-8)
    rg = ctx.lobpcg(g, "generalized", "none", X0, 1e-9, 500)
    np.testing.assert_allclose(rg.theta, [0, 1, 1], atol=1e-8)
    rn = ctx.lobpcg(gen.graph_from_edges(2, [(0, 1)]), "normalized", "none",
                    ctx.initial_guess("random", 2, 2, 0), 1e-10, 500)
    np.testing.assert_allclose(rn.theta, [0, 2], atol=1e-9)


def test_lobpcg_kernel_is_constant(ctx):
    g = gen.random_connected_graph(25, 40, seed=5)
    r = ctx.lobpcg(g, "combinatorial", "none", ctx.initial_guess("piecewise", g.n, 1), 1e-8, 500)
    assert abs(r.theta[0]) <= 1e-8 * 2 * np.diff(g.row_offsets).max()
    np.testing.assert_allclose(r.X[:, 0], r.X[0, 0], rtol=1e-6)


@pytest.mark.parametrize("problem", ["combinatorial", "generalized", "normalized"])
def test_lobpcg_oracle_equivalence(ctx, ref, problem):
    # eigensolver_test.cpp:238-258 / acceptance c1: theta within 1e-6 of the dense oracle
    for trial in range(6):
        n = 12 + 9 * trial
        g = gen.random_connected_graph(n, 2 * n, seed=700 + trial)
        X0 = ctx.initial_guess("random", n, 4, 7 + trial)
        r = ctx.lobpcg(g, problem, "jacobi", X0, 1e-8, 3000)
        A = _dense(ref.build_laplacian("normalized" if problem == "normalized" else "combinatorial", g), n)
        if problem == "generalized":
            d = np.diff(g.row_offsets).astype(float)
            w = np.linalg.eigvalsh(A / np.sqrt(np.outer(d, d)))
        else:
            w = np.linalg.eigvalsh(A)
        np.testing.assert_allclose(r.theta, w[:4], atol=1e-6)
        assert r.all_converged()
        q = ref.lobpcg(g, problem, "jacobi", X0, 1e-8, 3000)
        np.testing.assert_allclose(r.theta, q.theta, atol=1e-6)


def test_lobpcg_contracts(ctx, ref):
    # eigensolver_test.cpp:160-192: residual <= tol*bound, X^T B X = I, ascending theta
    g = gen.random_connected_graph(40, 80, seed=23)
    for problem in ("combinatorial", "generalized", "normalized"):
        X0 = ctx.initial_guess("random", g.n, 4, 11)
        r = ctx.lobpcg(g, problem, "jacobi", X0, 1e-6, 1000)
        assert r.all_converged()
        kind = "normalized" if problem == "normalized" else "combinatorial"
        A = _dense(ref.build_laplacian(kind, g), g.n)
        B = np.diag(np.diff(g.row_offsets).astype(float)) if problem == "generalized" else np.eye(g.n)
        bound = ref.build_laplacian(kind, g)["spectral_bound"]
        for j in range(4):
            res = A @ r.X[:, j] - r.theta[j] * (B @ r.X[:, j])
            assert np.linalg.norm(res) <= 1e-6 * bound
        assert np.abs(r.X.T @ B @ r.X - np.eye(4)).max() <= 1e-8
        assert np.all(np.diff(r.theta) >= 0)


def test_lobpcg_deterministic(ctx):
    g = gen.random_connected_graph(60, 150, seed=51)
    X0 = ctx.initial_guess("random", g.n, 3, 77)
    a = ctx.lobpcg(g, "combinatorial", "jacobi", X0, 1e-6)
    b = ctx.lobpcg(g, "combinatorial", "jacobi", X0, 1e-6)
    assert a.theta.tobytes() == b.theta.tobytes() and a.X.tobytes() == b.X.tobytes()
    assert a.iterations == b.iterations


def test_lobpcg_breakdown_after_retry(ctx):
    # eigensolver_test.cpp:274-291 / acceptance c9: rank-1 block -> BreakdownError(retried)
    X0 = np.zeros((4, 3))
    X0[0, :] = 1.0
    with pytest.raises(BreakdownError) as e:
        ctx.lobpcg(gen.ring(4), "combinatorial", "none", X0, 1e-6, 50)
    assert e.value.retried


def test_lobpcg_partial_convergence(ctx):
    g = gen.random_connected_graph(80, 160, seed=61)
    r = ctx.lobpcg(g, "combinatorial", "none", ctx.initial_guess("random", g.n, 4, 9), 1e-12, 2)
    assert r.iterations == 2 and not r.all_converged() and r.X.shape == (80, 4)


def test_locking_changes_path_not_answer(ctx):
    g = gen.random_connected_graph(45, 90, seed=83)
    X0 = ctx.initial_guess("random", g.n, 4, 55)
    a = ctx.lobpcg(g, "combinatorial", "jacobi", X0, 1e-8, 1000, locking=True)
    b = ctx.lobpcg(g, "combinatorial", "jacobi", X0, 1e-8, 1000, locking=False)
    np.testing.assert_allclose(a.theta, b.theta, atol=1e-8)


def test_lobpcg_tracks_reference_iterations(ctx, ref):
    # same X0, same algorithm: iteration counts should match (rounding-level differences)
    g = gen.grid2d(32, 32)
    X0 = ctx.initial_guess("random", g.n, 3, 42)
    a = ctx.lobpcg(g, "combinatorial", "jacobi", X0, 1e-3)
    b = ref.lobpcg(g, "combinatorial", "jacobi", X0, 1e-3)
    assert abs(a.iterations - b.iterations) <= max(2, b.iterations // 20)
    np.testing.assert_allclose(a.theta, b.theta, rtol=1e-6, atol=1e-9)


def _diag_csr(d):
    n = len(d)
    return np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.asarray(d, float)


def test_poly_apply_matches_reference(ctx, ref):
    g = gen.stencil3d(10, 9, 8, 7)
    R = np.random.default_rng(1).uniform(-1, 1, (g.n, 5))
    H, roots = ctx.poly_apply("combinatorial", g, 42, 25, R)
    Hr, deg = ref.poly_apply("combinatorial", g, 42, 25, R)
    assert len(roots) == deg == 25
    np.testing.assert_allclose(H, Hr, rtol=1e-7, atol=1e-9 * np.abs(Hr).max())


def test_poly_linearity(ctx):
    # preconditioner_test.cpp:142-186
    g = gen.grid2d(12, 12)
    rng = np.random.default_rng(2)
    r1, r2 = rng.uniform(-1, 1, (g.n, 2)), rng.uniform(-1, 1, (g.n, 2))
    h1, _ = ctx.poly_apply("combinatorial", g, 5, 25, r1)
    h1b, _ = ctx.poly_apply("combinatorial", g, 5, 25, r1)
    assert h1.tobytes() == h1b.tobytes()
    h0, _ = ctx.poly_apply("combinatorial", g, 5, 25, np.zeros((g.n, 2)))
    assert np.all(h0 == 0)
    h3, _ = ctx.poly_apply("combinatorial", g, 5, 25, 3.0 * r1)
    np.testing.assert_allclose(h3, 3.0 * h1, rtol=1e-12, atol=1e-12 * np.abs(h1).max())
    h2, _ = ctx.poly_apply("combinatorial", g, 5, 25, r2)
    h12, _ = ctx.poly_apply("combinatorial", g, 5, 25, r1 + r2)
    np.testing.assert_allclose(h12, h1 + h2, rtol=1e-11, atol=1e-11 * np.abs(h12).max())


def test_partition_grid_vs_reference(ctx, ref):
    g = gen.grid2d(64, 64)
    cfg = RunConfig(num_parts=4, precond="jacobi", seed=42)
    a = ctx.partition_graph(g, cfg)
    b = ref.partition_graph(g, cfg)
    assert a.report.problem == b.report.problem == "combinatorial"
    assert a.report.tol == b.report.tol == 1e-3
    assert a.report.imbalance <= b.report.imbalance + 1e-12
    assert abs(a.report.cutsize - b.report.cutsize) <= 0.02 * b.report.cutsize
    assert abs(a.report.iterations - b.report.iterations) <= max(3, b.report.iterations // 10)
    redo = ctx.make_partition(g, a.partition.assignment, 4)
    assert redo.cutsize == a.report.cutsize


def test_partition_poly_vs_reference(ctx, ref):
    g = gen.stencil3d(16, 16, 16, 7)
    cfg = RunConfig(num_parts=8, precond="polynomial", seed=42)
    a = ctx.partition_graph(g, cfg)
    b = ref.partition_graph(g, cfg)
    assert a.report.poly_degree == 25
    assert abs(a.report.cutsize - b.report.cutsize) <= 0.02 * b.report.cutsize
    assert a.report.imbalance <= b.report.imbalance + 1e-12
    assert all(a.report.converged)


def test_pipeline_kats(ctx):
    # pipeline_test.cpp:66-96
    r = ctx.partition_graph(gen.ring(8), RunConfig(num_parts=2, tol=1e-6, seed=5, precond="jacobi"))
    assert r.report.cutsize == 2.0 and list(r.partition.part_weights) == [4.0, 4.0]
    a = r.partition.assignment
    assert sum(a[i] != a[(i + 1) % 8] for i in range(8)) == 2
    r = ctx.partition_graph(gen.grid2d(4, 4), RunConfig(num_parts=4, tol=1e-8, seed=3, precond="jacobi"))
    assert r.report.eigenvectors == 3 and list(r.partition.part_weights) == [4.0] * 4
    with pytest.raises(InfeasibleError):
        ctx.partition_graph(gen.ring(5), RunConfig(num_parts=6, precond="jacobi"))


def test_pipeline_irregular_normalized(ctx, ref):
    g, _ = gen.largest_connected_component(gen.symmetrize_pattern(*gen.rmat_edges(12, 16, seed=3)))
    cfg = RunConfig(num_parts=8, precond="jacobi", problem="normalized", seed=42)
    a = ctx.partition_graph(g, cfg)
    b = ref.partition_graph(g, cfg)
    assert not a.report.regular and a.report.tol == 1e-2
    assert a.report.init == "piecewise"
    assert abs(a.report.cutsize - b.report.cutsize) <= 0.02 * b.report.cutsize
    np.testing.assert_allclose(a.report.theta, b.report.theta, rtol=1e-3, atol=1e-2)


def test_cpp_shim_caller():
    # a reference-style C++ caller compiled against include/specpart_b200.hpp
    import subprocess
    from pathlib import Path
    exe = Path(__file__).resolve().parent.parent / "build" / "shim_test"
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cpp_reference_caller_run_partition():
    # tools/specpart.cpp:63-184's call sequence (parse -> symmetrize -> LCC -> partition_graph,
    # and the --init-file stage-by-stage path) compiled against the shim (tests/cpp/caller_test.cpp)
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    exe = root / "build" / "caller_test"
    for mtx in ("grid32.mtx", "messy.mtx"):
        r = subprocess.run([str(exe), str(root / "tests" / "golden" / "cli" / mtx)], capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "0 failures" in r.stdout
