"""GPU preconditioners vs the reference (src/preconditioners.cpp) through the apply seams.

Known-answer tests of tests/preconditioner_test.cpp:38-118 on explicit diagonal operators
(sp_precond_apply_csr), acceptance c12 (tests/acceptance.cpp:361-403: degree-m GMRES
polynomial = exact inverse for m distinct eigenvalues), the linearity properties of
preconditioner_test.cpp:142-186 for every preconditioner (sp_precond_apply), and H = M R
against the reference's own M->apply for Jacobi, polynomial and AMG.
"""
import numpy as np
import pytest

from paper_2105_00578_b200 import generators as gen

pytestmark = pytest.mark.gpu


def diag_op(d):
    n = len(d)
    return np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.asarray(d, dtype=np.float64)


def test_jacobi_kats(ctx):
    o, c, v = diag_op([2.0, 4.0])
    H, _ = ctx.precond_apply_csr(o, c, v, "jacobi", np.ones((2, 1)))
    assert np.allclose(H[:, 0], [0.5, 0.25])
    o, c, v = diag_op([1.0, 1.0, 1.0])
    R = np.random.default_rng(8).uniform(-1, 1, (3, 2))
    H, _ = ctx.precond_apply_csr(o, c, v, "jacobi", R)
    assert H.tobytes() == np.asfortranarray(R).tobytes()
    # near-zero diagonal -> identity row (preconditioners.cpp:44-49)
    o, c, v = diag_op([2.0, 0.0])
    H, _ = ctx.precond_apply_csr(o, c, v, "jacobi", np.array([[1.0], [3.0]]))
    assert np.allclose(H[:, 0], [0.5, 3.0])
    # unit-degree laplacian row: graph_from_edges(2, {0,1})
    g = gen.graph_from_edges(2, [(0, 1)])
    H = ctx.precond_apply("combinatorial", g, "jacobi", np.array([[1.0], [0.0]]))
    assert H[0, 0] == 1.0 and H[1, 0] == 0.0


def test_polynomial_kats(ctx, ref):
    # exact on 2I at degree 1
    o, c, v = diag_op([2.0] * 4)
    R = np.random.default_rng(12).uniform(-1, 1, (4, 2))
    H, roots = ctx.precond_apply_csr(o, c, v, "polynomial", R, seed=4, degree=1)
    assert np.allclose(H, 0.5 * R, rtol=1e-14, atol=0) and len(roots) == 1
    # early Arnoldi breakdown truncates: 3I, degree 9 -> achieved 1 (single distinct eigenvalue)
    o, c, v = diag_op([3.0] * 5)
    H, roots = ctx.precond_apply_csr(o, c, v, "polynomial", np.ones((5, 1)), seed=4, degree=9)
    Hr, ach = ref.poly_apply_csr(o, c, v, 4, 9, np.ones((5, 1)))
    assert len(roots) == ach == 1
    np.testing.assert_allclose(H, Hr, rtol=1e-13)
    # {1, 3} repeated, degree 2 -> exact inverse to 1e-10
    d = [1.0, 3.0] * 5
    o, c, v = diag_op(d)
    R = np.random.default_rng(5).uniform(-1, 1, (10, 3))
    H, roots = ctx.precond_apply_csr(o, c, v, "polynomial", R, seed=99, degree=2)
    np.testing.assert_allclose(H, R / np.asarray(d)[:, None], rtol=1e-10, atol=0)


def test_c12_polynomial_exactness(ctx, ref):
    rng = np.random.default_rng(5150)
    for m in range(1, 11):
        distinct = 0.5 + np.arange(m) + 0.25 * rng.random(m)
        n = 40
        d = distinct[np.arange(n) % m]
        o, c, v = diag_op(d)
        R = np.random.default_rng(m).uniform(-1, 1, (n, 2))
        H, roots = ctx.precond_apply_csr(o, c, v, "polynomial", R, seed=31 + m, degree=m)
        want = R / d[:, None]
        assert np.all(np.abs(H - want) <= 1e-10 * np.maximum(1.0, np.abs(want))), m
        Hr, ach = ref.poly_apply_csr(o, c, v, 31 + m, m, R)
        assert len(roots) == ach


GRAPHS = [("grid24", gen.grid2d(24, 24)), ("st7_12", gen.stencil3d(12, 12, 12, 7)),
          ("rmat11", gen.rmat(11, 16, seed=2)[0]), ("rand300", gen.random_connected_graph(300, 900, seed=4))]


# Tolerances: Jacobi is elementwise (exact). AMG's direct coarse solve of the shifted
# singular L_C (shift 1e-8 trace/n, preconditioners.cpp:619-633) amplifies the Galerkin
# products' rounding by up to ~1e8. The degree-25 product-form GMRES polynomial is only
# compared where its SpMMs are bit-exact (meshes, L_C): its roots include harmonic Ritz
# values near 0 (on L_N the mean-subtracted seed vector of polynomial_build keeps a
# component in the null space D^1/2 1, :327-336), so prod (I - A/theta_i) amplifies any
# rounding difference by orders of magnitude — the reference's own algorithm, not a
# device effect; the irregular graphs' binned SpMMs sum in another order.
TOL = {"jacobi": 1e-14, "polynomial": 1e-9, "amg": 1e-6}


@pytest.mark.parametrize("precond", ["jacobi", "polynomial", "amg"])
@pytest.mark.parametrize("name,g", GRAPHS, ids=[n for n, _ in GRAPHS])
def test_apply_matches_reference(ctx, ref, name, g, precond):
    irregular = name.startswith(("rmat", "rand"))
    if precond == "polynomial" and irregular:
        pytest.skip("ill-conditioned product form: compared on meshes only (see TOL)")
    kind = "normalized" if irregular else "combinatorial"
    R = np.random.default_rng(3).uniform(-1, 1, (g.n, 5))
    H = ctx.precond_apply(kind, g, precond, R, seed=17)
    Hr = ref.precond_apply(kind, g, precond, R, seed=17)
    scale = np.max(np.abs(Hr))
    assert np.max(np.abs(H - Hr)) <= TOL[precond] * scale, (name, precond, np.max(np.abs(H - Hr)) / scale)


@pytest.mark.parametrize("precond", ["jacobi", "polynomial", "amg"])
def test_apply_is_linear_and_deterministic(ctx, precond):
    # preconditioner_test.cpp:142-186: deterministic, apply(0) = 0, homogeneity, additivity
    g = gen.stencil3d(10, 9, 8, 27)
    rng = np.random.default_rng(21)
    A, B = rng.uniform(-1, 1, (g.n, 3)), rng.uniform(-1, 1, (g.n, 3))
    HA = ctx.precond_apply("combinatorial", g, precond, A, seed=5)
    assert HA.tobytes() == ctx.precond_apply("combinatorial", g, precond, A, seed=5).tobytes()
    assert not np.any(ctx.precond_apply("combinatorial", g, precond, np.zeros((g.n, 3)), seed=5))
    H3 = ctx.precond_apply("combinatorial", g, precond, 3.0 * A, seed=5)
    np.testing.assert_allclose(H3, 3.0 * HA, rtol=0, atol=1e-12 * np.max(np.abs(H3)))
    HB = ctx.precond_apply("combinatorial", g, precond, B, seed=5)
    HAB = ctx.precond_apply("combinatorial", g, precond, A + B, seed=5)
    np.testing.assert_allclose(HAB, HA + HB, rtol=0, atol=1e-11 * np.max(np.abs(HAB)))
