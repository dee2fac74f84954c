"""GPU parity: kernel-level seams of the CUDA library vs the CPU reference.

Bit-exact where the reference is (Laplacian assembly: laplacian_test.cpp:30-211;
SpMM vs spmv_block_serial: kernels_test.cpp:26-35; initial blocks; MJ; cut /
imbalance: graph_test.cpp:225-275), fp tolerance where it is not (Gram:
kernels_test.cpp:37-48 allows 1e-13).
"""
import numpy as np
import pytest

from paper_2105_00578_b200 import DegenerateDegreeError, InfeasibleError, InvalidArgument
from paper_2105_00578_b200 import generators as gen
from paper_2105_00578_b200.api import Graph

pytestmark = pytest.mark.gpu


def _graphs():
    yield "path3", gen.path(3)
    yield "edge", gen.graph_from_edges(2, [(0, 1)])
    yield "k3", gen.graph_from_edges(3, [(0, 1), (1, 2), (0, 2)])
    yield "star", gen.graph_from_edges(4, [(0, 1), (0, 2), (0, 3)])
    yield "ring8", gen.ring(8)
    yield "grid20", gen.grid2d(20, 17)
    yield "st7", gen.stencil3d(9, 8, 7, 7)
    yield "st27", gen.stencil3d(6, 7, 5, 27)
    for s in range(4):
        yield f"rand{s}", gen.random_connected_graph(30 + 17 * s, 60 + 40 * s, seed=s)
    # rows longer than one warp's 32-term group (normal_bound_kernel's unrolled path)
    yield "star100", gen.graph_from_edges(101, [(0, i) for i in range(1, 101)] + [(i, i + 1) for i in range(1, 100)])
    yield "rmat10", gen.rmat(10, 16, seed=3)[0]
    # weighted costs: laplacian_test.cpp:173-211 style
    g = gen.random_connected_graph(50, 120, seed=9)
    rng = np.random.default_rng(3)
    w = rng.uniform(0.5, 3.0, g.col_indices.shape[0])
    # symmetric costs: w_ij = w_ji
    n = g.n
    rows = np.repeat(np.arange(n), np.diff(g.row_offsets))
    key_lo = np.minimum(rows, g.col_indices) * n + np.maximum(rows, g.col_indices)
    _, inv = np.unique(key_lo, return_inverse=True)
    sym = rng.uniform(0.5, 3.0, inv.max() + 1)[inv]
    yield "weighted", Graph(g.row_offsets, g.col_indices, sym, None)


GRAPHS = list(_graphs())


@pytest.mark.parametrize("kind", ["combinatorial", "normalized", "degree"])
@pytest.mark.parametrize("name,g", GRAPHS, ids=[n for n, _ in GRAPHS])
def test_laplacian_bit_exact(ctx, ref, kind, name, g):
    a = ctx.build_laplacian(kind, g)
    b = ref.build_laplacian(kind, g)
    for key in ("row_offsets", "col_indices"):
        assert np.array_equal(a[key], b[key]), key
    assert a["values"].tobytes() == b["values"].tobytes()
    assert a["diag"].tobytes() == b["diag"].tobytes()
    assert a["spectral_bound"] == b["spectral_bound"]
    assert a["is_diagonal"] == b["is_diagonal"]


def test_laplacian_kats(ctx):
    # laplacian_test.cpp:30-87
    L = ctx.build_laplacian("combinatorial", gen.path(3))
    dense = np.zeros((3, 3))
    for i in range(3):
        for k in range(L["row_offsets"][i], L["row_offsets"][i + 1]):
            dense[i, L["col_indices"][k]] = L["values"][k]
    assert np.array_equal(dense, [[1, -1, 0], [-1, 2, -1], [0, -1, 1]])
    N = ctx.build_laplacian("normalized", gen.graph_from_edges(3, [(0, 1), (1, 2), (0, 2)]))
    off = N["values"][N["col_indices"] != np.repeat(np.arange(3), 3)]
    assert np.allclose(off, -0.5)
    D = ctx.build_laplacian("degree", gen.graph_from_edges(4, [(0, 1), (0, 2), (0, 3)]))
    assert list(D["diag"]) == [3, 1, 1, 1] and D["is_diagonal"]


def test_normalized_rejects_isolated_vertex(ctx):
    g = gen.graph_from_edges(3, [(0, 1)])
    with pytest.raises(DegenerateDegreeError):
        ctx.build_laplacian("normalized", g)


@pytest.mark.parametrize("kind", ["combinatorial", "normalized", "degree"])
@pytest.mark.parametrize("m", [1, 3, 5, 7, 9, 21, 27, 40])
def test_spmm_bit_exact(ctx, ref, kind, m):
    g = gen.stencil3d(9, 9, 9, 27)
    rng = np.random.default_rng(m)
    X = rng.uniform(-1, 1, (g.n, m))
    assert ctx.spmm(kind, g, X).tobytes() == ref.spmm(kind, g, X).tobytes()


@pytest.mark.parametrize("name,g", GRAPHS[-7:], ids=[n for n, _ in GRAPHS[-7:]])
def test_spmm_bit_exact_irregular(ctx, ref, name, g):
    X = np.random.default_rng(1).uniform(-1, 1, (g.n, 7))
    for kind in ("combinatorial", "normalized"):
        assert ctx.spmm(kind, g, X).tobytes() == ref.spmm(kind, g, X).tobytes()


def test_spmm_csr_matches_spmv_block(ctx, ref):
    L = ref.build_laplacian("combinatorial", gen.stencil3d(9, 9, 9, 27))
    X = np.random.default_rng(2).uniform(-1, 1, (729, 5))
    a = ctx.spmm_csr(L["row_offsets"], L["col_indices"], L["values"], X)
    b = ref.spmm_csr(L["row_offsets"], L["col_indices"], L["values"], X)
    assert a.tobytes() == b.tobytes()


def test_cut_identity_exact(ctx):
    # acceptance c2 (acceptance.cpp:99-122): x^T L_C x / 4 == cutsize, exactly
    for s in range(20):
        g = gen.random_connected_graph(10 + s, 2 * (10 + s), seed=100 + s)
        part = np.random.default_rng(s).integers(0, 2, g.n).astype(np.int32)
        if part.min() == part.max():
            part[0] = 1 - part[0]
        x = np.where(part == 0, 1.0, -1.0)
        Lx = ctx.spmm("combinatorial", g, x[:, None])[:, 0]
        p = ctx.make_partition(g, part, 2)
        assert float(x @ Lx) / 4.0 == p.cutsize


def test_gram_matches_and_is_deterministic(ctx, ref):
    rng = np.random.default_rng(3)
    U = rng.uniform(-1, 1, (20000, 4))
    V = rng.uniform(-1, 1, (20000, 3))
    a = ctx.gram(U, V)
    b = ctx.gram(U, V)
    assert a.tobytes() == b.tobytes()
    np.testing.assert_allclose(a, U.T @ V, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(a, ref.gram(U, V), rtol=1e-12, atol=1e-12)
    d = rng.uniform(1, 5, 20000)
    np.testing.assert_allclose(ctx.gram(U, V, d), U.T @ (d[:, None] * V), rtol=1e-12, atol=1e-11)


@pytest.mark.parametrize("mu,mv", [(1, 1), (9, 9), (27, 27), (18, 9), (40, 5)])
def test_gram_shapes(ctx, mu, mv):
    rng = np.random.default_rng(mu * 100 + mv)
    n = 5000 + mu
    U, V = rng.standard_normal((n, mu)), rng.standard_normal((n, mv))
    np.testing.assert_allclose(ctx.gram(U, V), U.T @ V, rtol=1e-11, atol=1e-10)


@pytest.mark.parametrize("init,n,d,seed", [("random", 1000, 3, 42), ("random", 777, 7, 5), ("piecewise", 1001, 4, 0),
                                           ("piecewise", 10, 9, 0)])
def test_initial_guess_bit_identical(ctx, ref, init, n, d, seed):
    assert ctx.initial_guess(init, n, d, seed).tobytes() == ref.initial_guess(init, n, d, seed).tobytes()


def test_mj_identical_to_reference(ctx, ref):
    rng = np.random.default_rng(15)
    for trial in range(25):
        n = int(rng.integers(1, 300))
        k = int(rng.integers(1, n + 1))
        dims = int(rng.integers(1, 5))
        coords = rng.uniform(-1, 1, (n, dims))
        a = ctx.mj_partition(coords, None, k)
        b = ref.mj_partition(coords, None, k)
        assert np.array_equal(a.assignment, b.assignment), (n, k, dims)
        assert np.array_equal(a.part_weights, b.part_weights)


def test_mj_ties_weights_and_zero_sign(ctx, ref):
    # partitioner_test.cpp:213-236
    assert list(ctx.mj_partition(np.ones((4, 1)), None, 2).assignment) == [0, 0, 1, 1]
    p = ctx.mj_partition(np.array([[0.0], [1.0], [2.0], [3.0]]), [3.0, 1.0, 1.0, 1.0], 2)
    assert list(p.assignment) == [0, 1, 1, 1]
    # -0.0 == +0.0 ties break by id
    c = np.array([[0.0], [-0.0], [0.0], [-0.0], [1.0], [-1.0]])
    assert np.array_equal(ctx.mj_partition(c, None, 3).assignment, ref.mj_partition(c, None, 3).assignment)
    rng = np.random.default_rng(4)
    for trial in range(10):
        n = 200
        coords = np.round(rng.uniform(-1, 1, (n, 3)), 1)  # many ties
        w = rng.uniform(0.1, 2.0, n)
        for K in (2, 5, 8, 13):
            a = ctx.mj_partition(coords, w, K)
            b = ref.mj_partition(coords, w, K)
            assert np.array_equal(a.assignment, b.assignment)
    with pytest.raises(InfeasibleError):
        ctx.mj_partition(np.array([[0.0], [1.0]]), None, 3)


def test_mj_large_identical(ctx, ref):
    rng = np.random.default_rng(7)
    coords = rng.standard_normal((200000, 6))
    for K in (64, 100):
        a = ctx.mj_partition(coords, None, K)
        b = ref.mj_partition(coords, None, K)
        assert np.array_equal(a.assignment, b.assignment)


@pytest.mark.parametrize("case", ["ties", "clustered", "tiny_nodes", "signed_zero"])
def test_mj_select_unit_weights(ctx, ref, case):
    # the unit-weight MJ cuts by radix select (mj.cu): buckets past 4,096 points need more
    # digit passes (heavy ties reach the id digits), nodes of a few points skip them
    rng = np.random.default_rng(11)
    if case == "ties":
        coords = np.round(rng.uniform(-1, 1, (150000, 3)), 2)  # ~200 distinct values per axis
        ks = (2, 7, 64, 100)
    elif case == "clustered":
        coords = 1e-3 * (1.0 + 1e-9 * rng.standard_normal((120000, 4)))  # one binade, 12+ equal top bits
        ks = (3, 64, 256)
    elif case == "tiny_nodes":
        coords = rng.uniform(-1, 1, (300, 2))
        ks = (150, 299, 300)
    else:
        coords = rng.choice(np.array([0.0, -0.0, 1e-300, -1e-300, 2.0]), size=(20000, 2))
        ks = (5, 17)
    for K in ks:
        a = ctx.mj_partition(coords, None, K)
        b = ref.mj_partition(coords, None, K)
        assert np.array_equal(a.assignment, b.assignment), (case, K)
        assert np.array_equal(a.part_weights, b.part_weights), (case, K)


def test_make_partition_exact(ctx, ref):
    g = gen.stencil3d(12, 11, 10, 27)
    rng = np.random.default_rng(8)
    for K in (2, 7, 64):
        a = rng.integers(0, K, g.n).astype(np.int32)
        a[:K] = np.arange(K)
        for doubled in (False, True):
            p, q = ctx.make_partition(g, a, K, doubled), ref.make_partition(g, a, K, doubled)
            assert p.cutsize == q.cutsize and p.imbalance == q.imbalance
            assert np.array_equal(p.part_weights, q.part_weights)
    # KATs: graph_test.cpp:225-255
    tri = gen.graph_from_edges(3, [(0, 1), (1, 2), (0, 2)])
    assert ctx.make_partition(tri, [0, 1, 1], 2).cutsize == 2.0
    assert ctx.make_partition(tri, [0, 1, 1], 2, True).cutsize == 4.0
    with pytest.raises(InvalidArgument):
        ctx.make_partition(tri, [0, 0, 0], 2)  # empty part
    with pytest.raises(InvalidArgument):
        ctx.make_partition(tri, [0, 1, 2], 2)  # out of range


# ---- the eigensolver's own irregular-graph SpMM (row-length bins, chunked hub rows) ----
def _hub_graph():
    """R-MAT LCC plus one hub row of 15,000 entries and one of 9,000 (both > the
    4,096-entry chunk, so the ordered multi-chunk finish runs), every bin populated."""
    g, _ = gen.rmat(14, 16, seed=5)
    n = g.n
    rows = np.repeat(np.arange(n), np.diff(g.row_offsets))
    edges = np.stack([rows, g.col_indices], axis=1)
    edges = edges[edges[:, 0] < edges[:, 1]]
    hub = [(0, j) for j in range(1, min(n, 15001))] + [(n - 1, j) for j in range(0, min(n - 1, 9000), 1)]
    return gen.graph_from_edges(n, np.concatenate([edges, np.array(hub)]))


HUB = _hub_graph()


def test_hub_graph_shape():
    deg = np.diff(HUB.row_offsets)
    assert deg.max() > 3 * 4096 and (deg > 4096).sum() >= 2
    for lo, hi in [(1, 16), (17, 64), (65, 256), (257, 512), (513, 4096)]:
        assert ((deg >= lo) & (deg <= hi)).any(), (lo, hi)


def _abs_bound(ref, kind, g, X):
    """sum_k |a_ik x_k| per (row, column), from the reference's own L."""
    import scipy.sparse as sp
    L = ref.build_laplacian(kind, g)
    A = sp.csr_matrix((np.abs(L["values"]), L["col_indices"], L["row_offsets"]), shape=(g.n, g.n))
    return A @ np.abs(X), np.diff(L["row_offsets"])


@pytest.mark.parametrize("m", [1, 7, 9, 21, 27])
def test_solver_spmm_irregular_integer_exact(ctx, ref, m):
    # integer-valued X: every partial sum of L_C x is an exact integer, so any
    # summation order must reproduce spmv_block bit for bit
    X = np.random.default_rng(m).integers(-8, 9, (HUB.n, m)).astype(np.float64)
    assert ctx.classify(HUB).regular is False
    assert ctx.spmm_solver("combinatorial", HUB, X).tobytes() == ref.spmm("combinatorial", HUB, X).tobytes()


@pytest.mark.parametrize("kind", ["combinatorial", "normalized"])
@pytest.mark.parametrize("m", [1, 7, 9, 21, 27])
def test_solver_spmm_irregular_within_rounding(ctx, ref, kind, m):
    # any-order summation bound: |fl(sum) - sum| <= gamma_{len} * sum|terms| for both
    # the reference's sequential row sums and the device's chunked/butterfly sums
    X = np.random.default_rng(100 + m).uniform(-1, 1, (HUB.n, m))
    y = ctx.spmm_solver(kind, HUB, X)
    y_ref = ref.spmm(kind, HUB, X)
    S, lens = _abs_bound(ref, kind, HUB, X)
    eps = np.finfo(np.float64).eps / 2
    gam = (lens * eps / (1 - lens * eps))[:, None]
    err = np.abs(y - y_ref)
    assert np.all(err <= 2 * gam * S + 1e-300), float(np.max(err / (gam * S + 1e-300)))
    # rows short enough for a single ordered chain are far tighter in practice
    assert np.median((err / (eps * S + 1e-300))[lens > 100]) < 64


# ---- multi-chunk mt19937_64 jump-ahead (rng.cu) and row slices -------------------
@pytest.mark.parametrize("n,d", [(300_001, 9), (1_000_003, 3)])
def test_initial_guess_multi_chunk(ctx, ref, n, d):
    assert n * d > 4 * (1 << 18)  # at least four 2^18-draw chunks
    full = ctx.initial_guess("random", n, d, 42)
    assert full.tobytes() == ref.initial_guess("random", n, d, 42).tobytes()
    rng = np.random.default_rng(n)
    slices = [(0, 1), (1, 262_143), (262_143, 2), (n - 5, 5), (n // 3, n // 3 + 7)]
    slices += [(int(a), int(rng.integers(1, n - a))) for a in rng.integers(0, n - 1, 4)]
    for row0, nloc in slices:
        part = ctx.initial_guess_rows("random", n, d, 42, row0, nloc)
        assert part.tobytes() == np.asfortranarray(full[row0:row0 + nloc]).tobytes(), (row0, nloc)
    pw = ref.initial_guess("piecewise", n, d, 0)
    for row0, nloc in slices[:4]:
        part = ctx.initial_guess_rows("piecewise", n, d, 0, row0, nloc)
        assert part.tobytes() == np.asfortranarray(pw[row0:row0 + nloc]).tobytes(), (row0, nloc)


# ---- structured-mesh SpMM (spmm_mesh.cu: TMA 3-D tiles, z-marching): bit-exact -------
MESHES = [("st7_40x12x10", gen.stencil3d(40, 12, 10, 7)), ("st27_34x8x6", gen.stencil3d(34, 8, 6, 27)),
          ("grid_66x40", gen.grid2d(66, 40)), ("st7_64x64x64", gen.stencil3d(64, 64, 64, 7)),
          ("st27_32x32x40", gen.stencil3d(32, 32, 40, 27))]


@pytest.mark.parametrize("m", [1, 3, 7, 9, 21])
@pytest.mark.parametrize("name,g", MESHES, ids=[n for n, _ in MESHES])
def test_spmm_bit_exact_structured_mesh(ctx, ref, name, g, m):
    X = np.random.default_rng(m).uniform(-1, 1, (g.n, m))
    assert ctx.spmm("combinatorial", g, X).tobytes() == ref.spmm("combinatorial", g, X).tobytes()


@pytest.mark.parametrize("n,k,m", [(1, 1, 1), (1000, 9, 9), (20001, 27, 9), (5000, 18, 4), (70001, 3, 3), (300, 40, 21)])
def test_block_combine_matches_mult(ctx, ref, n, k, m):
    """sp_block_combine vs kernels::mult / mult_sub (kernels.cpp:127-157)."""
    rng = np.random.default_rng(n + k * 7 + m)
    X, C, Y = rng.uniform(-1, 1, (n, k)), rng.uniform(-1, 1, (k, m)), rng.uniform(-1, 1, (n, m))
    bound = np.abs(X) @ np.abs(C) * (k + 2) * np.finfo(float).eps
    a = ctx.mult(X, C)
    assert a.tobytes() == ctx.mult(X, C).tobytes()
    assert np.all(np.abs(a - ref.mult(X, C)) <= bound)
    b = ctx.mult(X, C, Y)
    assert np.all(np.abs(b - ref.mult(X, C, Y)) <= bound + np.abs(Y) * np.finfo(float).eps)


def test_block_combine_rejects_bad_shapes(ctx):
    from paper_2105_00578_b200 import DimensionError
    with pytest.raises(DimensionError):
        ctx.mult(np.ones((4, 3)), np.ones((2, 2)))
    with pytest.raises(DimensionError):
        ctx.mult(np.ones((4, 65)), np.ones((65, 2)))


def test_two_step_polynomial_kernel_bit_identical(tmp_path):
    """spmm_mesh_poly2_kernel (two polynomial steps per pass) against one step per launch
    (SPB_POLY2=0): the same bytes for every degree (odd / even step counts) and width."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    outs = []
    for env_val in ("0", "1"):
        f = tmp_path / f"poly2_{env_val}.bin"
        env = dict(os.environ, SPB_POLY2=env_val)
        r = subprocess.run([sys.executable, str(here / "poly2_workload.py"), str(f)], capture_output=True, text=True,
                           timeout=600, env=env)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(f.read_bytes())
    assert len(outs[0]) > 0 and outs[0] == outs[1]
