"""GPU parity: device ingestion (ingest.cu) vs the compiled reference.

symmetrize + largest_connected_component (graph.cpp:44-64, 118-171) through
ref_symmetrize_lcc (oracle/ref_driver.cpp), bit-exact on the CSR and the old-id
map; classify (graph.cpp:173-182) against its definition. Inputs are raw square
patterns with duplicates, self-loops, unsorted rows, isolated vertices and ties
between equal-size components (the cases graph_test.cpp exercises).
"""
import numpy as np
import pytest

from paper_2105_00578_b200 import InvalidArgument
from paper_2105_00578_b200 import generators as gen
from paper_2105_00578_b200.api import RunConfig

pytestmark = pytest.mark.gpu


def raw_csr(n, rows, cols, seed=0):
    """Square pattern in CSR with duplicates and self-loops kept, rows unsorted."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int32)
    perm = np.random.default_rng(seed).permutation(rows.shape[0])
    rows, cols = rows[perm], cols[perm]
    order = np.argsort(rows, kind="stable")
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=offs[1:])
    return offs, cols[order]


def _cases():
    rng = np.random.default_rng(11)
    # few random patterns: many small components, duplicates, self-loops
    for n, m in [(1, 0), (1, 3), (2, 1), (7, 5), (64, 40), (300, 200), (1000, 3000)]:
        r = rng.integers(0, n, m)
        c = rng.integers(0, n, m)
        yield f"rand{n}_{m}", n, r, c
    # ties between equal-size components: the one holding the smallest id wins
    yield "tie", 8, np.array([5, 6, 1, 3, 2, 4]), np.array([6, 7, 3, 0, 4, 2])
    # no edges at all: every vertex alone, vertex 0 wins
    yield "isolated", 5, np.array([3]), np.array([3])
    # connected (n_new == n path)
    g = gen.grid2d(13, 9)
    rows = np.repeat(np.arange(g.n), np.diff(g.row_offsets))
    keep = rows < g.col_indices  # one direction only: symmetrize restores the other
    yield "grid_upper", g.n, rows[keep], g.col_indices[keep]
    # power-law: raw R-MAT edge lists (hub rows, most vertices outside the LCC)
    for scale, ef in [(10, 8), (14, 16)]:
        n, s, d = gen.rmat_edges(scale, ef, seed=scale)
        yield f"rmat{scale}", n, s, d


CASES = list(_cases())


@pytest.mark.parametrize("name,n,r,c", CASES, ids=[x[0] for x in CASES])
def test_symmetrize_lcc_bit_exact(ctx, ref, name, n, r, c):
    offs, cols = raw_csr(n, r, c, seed=len(name))
    want, want_old = ref.symmetrize_lcc(n, offs, cols)
    dg = ctx.ingest(offs, cols, lcc=True)
    got, got_old = dg.download()
    info = dg.info()
    dg.free()
    assert np.array_equal(got.row_offsets, want.row_offsets)
    assert np.array_equal(got.col_indices, want.col_indices)
    assert np.array_equal(got_old, want_old)
    assert info.n == want.n and info.nnz == want.row_offsets[-1]


@pytest.mark.parametrize("name,n,r,c", CASES[:9], ids=[x[0] for x in CASES[:9]])
def test_symmetrize_only(ctx, name, n, r, c):
    offs, cols = raw_csr(n, r, c, seed=3)
    want = gen.symmetrize_pattern(n, np.asarray(r), np.asarray(c))
    got = ctx.symmetrize(offs, cols)
    assert np.array_equal(got.row_offsets, want.row_offsets)
    assert np.array_equal(got.col_indices, want.col_indices)


def test_connected_graph_is_identity(ctx):
    g = gen.stencil3d(6, 5, 4, 27)
    got, old = ctx.largest_connected_component(g)
    assert np.array_equal(got.row_offsets, g.row_offsets) and np.array_equal(got.col_indices, g.col_indices)
    assert np.array_equal(old, np.arange(g.n))


def test_tie_picks_smallest_id(ctx, ref):
    # components {5,6,7}, {0,1,3} (both size 3) and {2,4}: graph.cpp:134-141 keeps the one with vertex 0
    offs, cols = raw_csr(8, [5, 6, 1, 3, 2], [6, 7, 3, 0, 4])
    got, old = ctx.ingest(offs, cols).download()
    assert list(old) == [0, 1, 3]


@pytest.mark.parametrize("name,g", [("grid", gen.grid2d(20, 30)), ("st27", gen.stencil3d(7, 6, 5, 27)),
                                    ("star", gen.graph_from_edges(40, [(0, i) for i in range(1, 40)]))])
def test_classify(ctx, name, g):
    k = ctx.classify(g)
    deg = np.diff(g.row_offsets)
    avg = g.row_offsets[-1] / g.n
    assert k.max_degree == deg.max()
    assert k.avg_degree == avg
    assert k.ratio == deg.max() / avg
    assert k.regular == (deg.max() / avg <= 10.0)


def test_errors(ctx):
    with pytest.raises(InvalidArgument):
        ctx.ingest(np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.int32))
    with pytest.raises(InvalidArgument):
        ctx.ingest(np.array([0, 1, 1]), np.array([5], dtype=np.int32))
    with pytest.raises(InvalidArgument):
        ctx.ingest(np.array([0, 1, 1]), np.array([-1], dtype=np.int32))
    with pytest.raises(InvalidArgument):
        ctx.classify(gen.Graph(np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.int32)))


def test_ingest_then_partition_resident(ctx):
    """The CLI pipeline on the device: raw pattern -> symmetrize -> LCC -> partition,
    identical to partition_graph on the downloaded component."""
    n, s, d = gen.rmat_edges(12, 16, seed=5)
    offs, cols = raw_csr(n, s, d)
    dg = ctx.ingest(offs, cols)
    g, old = dg.download()
    cfg = RunConfig(num_parts=8, problem="normalized", precond="jacobi", seed=42)
    a = ctx.partition_resident(dg, cfg)
    b = ctx.partition_graph(g, cfg)
    dg.free()
    assert np.array_equal(a.partition.assignment, b.partition.assignment)
    assert a.partition.cutsize == b.partition.cutsize
