"""CPU: host-side logic that mirrors the reference's pure functions."""
import numpy as np
import pytest

from paper_2105_00578_b200 import InfeasibleError, InvalidArgument
from paper_2105_00578_b200 import eigenvector_count, select_defaults, select_initial_vectors, select_precond_auto
from paper_2105_00578_b200 import generators as gen


def test_eigenvector_count_table():
    # partitioner_test.cpp:32-46 / acceptance c3: floor(log2 K) + 1 for K in [2, 4096]
    for k in range(2, 4097):
        e = 0
        while (1 << (e + 1)) <= k:
            e += 1
        assert eigenvector_count(k) == e + 1
    assert eigenvector_count(4) == 3 and eigenvector_count(24) == 5 and eigenvector_count(256) == 9
    with pytest.raises(InfeasibleError):
        eigenvector_count(1)


def test_decision_table():
    # pipeline_test.cpp:30-46 / acceptance c4
    assert select_defaults(True, "jacobi") == ("combinatorial", 1e-3)
    assert select_defaults(True, "polynomial") == ("combinatorial", 1e-3)
    assert select_defaults(True, "amg") == ("combinatorial", 1e-2)
    assert select_defaults(False, "jacobi") == ("generalized", 1e-2)
    assert select_defaults(False, "polynomial") == ("normalized", 1e-2)
    assert select_defaults(False, "amg") == ("generalized", 1e-2)
    assert select_precond_auto(True) == "amg" and select_precond_auto(False) == "polynomial"
    assert select_initial_vectors(True) == "random" and select_initial_vectors(False) == "piecewise"
    with pytest.raises(InvalidArgument):
        select_defaults(True, "auto")


def test_mesh_sizes_match_survey_formulas():
    # 7-point edges 3N^2(N-1); 27-point 3N^2(N-1) + 6N(N-1)^2 + 4(N-1)^3
    for N in (4, 7):
        g7 = gen.stencil3d(N, N, N, 7)
        g27 = gen.stencil3d(N, N, N, 27)
        assert g7.edge_count() == 3 * N * N * (N - 1)
        assert g27.edge_count() == 3 * N * N * (N - 1) + 6 * N * (N - 1) ** 2 + 4 * (N - 1) ** 3
    g = gen.grid2d(7, 5)
    assert g.edge_count() == 7 * 4 + 5 * 6


def test_rmat_symmetric_connected():
    g, old = gen.rmat(10, 8, seed=2)
    n = g.n
    rows = np.repeat(np.arange(n), np.diff(g.row_offsets))
    a = set(zip(rows.tolist(), g.col_indices.tolist()))
    assert all((j, i) in a for i, j in a)           # symmetric pattern
    assert not any(i == j for i, j in a)            # no self-loops
    assert np.all(np.diff(old) > 0)                 # vertices keep their relative order
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    A = csr_matrix((np.ones(len(rows)), g.col_indices, g.row_offsets), shape=(n, n))
    assert connected_components(A, directed=False)[0] == 1


def test_rmat_lcc_matches_reference_semantics():
    from oracle.ref import REF_LIB, RefLib
    if not REF_LIB.exists():
        pytest.skip("compiled reference not available")
    n, s, d = gen.rmat_edges(9, 8, seed=4)
    raw = gen._csr_from_pairs(n, s, d)  # directed pattern, duplicates collapsed
    mine, old = gen.largest_connected_component(gen.symmetrize_pattern(n, s, d))
    ref, rold = RefLib(REF_LIB).symmetrize_lcc(n, raw.row_offsets, raw.col_indices)
    assert np.array_equal(mine.row_offsets, ref.row_offsets) and np.array_equal(mine.col_indices, ref.col_indices)
    assert np.array_equal(old, rold)
