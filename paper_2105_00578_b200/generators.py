"""Synthetic inputs for tests and benchmarks (host tooling, not the hot path).

Mesh generators produce exactly the CSR of the reference's generators
(src/generators.cpp:126-162: vertex id (z*ny + y)*nx + x, unit costs, columns
ascending) without building an edge list: per-row neighbours are enumerated in
lexicographic stencil order, which is ascending id order.

R-MAT is new (the reference has none): Graph500 Kronecker
generator (a, b, c, d) = (0.57, 0.19, 0.19, 0.05), edgefactor 16, a seeded
random vertex relabel, then the reference's symmetrize (graph.cpp:44-64) and
largest_connected_component (graph.cpp:118-171) semantics.
"""
from __future__ import annotations

import numpy as np

from .api import Graph


def _stencil(nx: int, ny: int, nz: int, offsets) -> Graph:
    n = nx * ny * nz
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    x, y, z = x.ravel(), y.ravel(), z.ravel()
    ids = np.arange(n, dtype=np.int64)
    cols_per_off, valid_per_off = [], []
    for dz, dy, dx in offsets:
        X, Y, Z = x + dx, y + dy, z + dz
        ok = (X >= 0) & (X < nx) & (Y >= 0) & (Y < ny) & (Z >= 0) & (Z < nz)
        valid_per_off.append(ok)
        cols_per_off.append(ids + (dz * ny + dy) * nx + dx)
    valid = np.stack(valid_per_off, axis=1)          # n x k, row-major = row then offset order
    cols = np.stack(cols_per_off, axis=1)
    deg = valid.sum(axis=1)
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=offs[1:])
    col_idx = cols[valid].astype(np.int32)
    return Graph(offs, col_idx)


def grid2d(w: int, h: int) -> Graph:
    """grid2d_graph (generators.cpp:126-137): 5-point grid, id = y*w + x."""
    return _stencil(w, h, 1, [(0, -1, 0), (0, 0, -1), (0, 0, 1), (0, 1, 0)])


def stencil3d(nx: int, ny: int, nz: int, points: int = 27) -> Graph:
    """stencil3d_graph (generators.cpp:139-162): 7- or 27-point box stencil."""
    if points not in (7, 27):
        raise ValueError("stencil3d: stencil must be 7 or 27")
    offs = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if dx == dy == dz == 0:
                    continue
                if points == 7 and abs(dx) + abs(dy) + abs(dz) != 1:
                    continue
                offs.append((dz, dy, dx))
    return _stencil(nx, ny, nz, offs)


def graph_from_edges(n: int, edges) -> Graph:
    """graph_from_edges (graph.cpp:66-81): both directions, self-loops dropped,
    duplicates collapsed, unit costs."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    e = e[e[:, 0] != e[:, 1]]
    rows = np.concatenate([e[:, 0], e[:, 1]])
    cols = np.concatenate([e[:, 1], e[:, 0]])
    return _csr_from_pairs(n, rows, cols)


def _csr_from_pairs(n: int, rows: np.ndarray, cols: np.ndarray) -> Graph:
    key = np.unique(rows.astype(np.int64) * n + cols.astype(np.int64))
    r = key // n
    c = (key % n).astype(np.int32)
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=offs[1:])
    return Graph(offs, c)


def ring(n: int) -> Graph:
    return graph_from_edges(n, [(i, (i + 1) % n) for i in range(n)])


def path(n: int) -> Graph:
    return graph_from_edges(n, [(i, i + 1) for i in range(n - 1)])


def symmetrize_pattern(n: int, rows: np.ndarray, cols: np.ndarray) -> Graph:
    """symmetrize (graph.cpp:44-64): pattern of A + A^T, diagonal dropped."""
    keep = rows != cols
    rows, cols = rows[keep], cols[keep]
    return _csr_from_pairs(n, np.concatenate([rows, cols]), np.concatenate([cols, rows]))


def largest_connected_component(g: Graph):
    """largest_connected_component (graph.cpp:118-171): ties -> component holding
    the smallest vertex id; vertices keep their relative order."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components

    n = g.n
    A = csr_matrix((np.ones(g.col_indices.shape[0], dtype=np.int8), g.col_indices, g.row_offsets), shape=(n, n))
    ncomp, labels = connected_components(A, directed=False)
    sizes = np.bincount(labels, minlength=ncomp)
    # smallest vertex id of each component
    first = np.full(ncomp, n, dtype=np.int64)
    np.minimum.at(first, labels, np.arange(n))
    best = max(range(ncomp), key=lambda c: (sizes[c], -first[c]))
    old = np.flatnonzero(labels == best).astype(np.int64)
    new_id = np.full(n, -1, dtype=np.int64)
    new_id[old] = np.arange(old.shape[0])
    deg = np.diff(g.row_offsets)[old]
    offs = np.zeros(old.shape[0] + 1, dtype=np.int64)
    np.cumsum(deg, out=offs[1:])
    starts = g.row_offsets[old]
    idx = np.repeat(starts - offs[:-1], deg) + np.arange(offs[-1])
    cols = new_id[g.col_indices[idx]].astype(np.int32)
    return Graph(offs, cols), old


def rmat_edges(scale: int, edgefactor: int = 16, seed: int = 1, a=0.57, b=0.19, c=0.19):
    """Graph500 Kronecker edge list with a random relabel of the 2^scale vertices."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = edgefactor * n
    ab, c_norm, a_norm = a + b, c / (1.0 - (a + b)), a / (a + b)
    src = np.zeros(m, dtype=np.int64)
    dst = np.zeros(m, dtype=np.int64)
    chunk = 1 << 24
    for lo in range(0, m, chunk):
        hi = min(m, lo + chunk)
        s = np.zeros(hi - lo, dtype=np.int64)
        d = np.zeros(hi - lo, dtype=np.int64)
        for bit in range(scale):
            ii = rng.random(hi - lo) > ab
            jj = rng.random(hi - lo) > np.where(ii, c_norm, a_norm)
            s |= ii.astype(np.int64) << bit
            d |= jj.astype(np.int64) << bit
        src[lo:hi], dst[lo:hi] = s, d
    perm = rng.permutation(n)
    return n, perm[src], perm[dst]


def rmat(scale: int, edgefactor: int = 16, seed: int = 1):
    """R-MAT graph after symmetrize + LCC. Returns (Graph, original_ids)."""
    n, s, d = rmat_edges(scale, edgefactor, seed)
    g = symmetrize_pattern(n, s, d)
    return largest_connected_component(g)


def random_connected_graph(n: int, extra: int, seed: int) -> Graph:
    """Spanning tree plus random extra edges (tests/test_support.hpp:53-72 shape)."""
    rng = np.random.default_rng(seed)
    order = rng.permutation(n)
    edges = [(order[i], order[rng.integers(0, i)]) for i in range(1, n)]
    for _ in range(extra):
        edges.append((rng.integers(0, n), rng.integers(0, n)))
    return graph_from_edges(n, edges)
