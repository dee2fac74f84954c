"""Regenerates tests/golden/golden.npz from the compiled reference (oracle/_ref).

Run in the build container (needs /root/reference to have built oracle/_ref):
    python tests/golden/make_golden.py
The fixtures pin the C restatement (oracle/specpart_oracle.c) and the host
logic on machines without the reference, and are the known-answer vectors the
GPU tests compare against at small sizes. Inputs are deterministic (fixed seeds).
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.ref import RefLib  # noqa: E402
from paper_2105_00578_b200 import RunConfig  # noqa: E402
from paper_2105_00578_b200 import generators as gen  # noqa: E402
from paper_2105_00578_b200.api import Graph  # noqa: E402


def weighted(g, seed):
    rng = np.random.default_rng(seed)
    n = g.n
    rows = np.repeat(np.arange(n), np.diff(g.row_offsets))
    key = np.minimum(rows, g.col_indices) * n + np.maximum(rows, g.col_indices)
    _, inv = np.unique(key, return_inverse=True)
    return Graph(g.row_offsets, g.col_indices, rng.uniform(0.5, 3.0, inv.max() + 1)[inv], None)


def graphs():
    return {
        "path3": gen.path(3),
        "k3": gen.graph_from_edges(3, [(0, 1), (1, 2), (0, 2)]),
        "star4": gen.graph_from_edges(4, [(0, 1), (0, 2), (0, 3)]),
        "wpath3": Graph([0, 1, 3, 4], [1, 0, 2, 1], [2.0, 2.0, 5.0, 5.0], None),  # laplacian_test.cpp:173-211
        "grid6x5": gen.grid2d(6, 5),
        "st7_4": gen.stencil3d(4, 4, 3, 7),
        "st27_3": gen.stencil3d(3, 3, 3, 27),
        "rand40": gen.random_connected_graph(40, 80, seed=11),
        "wrand30": weighted(gen.random_connected_graph(30, 50, seed=12), 3),
    }


def main():
    ref = RefLib()
    assert ref.kind == "reference", "golden fixtures must come from the compiled reference"
    out = {}
    for name, g in graphs().items():
        out[f"{name}/offs"] = g.row_offsets
        out[f"{name}/cols"] = g.col_indices
        if g.values is not None:
            out[f"{name}/vals"] = g.values
        for kind in ("combinatorial", "normalized", "degree"):
            L = ref.build_laplacian(kind, g)
            for k in ("row_offsets", "col_indices", "values", "diag"):
                out[f"{name}/{kind}/{k}"] = L[k]
            out[f"{name}/{kind}/bound"] = np.array([L["spectral_bound"]])
            out[f"{name}/{kind}/is_diagonal"] = np.array([int(L["is_diagonal"])])
        X = np.random.default_rng(5).uniform(-1, 1, (g.n, 3))
        out[f"{name}/X"] = X
        for kind in ("combinatorial", "normalized"):
            out[f"{name}/spmm_{kind}"] = np.asarray(ref.spmm(kind, g, X))
        a = np.random.default_rng(7).integers(0, 3, g.n).astype(np.int32)
        a[:3] = [0, 1, 2]
        p = ref.make_partition(g, a, 3, False)
        out[f"{name}/assignment"] = a
        out[f"{name}/cut"] = np.array([p.cutsize])
        out[f"{name}/imbalance"] = np.array([p.imbalance])
        out[f"{name}/part_weights"] = p.part_weights
    # initial blocks (eigensolver.cpp:20-51)
    out["init/random_50_3_42"] = np.asarray(ref.initial_guess("random", 50, 3, 42))
    out["init/random_17_5_7"] = np.asarray(ref.initial_guess("random", 17, 5, 7))
    out["init/piecewise_11_4"] = np.asarray(ref.initial_guess("piecewise", 11, 4))
    # MJ (partitioner.cpp:140-170)
    rng = np.random.default_rng(15)
    for t in range(6):
        n = int(rng.integers(5, 200))
        k = int(rng.integers(2, min(n, 40)))
        dims = int(rng.integers(1, 5))
        coords = np.round(rng.uniform(-1, 1, (n, dims)), 2)
        w = rng.uniform(0.5, 2.0, n) if t % 2 else None
        p = ref.mj_partition(coords, w, k)
        out[f"mj{t}/coords"] = coords
        if w is not None:
            out[f"mj{t}/weights"] = w
        out[f"mj{t}/K"] = np.array([k])
        out[f"mj{t}/assignment"] = p.assignment
    # sym_eig (dense.cpp:29-84)
    A = np.random.default_rng(3).standard_normal((7, 7))
    A = A + A.T
    vals, vecs = ref.sym_eig(A)
    out["symeig/A"], out["symeig/values"], out["symeig/vectors"] = A, vals, np.asarray(vecs)
    # LOBPCG and pipeline KATs
    g = gen.random_connected_graph(40, 80, seed=23)
    X0 = np.asarray(ref.initial_guess("random", g.n, 4, 11))
    for problem in ("combinatorial", "generalized", "normalized"):
        r = ref.lobpcg(g, problem, "jacobi", X0, 1e-8, 1000)
        out[f"lobpcg/{problem}/theta"] = r.theta
        out[f"lobpcg/{problem}/iterations"] = np.array([r.iterations])
    out["lobpcg/offs"], out["lobpcg/cols"], out["lobpcg/X0"] = g.row_offsets, g.col_indices, X0
    for name, g, cfg in [("grid16", gen.grid2d(16, 16), RunConfig(num_parts=4, precond="jacobi", seed=42)),
                         ("st7_8", gen.stencil3d(8, 8, 8, 7), RunConfig(num_parts=8, precond="polynomial", seed=42)),
                         ("ring8", gen.ring(8), RunConfig(num_parts=2, precond="jacobi", tol=1e-6, seed=5))]:
        r = ref.partition_graph(g, cfg)
        out[f"pipe/{name}/assignment"] = r.partition.assignment
        out[f"pipe/{name}/cut"] = np.array([r.report.cutsize])
        out[f"pipe/{name}/iterations"] = np.array([r.report.iterations])
        out[f"pipe/{name}/theta"] = np.array(r.report.theta)
    np.savez_compressed(Path(__file__).with_name("golden.npz"), **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
