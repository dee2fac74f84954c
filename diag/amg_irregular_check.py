"""Diagnostic: LOBPCG on an irregular graph (generalized problem) with jacobi / amg / none,
device vs the reference; AMG apply vs the reference's."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle.ref import RefLib  # noqa: E402
from paper_2105_00578_b200 import Context  # noqa: E402
from paper_2105_00578_b200 import generators as gen  # noqa: E402

ctx, ref = Context(0), RefLib()
g, _ = gen.rmat(13, 16, seed=7)
X0 = ctx.initial_guess("piecewise", g.n, 4, 0)
for prob in ("generalized", "combinatorial", "normalized"):
    for pc in ("jacobi", "amg", "none"):
        a = ctx.lobpcg(g, prob, pc, X0, 1e-2, max_iters=400, poly_seed=5)
        b = ref.lobpcg(g, prob, pc, X0, 1e-2, max_iters=400, poly_seed=5)
        print(prob, pc, "gpu", a.iterations, a.converged.tolist(), np.round(a.theta, 6).tolist(), "| ref", b.iterations,
              b.converged.tolist(), np.round(b.theta, 6).tolist(), flush=True)
R = np.random.default_rng(3).uniform(-1, 1, (g.n, 4))
H, Hr = ctx.precond_apply("combinatorial", g, "amg", R, seed=5), ref.precond_apply("combinatorial", g, "amg", R, seed=5)
print("amg apply rel diff", np.max(np.abs(H - Hr)) / np.max(np.abs(Hr)))
for k in (1, 2, 3):
    H = ctx.precond_apply("combinatorial", g, "amg", R[:, :k], seed=5)
    Hr = ref.precond_apply("combinatorial", g, "amg", R[:, :k], seed=5)
    print("k", k, "amg apply rel diff", np.max(np.abs(H - Hr)) / np.max(np.abs(Hr)))
