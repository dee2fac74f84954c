"""Run by tests/test_gpu_kernels.py::test_two_step_polynomial_kernel_bit_identical in two processes
(SPB_POLY2=0 and default): the polynomial preconditioner on meshes, outputs written as raw bytes."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_00578_b200 import Context  # noqa: E402
from paper_2105_00578_b200 import generators as gen  # noqa: E402

ctx = Context(0)
out = []
for g, m in ((gen.stencil3d(40, 36, 20, 7), 7), (gen.stencil3d(33, 30, 17, 7), 3), (gen.grid2d(70, 66), 5)):
    R = np.random.default_rng(g.n).uniform(-1, 1, (g.n, m))
    for degree in (25, 6, 3):
        H = ctx.precond_apply("combinatorial", g, "polynomial", R, seed=5, degree=degree)
        out.append(H.tobytes())
Path(sys.argv[1]).write_bytes(b"".join(out))
