"""GPU: the shuffle path of the pattern-compressed ELL SpMM (ell_uniform_rows in csrc/spmm.cu)
is bit-identical to the per-slot gather path (SPB_ELL_SHFL=0): the GMRES-polynomial apply (whose
Arnoldi and product steps run through the solver's ELL SpMM) and a full partition give the same
bytes both ways, on meshes wide enough (nx >= 64) to have uniform interior tiles, and match the
reference (preconditioners.cpp:171-193, 315-382) within the polynomial tolerance."""
import hashlib
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2105_00578_b200 import generators as gen

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2105_00578_b200 import Context, generators as gen
from paper_2105_00578_b200.api import RunConfig
ctx = Context(0)
out = {}
for name, g in [("st27", gen.stencil3d(96, 7, 6, 27)), ("st7", gen.stencil3d(64, 9, 7, 7)),
                ("grid", gen.grid2d(128, 40))]:
    R = np.random.default_rng(1).uniform(-1, 1, (g.n, 5))
    H, roots = ctx.poly_apply("combinatorial", g, 42, 25, R)
    out[name + "_poly"] = hashlib.sha256(np.ascontiguousarray(H).tobytes()).hexdigest()
    r = ctx.partition_graph(g, RunConfig(num_parts=8, precond="polynomial", seed=42))
    out[name + "_part"] = hashlib.sha256(np.asarray(r.partition.assignment).tobytes()).hexdigest()
    out[name + "_theta"] = [float(t) for t in r.report.theta]
print(json.dumps(out))
"""


def _run(shfl):
    env = dict(os.environ, SPB_ELL_SHFL=str(shfl))
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_shuffle_path_bit_identical():
    a, b = _run(0), _run(1)
    assert a == b


@pytest.mark.gpu
def test_shuffle_path_27pt_poly_matches_reference(ctx, ref):
    g = gen.stencil3d(96, 7, 6, 27)
    R = np.random.default_rng(1).uniform(-1, 1, (g.n, 5))
    H, roots = ctx.poly_apply("combinatorial", g, 42, 25, R)
    Hr, deg = ref.poly_apply("combinatorial", g, 42, 25, R)
    assert len(roots) == deg == 25
    np.testing.assert_allclose(H, Hr, rtol=1e-7, atol=1e-9 * np.abs(Hr).max())
