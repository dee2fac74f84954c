"""GPU, N >= 2 (skipped on one GPU): the 1-D row-partitioned path over NCCL."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
# copy-engine halo + P2P sums (default), SM-issued halo pushes fused into the SpMM, NCCL fallback
@pytest.mark.parametrize("path", ["ce", "fused", "nccl"])
def test_row_partitioned_matches_reference(path):
    import os
    env = dict(os.environ, SPB_P2P="0" if path == "nccl" else "1", SPB_HALO_CE="0" if path == "fused" else "1")
    n = min(_ngpus(), 4)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "tests" / "dist_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(ROOT), env=env)
    line = [l for l in r.stdout.splitlines() if l.startswith("DIST_RESULT ")]
    assert r.returncode == 0 and line, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(line[0][len("DIST_RESULT "):])
    for name, o in res.items():
        assert o["ok"], (name, o)


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_slab_two_step_kernel_bit_identical():
    """On z-slabs the two-step polynomial kernel (two halo planes per side) gives the same eigenvalues,
    bit for bit, and the same assignment as one step per launch (SPB_POLY2=0), in half the launches."""
    import os
    n = min(_ngpus(), 4)
    res = []
    for val in ("0", "1"):
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "tests" / "dist_poly2.py")]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(ROOT),
                           env=dict(os.environ, SPB_POLY2=val))
        line = [l for l in r.stdout.splitlines() if l.startswith("POLY2_RESULT ")]
        assert r.returncode == 0 and line, r.stdout[-3000:] + r.stderr[-3000:]
        res.append(json.loads(line[0][len("POLY2_RESULT "):]))
    for name in res[0]:
        a, b = res[0][name], res[1][name]
        assert a["theta"] == b["theta"] and a["assignment"] == b["assignment"] and a["iterations"] == b["iterations"], name
        assert b["poly_launches"] < a["poly_launches"], (name, a["poly_launches"], b["poly_launches"])
