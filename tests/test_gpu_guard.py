"""GPU memory-safety check without compute-sanitizer (closed on the B200 pool): every kernel
family runs in a process with SPECPART_B200_GUARD=1, where each device buffer is bracketed by
64 KiB guard bands verified on release (csrc/guard.cu); an out-of-bounds store anywhere in the
pool shows up as changed guard bytes. The run must finish cleanly with zero such bytes."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent


def test_guard_bands_intact_over_every_kernel_family():
    env = dict(os.environ, SPECPART_B200_GUARD="1")
    r = subprocess.run([sys.executable, str(HERE / "guard_workload.py")], capture_output=True, text=True,
                       timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["status"] == 0 and out["violations"] == 0, (out, r.stderr[-3000:])
    assert out["buffers"] > 500, out
    assert "guard]" not in r.stderr, r.stderr[-3000:]


def test_guard_mode_is_off_by_default(ctx):
    import ctypes as C
    v, b = C.c_int64(), C.c_int64()
    assert ctx.lib.sp_debug_guard_check(C.byref(v), C.byref(b)) == 0
    assert v.value == -1 and b.value == -1
