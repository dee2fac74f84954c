"""Diagnostic: one block-kernel shape, for ncu (python tests/bench_one_blockop.py n mu mv mw transform gram)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_00578_b200 import Context  # noqa: E402

a = [int(x) for x in sys.argv[1:7]]
ctx = Context(0)
ms = C.c_double()
ctx._check(ctx.lib.sp_bench_blockop(ctx._h, a[0], a[1], a[2], a[3], a[4], a[5], 3, C.byref(ms)))
print("ms", ms.value)
