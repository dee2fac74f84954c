"""Diagnostic (not a test): device time of the tall-skinny block kernel per LOBPCG shape."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_00578_b200 import Context  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 21
m = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ctx = Context(0)
# (name, mu, mv, mw, transform, gram, columns read, columns written)
shapes = [
    ("orth_g0 [X|H]^T H", 2 * m, m, 0, 0, 1, 3 * m, 0),
    ("orth_p1 H-XC, X^T W", 2 * m, m, 0, 1, 2, 3 * m, m),
    ("orth_p2 W-XC, W^T W", 2 * m, m, 0, 1, 3, 3 * m, m),
    ("orth_cb WT, Gram", 0, m, m, 2, 3, m, m),
    ("rr_gram S^T AS", 3 * m, 3 * m, 0, 0, 2, 6 * m, 0),
    ("combine S Y", 0, 3 * m, 2 * m, 2, 0, 3 * m, 2 * m),
    ("arnoldi V^T w", 24, 1, 0, 0, 2, 25, 0),
    ("arnoldi w - V h, w^T w", 24, 1, 0, 1, 3, 25, 1),
]
if len(sys.argv) > 3 and sys.argv[3] == "micro":
    shapes = [
        ("self 1x1", 0, 1, 0, 0, 3, 1, 0),
        ("self 8x8", 0, 8, 0, 0, 3, 8, 0),
        ("self 16x16", 0, 16, 0, 0, 3, 16, 0),
        ("U32^T v", 32, 1, 0, 0, 2, 33, 0),
        ("combine 8->8", 0, 8, 8, 2, 0, 8, 8),
        ("combine 2->2", 0, 2, 2, 2, 0, 2, 2),
        ("combine 16->16", 0, 16, 16, 2, 0, 16, 16),
    ]
out = []
for name, mu, mv, mw, tr, gr, rd, wr in shapes:
    ms = C.c_double()
    ctx._check(ctx.lib.sp_bench_blockop(ctx._h, n, mu, mv, mw, tr, gr, 20, C.byref(ms)))
    gbs = (rd + wr) * n * 8 / (ms.value * 1e-3) / 1e9
    out.append(dict(shape=name, us=round(ms.value * 1e3, 1), gbs=round(gbs)))
    print(f"{name:28s} {ms.value * 1e3:8.1f} us  {gbs:7.0f} GB/s", flush=True)
print("BLOCKOPS " + json.dumps(out))
