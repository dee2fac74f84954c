"""Diagnostic: wall time of sp_initial_guess (random) at the cfg2 sizes."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_00578_b200 import Context  # noqa: E402

ctx = Context(0)
for n, d in ((2097152, 1), (2097152, 7), (262144, 1)):
    ctx.initial_guess("random", n, d, 42)
    t = time.perf_counter()
    for _ in range(5):
        ctx.initial_guess("random", n, d, 42)
    print(f"n={n} d={d}: {(time.perf_counter() - t) / 5 * 1e3:.3f} ms per call (incl. the D2H copy)", flush=True)
