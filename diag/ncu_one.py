"""Diagnostic (not a test): one warm-up + one profiled partition for ncu launch lists."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2105_00578_b200 import Context  # noqa: E402

c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
g = bench.make_graph(c["gen"])
ctx = Context(0)
dg = ctx.upload(g)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for _ in range(reps):
    r = ctx.partition_resident(dg, bench.run_config(c), copy_assignment=False)
print("launches per partition", r.report.device["kernel_launches"], "total", r.report.times["total_s"])
