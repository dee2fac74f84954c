"""Diagnostic (not a test): phase profile of rank 0 under torchrun (SPB_PROFILE on rank 0 only)."""
import os
import sys
from pathlib import Path

if os.environ.get("RANK", "0") == "0":
    os.environ["SPB_PROFILE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2105_00578_b200.dist import create_context  # noqa: E402

dist.init_process_group("gloo")
c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
g = bench.make_graph(c["gen"])
ctx = create_context()
dg = ctx.upload(g)
for i in range(2):
    r = ctx.partition_resident(dg, bench.run_config(c), copy_assignment=False)
    if dist.get_rank() == 0:
        print(f"run {i}: total {r.report.times['total_s']:.4f}s iters {r.report.iterations} cut {r.report.cutsize}",
              flush=True)
ctx.close()
dist.destroy_process_group()
