"""Diagnostic: where the end-to-end (host CSR -> host assignment) time goes on cfg2."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2105_00578_b200 import Context  # noqa: E402
from paper_2105_00578_b200.api import Graph  # noqa: E402

c = bench.CONFIGS["cfg2"]
g = bench.make_graph(c["gen"])
ctx = Context(0)
offs_p = torch.from_numpy(g.row_offsets).pin_memory()
cols_p = torch.from_numpy(g.col_indices).pin_memory()
gp = Graph(offs_p.numpy(), cols_p.numpy())
print("pinned view shares memory:", gp.row_offsets.ctypes.data == offs_p.data_ptr())
cfg = bench.run_config(c)
dg = ctx.upload(gp)
for _ in range(3):
    ctx.partition_resident(dg, cfg, copy_assignment=False)
    ctx.partition_graph(gp, cfg)
for label, fn in [("resident", lambda: ctx.partition_resident(dg, cfg, copy_assignment=False)),
                  ("resident+asg", lambda: ctx.partition_resident(dg, cfg, copy_assignment=True)),
                  ("e2e pinned", lambda: ctx.partition_graph(gp, cfg)),
                  ("e2e pageable", lambda: ctx.partition_graph(g, cfg))]:
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        t1 = time.perf_counter()
        print(f"{label:14s} wall {1e3 * (t1 - t0):7.1f} ms  total_s {1e3 * r.report.times['total_s']:7.1f} ms", flush=True)
