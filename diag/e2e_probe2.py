"""Diagnostic: repeated pinned e2e partitions (run with SPB_PROFILE=1 and an nvidia-smi poller)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2105_00578_b200 import Context  # noqa: E402
from paper_2105_00578_b200.api import Graph  # noqa: E402

c = bench.CONFIGS["cfg2"]
g = bench.make_graph(c["gen"])
ctx = Context(0)
gp = Graph(torch.from_numpy(g.row_offsets).pin_memory().numpy(), torch.from_numpy(g.col_indices).pin_memory().numpy())
out = torch.empty(g.n, dtype=torch.int32).pin_memory().numpy()
cfg = bench.run_config(c)
for i in range(25):
    t0 = time.perf_counter()
    r = ctx.partition_graph(gp, cfg, out=out)
    print(f"[probe] e2e {i} wall {1e3 * (time.perf_counter() - t0):8.1f} ms", file=sys.stderr, flush=True)
