"""Diagnostic (not a test): profile one partition of a BASELINE config with SPB_PROFILE=1."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("SPB_PROFILE", "1")

import bench  # noqa: E402
from paper_2105_00578_b200 import Context  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
c = bench.CONFIGS[cfgname]
t = time.time()
g = bench.make_graph(c["gen"])
print(f"graph {cfgname}: n={g.n} nnz={g.row_offsets[-1]} gen {time.time()-t:.1f}s", flush=True)
ctx = Context(0)
ctx.set_timing(True)
dg = ctx.upload(g)
for i in range(2):
    r = ctx.partition_resident(dg, bench.run_config(c), copy_assignment=False)
    rep = r.report
    print(f"run {i}: total {rep.times['total_s']:.4f}s iters {rep.iterations} cut {rep.cutsize} imb {rep.imbalance}"
          f" spmm {rep.device['spmm_launches']} launches {rep.device['spmm_ms']:.2f} ms "
          f"{rep.device['spmm_bytes']/max(rep.device['spmm_ms'],1e-9)/1e6:.1f} GB/s  kernels {rep.device['kernel_launches']}",
          flush=True)
