"""Multi-GPU check, launched by tests/test_gpu_dist.py under torchrun (one process
per GPU): row-sharded partitions vs the CPU reference, identical on every rank."""
import hashlib
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2105_00578_b200 import RunConfig  # noqa: E402
from paper_2105_00578_b200 import generators as gen  # noqa: E402
from paper_2105_00578_b200.dist import create_context  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    ctx = create_context()
    rg, _ = gen.largest_connected_component(gen.symmetrize_pattern(*gen.rmat_edges(12, 16, seed=3)))
    cases = [
        ("grid64_jacobi", gen.grid2d(64, 64), RunConfig(num_parts=4, precond="jacobi", seed=42)),
        ("st7_16_poly", gen.stencil3d(16, 16, 16, 7), RunConfig(num_parts=8, precond="polynomial", seed=42)),
        ("st27_12_gen_poly", gen.stencil3d(12, 12, 12, 27),
         RunConfig(num_parts=16, precond="polynomial", problem="generalized", seed=42)),
        ("rmat12_norm_jacobi", rg, RunConfig(num_parts=8, precond="jacobi", problem="normalized", seed=42)),
    ]
    out = {}
    for name, g, cfg in cases:
        r = ctx.partition_graph(g, cfg)
        h = hashlib.sha1(r.partition.assignment.tobytes()).hexdigest()
        hs = [None] * world
        dist.all_gather_object(hs, h)
        out[name] = dict(cut=r.report.cutsize, imbalance=r.report.imbalance, iterations=r.report.iterations,
                         same_on_all_ranks=len(set(hs)) == 1, theta=r.report.theta, n_gpus=r.report.device["n_gpus"])
    if rank == 0:
        from oracle.ref import RefLib
        ref = RefLib()
        for name, g, cfg in cases:
            b = ref.partition_graph(g, cfg)
            o = out[name]
            o.update(ref_cut=b.report.cutsize, ref_imbalance=b.report.imbalance, ref_iterations=b.report.iterations,
                     theta_maxdiff=float(np.max(np.abs(np.array(o["theta"]) - np.array(b.report.theta)))))
            o["ok"] = bool(o["same_on_all_ranks"] and abs(o["cut"] - o["ref_cut"]) <= 0.02 * o["ref_cut"]
                           and o["imbalance"] <= o["ref_imbalance"] + 1e-12 and o["n_gpus"] == world)
        print("DIST_RESULT " + json.dumps(out), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
