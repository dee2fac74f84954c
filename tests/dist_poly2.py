"""Run under torchrun by tests/test_gpu_dist.py::test_slab_two_step_kernel_bit_identical: row-partitioned
polynomial partitions of 7-point meshes; rank 0 prints the eigenvalues (hex) and the assignment hash, which
must not depend on SPB_POLY2 (two polynomial steps per slab launch vs one)."""
import hashlib
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch.distributed as dist  # noqa: E402

from paper_2105_00578_b200 import RunConfig  # noqa: E402
from paper_2105_00578_b200 import generators as gen  # noqa: E402
from paper_2105_00578_b200.dist import create_context  # noqa: E402


def main():
    dist.init_process_group("gloo")
    ctx = create_context()
    out = {}
    for name, g, cfg in (("st7_32", gen.stencil3d(32, 32, 32, 7), RunConfig(num_parts=16, precond="polynomial", seed=7)),
                         ("st7_24x40", gen.stencil3d(24, 40, 16, 7), RunConfig(num_parts=8, precond="polynomial", seed=3))):
        r = ctx.partition_graph(g, cfg)
        out[name] = dict(theta=[float(t).hex() for t in r.report.theta], iterations=r.report.iterations,
                         assignment=hashlib.sha1(r.partition.assignment.tobytes()).hexdigest(),
                         mesh_launches=r.report.device["mesh_launches"], poly_launches=r.report.device["poly_launches"])
    if dist.get_rank() == 0:
        print("POLY2_RESULT " + json.dumps(out), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
