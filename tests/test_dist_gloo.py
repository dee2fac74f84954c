"""CPU, world_size 2 over gloo: the host-side multi-GPU plumbing (NCCL id exchange,
row partition). The data-path collectives themselves run on GPUs (tests/test_gpu_dist.py)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_00578_b200.dist import row_partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_00578_b200.api import Context
        try:
            nid = Context.nccl_unique_id() if rank == 0 else None
        except Exception:  # NCCL absent on this host: ship a stand-in id
            nid = bytes(range(128)) if rank == 0 else None
        obj = [nid]
        dist.broadcast_object_list(obj, src=0)
        q.put((rank, obj[0]))
    finally:
        dist.destroy_process_group()


def test_nccl_id_reaches_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(got[0]) == 128 and got[0] == got[1]


@pytest.mark.parametrize("n,world", [(10, 2), (11, 2), (2097152, 8), (7, 8), (1, 4), (8862726, 8)])
def test_row_partition_covers_rows_once(n, world):
    parts = row_partition(n, world)
    covered = []
    for r0, nl in parts:
        covered.extend(range(r0, r0 + nl)) if n < 100 else covered.append((r0, nl))
    if n < 100:
        assert covered == list(range(n))
    else:
        assert sum(nl for _, nl in parts) == n
        assert all(parts[k][0] == k * ((n + world - 1) // world) for k in range(world))
