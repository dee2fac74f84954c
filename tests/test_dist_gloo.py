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


# ---- the halo plan of csrc/halo.cu, restated on the host and run over gloo -------------
def _halo_plan(offs, cols, n, world, rank):
    """localize_operator (halo.cu:1-17): own rows [row0, row0+nloc); the foreign columns in
    ascending id (hence grouped by owner); columns rewritten to local ids (own j -> j-row0,
    halo j -> base + slot, base = nloc rounded up to 32 rows after the zero row); dpos[i] =
    stored columns with global id < global i (where build_combinatorial splices the diagonal)."""
    import numpy as np
    r0, nl = row_partition(n, world)[rank]
    k0, k1 = offs[r0], offs[r0 + nl]
    lc = cols[k0:k1].astype(np.int64)
    foreign = (lc < r0) | (lc >= r0 + nl)
    halo = np.unique(lc[foreign])
    base = ((nl + 1 + 31) // 32) * 32
    loc = np.where(foreign, base + np.searchsorted(halo, lc), lc - r0)
    rows = np.repeat(np.arange(nl), np.diff(offs[r0:r0 + nl + 1]))
    dpos = np.bincount(rows, weights=(lc < (r0 + rows)), minlength=nl).astype(np.int64)
    return r0, nl, offs[r0:r0 + nl + 1] - k0, loc, halo, base, dpos


def _spmv_worker(rank, world, port, q):
    import numpy as np
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_00578_b200 import generators as gen
        g = gen.rmat(10, 8, seed=11)[0]
        n, offs, cols = g.n, g.row_offsets, g.col_indices
        deg = np.diff(offs).astype(np.float64)
        X = np.random.default_rng(5).integers(-9, 10, (n, 3)).astype(np.float64)
        r0, nl, loffs, loc, halo, base, dpos = _halo_plan(offs, cols, n, world, rank)
        # halo id lists go to their owners (all-gathered here), which become the send lists
        lists = [None] * world
        dist.all_gather_object(lists, halo.tolist())
        n_pad = (n + world - 1) // world
        send = {p: [j - r0 for j in lists[p] if r0 <= j < r0 + nl] for p in range(world) if p != rank}
        # one exchange round: pack the rows each peer needs, receive the halo rows in list order
        packs = [None] * world
        dist.all_gather_object(packs, {p: X[r0 + np.asarray(s, dtype=np.int64)].tolist() for p, s in send.items()})
        Xl = np.zeros((base + halo.size, 3))
        Xl[:nl] = X[r0:r0 + nl]
        got = []
        for p in range(world):
            if p != rank and packs[p].get(rank):
                got.extend(packs[p][rank])
        Xl[base:] = np.asarray(got).reshape(-1, 3)
        assert np.all(halo // n_pad != rank)
        # L_C rows in storage order: -x_j, the diagonal at slot dpos (laplacian.cpp:53-79)
        Y = np.zeros((nl, 3))
        for i in range(nl):
            acc = np.zeros(3)
            ks = range(loffs[i], loffs[i + 1])
            for t, k in enumerate(ks):
                if t == dpos[i]:
                    acc = acc + deg[r0 + i] * Xl[i]
                acc = acc - Xl[loc[k]]
            if dpos[i] == len(ks):
                acc = acc + deg[r0 + i] * Xl[i]
            Y[i] = acc
        ys = [None] * world
        dist.all_gather_object(ys, Y.tolist())
        q.put((rank, np.concatenate([np.asarray(y).reshape(-1, 3) for y in ys]).tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_plan_row_partitioned_spmv_is_exact(world):
    import numpy as np
    from paper_2105_00578_b200 import generators as gen
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spmv_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = gen.rmat(10, 8, seed=11)[0]
    X = np.random.default_rng(5).integers(-9, 10, (g.n, 3)).astype(np.float64)
    deg = np.diff(g.row_offsets).astype(np.float64)
    rows = np.repeat(np.arange(g.n), np.diff(g.row_offsets))
    Y = deg[:, None] * X
    np.subtract.at(Y, rows, X[g.col_indices])
    for r in range(world):
        assert got[r] == got[0]
    assert np.frombuffer(got[0]).reshape(-1, 3).tobytes() == Y.tobytes()


# ---- the two-plane slab halo of the two-step polynomial kernel (Solver ctor, csrc/solver.cu) ----
def _slab_ce2(nx, ny, nz, world, rank, rows_cap):
    """Copy plan of rank `rank`: (peer, src_row, dst_row, rows); the four-plane region starts at
    h2 = rows_cap rounded up to 32 rows, the same on every rank: [z0-2, z0-1 | z1, z1+1]."""
    P = nx * ny
    r0, nl = row_partition(nx * ny * nz, world)[rank]
    h2 = (rows_cap + 31) // 32 * 32
    segs = []
    if r0 > 0:
        segs.append((rank - 1, 0, h2 + 2 * P, 2 * P))
    if r0 + nl < nx * ny * nz:
        segs.append((rank + 1, nl - 2 * P, h2, 2 * P))
    return segs, h2


@pytest.mark.parametrize("nz,world", [(16, 2), (16, 4), (32, 8), (128, 8), (12, 3)])
def test_slab_two_plane_halo_lands_on_the_right_planes(nz, world):
    import numpy as np
    nx, ny = 8, 6
    P = nx * ny
    n = nx * ny * nz
    rows_cap = max(nl for _, nl in row_partition(n, world)) + 2 * P + 32
    # every rank's block as global row ids (own rows, then the 4-plane region), filled by the plan
    blocks = []
    for r in range(world):
        r0, nl = row_partition(n, world)[r]
        b = np.full((rows_cap + 31) // 32 * 32 + 4 * P, -1, dtype=np.int64)
        b[:nl] = np.arange(r0, r0 + nl)
        blocks.append(b)
    for r in range(world):
        segs, h2 = _slab_ce2(nx, ny, nz, world, r, rows_cap)
        for peer, src, dst, rows in segs:
            blocks[peer][dst:dst + rows] = blocks[r][src:src + rows]
    for r in range(world):
        r0, nl = row_partition(n, world)[r]
        h2 = (rows_cap + 31) // 32 * 32
        lo, hi = blocks[r][h2:h2 + 2 * P], blocks[r][h2 + 2 * P:h2 + 4 * P]
        if r0 > 0:
            assert np.array_equal(lo, np.arange(r0 - 2 * P, r0))           # planes z0-2, z0-1
        if r0 + nl < n:
            assert np.array_equal(hi, np.arange(r0 + nl, r0 + nl + 2 * P))  # planes z1, z1+1
