"""Multi-process (world size 2 and 3, gloo, CPU) checks of the N>1 host
logic: slab partition, halo plans (what one rank sends is what its
neighbour expects), the NCCL id bootstrap through torch.distributed, the
partition invariance of the seeded inputs, and bench.py's max-over-ranks
timing helper.  The device side of the NCCL path needs GPUs that are not
available here; its kernels are exercised on one GPU by the in-process slab
decomposition tests (tests/test_gpu_parity.py::test_slab_decomposition)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nz, spr, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import inputs
        import paper_2512_09642_b200 as sscg
        z0, nzl = sscg.partition(nz, world, spr, rank)
        plans = [sscg.halo_plan(nz, world, spr, rank, l) for l in range(spr)]
        parts = [None] * world
        dist.all_gather_object(parts, (z0, nzl, plans))
        # NCCL id bootstrap: rank 0 creates it, everyone receives the same bytes
        obj = [sscg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        # seeded inputs: each rank's slab equals the global slice
        nx, ny = 6, 5
        b_loc = inputs.rhs_uniform(nx, ny, nz, seed=42, z0=z0, nzl=nzl)
        gathered = [None] * world
        dist.all_gather_object(gathered, b_loc)
        # bench helper: device time is the max over ranks
        t = bench.max_over_ranks(dist, float(rank + 1) * 1.5, device="cpu")
        out_q.put((rank, parts, ids, gathered, t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nz,spr", [(2, 448 * 2, 1), (3, 100, 2), (2, 7, 3)])
def test_multirank_host_logic(world, nz, spr):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nz, spr, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    _, parts, ids, gathered, _ = res[0]
    # partition: contiguous, complete, every slab non-empty
    zs = [(z0, n) for z0, n, _ in parts]
    assert zs[0][0] == 0 and sum(n for _, n in zs) == nz
    for (a0, an), (b0, _) in zip(zs, zs[1:]):
        assert a0 + an == b0
    # halo plans: consistency between neighbours, Dirichlet at the ends
    slabs = [(r, l, pl) for r, (_, _, plans) in enumerate(parts) for l, pl in enumerate(plans)]
    assert slabs[0][2]["peer_lo"] == -1 and slabs[-1][2]["peer_hi"] == -1
    for (ra, la, a), (rb, lb, b) in zip(slabs, slabs[1:]):
        assert a["peer_hi"] == rb and b["peer_lo"] == ra
        assert a["send_hi_z"] == b["recv_lo_z"] and b["send_lo_z"] == a["recv_hi_z"]
        assert a["recv_hi_z"] == a["send_hi_z"] + 1 and b["recv_lo_z"] == b["send_lo_z"] - 1
    # identical NCCL id on every rank
    assert all(i == ids[0] for i in ids) and len(ids[0]) == 128
    # inputs are partition invariant
    import inputs
    full = inputs.rhs_uniform(6, 5, nz, seed=42)
    assert np.array_equal(np.concatenate(gathered), full)
    # max over ranks
    assert all(r[4] == pytest.approx(1.5 * world) for r in res)
