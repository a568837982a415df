"""Host logic of the row-slab decomposition on CPU: the slab plan, and the
torch.distributed halo exchange + all-reduce with world size 2 and 3 over gloo (CPU
tensors), checked against the rows the neighbours own."""
import os
import socket

import numpy as np
import pytest
import torch

from paper_2306_15049_b200.slab import SlabPlan


def test_plan_partition_and_halos():
    p = SlabPlan(4096, 4096, 10, 8)
    assert [s.row0 for s in p.slabs] == [512 * k for k in range(8)]
    assert p.slabs[0].top == 0 and p.slabs[-1].bot == 0
    for s in p.slabs[1:-1]:
        assert s.top == 20 and s.bot == 20 and s.ext_rows == 512 + 40
    q = SlabPlan(37, 8, 2, 3)          # ragged: 13, 12, 12 rows
    assert [s.own_rows for s in q.slabs] == [13, 12, 12]
    assert q.slabs[0].ext1 == 17 and q.slabs[2].ext0 == 21
    with pytest.raises(ValueError):
        SlabPlan(16, 16, 4, 4)          # 4-row slabs < halo 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ny, nx, r, q):
    import torch.distributed as dist
    from paper_2306_15049_b200.slab import DistComm, SlabPlan
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = SlabPlan(ny, nx, r, world)
        comm = DistComm(plan, rank)
        full = torch.arange(3 * ny * nx, dtype=torch.float64).reshape(3, ny * nx)
        T = plan.extend(full, rank)
        s = plan.slabs[rank]
        T[:, :s.top * nx] = -1.0
        T[:, (s.top + s.own_rows) * nx:] = -1.0
        comm.halo(T)
        ok_halo = bool(torch.equal(T, plan.extend(full, rank)))
        t = torch.tensor([float(rank + 1), 2.0 * rank], dtype=torch.float64)
        comm.allreduce(t)
        m = torch.tensor([float((rank * 7) % 5), -float(rank)], dtype=torch.float64)
        comm.allreduce(m, op="max")
        q.put((rank, ok_halo, t.tolist() + m.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_halo_and_allreduce_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(k, world, port, 30, 7, 2, q)) for k in range(world)]
    for p in ps:
        p.start()
    res = dict((r, (h, t)) for r, h, t in (q.get(timeout=120) for _ in ps))
    for p in ps:
        p.join(timeout=60)
    want = [sum(k + 1 for k in range(world)), sum(2.0 * k for k in range(world)),
            max(float((k * 7) % 5) for k in range(world)), 0.0]
    for k in range(world):
        assert res[k][0], f"rank {k}: halo rows differ from the neighbours' owned rows"
        assert res[k][1] == want
