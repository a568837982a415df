"""Host logic of shift sharding: assignment and the collectives, run
as world_size-2 gloo process groups on CPU (no GPU needed)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_15049_b200 import shard


def test_round_robin_and_lpt_cover_every_shift_once():
    for M, W in ((8, 2), (32, 3), (128, 8), (5, 8)):
        for owners in (shard.round_robin(M, W), shard.lpt_assign(np.arange(M)[::-1] * 7 % 11, W)):
            flat = sorted(l for o in owners for l in o)
            assert flat == list(range(M))
            assert len(owners) == W


def test_lpt_balances_iteration_costs():
    rng = np.random.default_rng(0)
    costs = np.exp(rng.uniform(0, 5, 128))          # spread ~150x like the shift ladder
    owners = shard.lpt_assign(costs, 8)
    loads = [sum(costs[l] + 1 for l in o) for o in owners]
    rr = [sum(costs[l] + 1 for l in o) for o in shard.round_robin(128, 8)]
    assert max(loads) <= max(rr)
    assert max(loads) <= (sum(costs) + 128) / 8 + max(costs) + 1   # LPT bound
    assert shard.lpt_assign(costs, 8) == owners                      # deterministic


def test_assignment_step0_round_robin_then_lpt():
    assert shard.assignment(0, 10, 2) == shard.round_robin(10, 2)
    it = np.array([5, 1, 1, 1, 1, 1, 1, 1, 1, 9])
    a1 = shard.assignment(1, 10, 2, it)
    assert a1 == shard.lpt_assign(it, 2)
    assert shard.assignment(3, 10, 1, it) == [list(range(10))]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = shard.Dist(True)
        M, N = 11, 6
        full = torch.arange(M * N, dtype=torch.float64).reshape(M, N)
        owners = shard.lpt_assign(np.arange(M) % 4, world)
        local = full[owners[rank]].clone()
        got = d.gather_rows(local, owners, M)
        ok1 = torch.equal(got, full)
        t = torch.full((3, 2), float(rank)) if rank == 0 else torch.zeros(3, 2)
        d.bcast(t)
        ok2 = bool(torch.all(t == 0.0))
        ok3 = d.bcast_int(42 if rank == 0 else -1, "cpu") == 42
        arr = d.gather_np(np.stack([np.array(owners[rank], float), np.ones(len(owners[rank])) * rank], 1),
                          owners, M, "cpu")
        ok4 = np.array_equal(arr[:, 0], np.arange(M)) and all(
            arr[l, 1] == r for r, o in enumerate(owners) for l in o)
        q.put((rank, ok1, ok2, ok3, ok4))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_broadcast():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(all(r[1:]) for r in res), res


def test_group_aware_assignment_keeps_groups_apart():
    """prefer group-pure GPUs, GPUs to groups in proportion to their work."""
    rng = np.random.default_rng(4)
    M, W = 128, 8
    groups = np.array([0 if l < 96 else 1 for l in range(M)])
    its = np.where(groups == 0, rng.integers(300, 1100, M), rng.integers(700, 20000, M))
    owners = shard.group_lpt_assign(its, groups, W)
    assert sorted(l for o in owners for l in o) == list(range(M)) and len(owners) == W
    assert all(len(set(groups[o].tolist())) == 1 for o in owners if o)       # group-pure
    nR = sum(1 for o in owners if o and groups[o[0]] == 1)
    costR = 80 * (its[groups == 1] + 1).sum()
    costL = 80 * (its[groups == 0] + 1).sum()
    assert nR >= round(W * costR / (costR + costL)) - 1 and nR >= 1
    assert shard.group_lpt_assign(its, groups, W) == owners                   # deterministic
    # fewer GPUs than groups: plain LPT
    assert shard.group_lpt_assign(its, groups, 1) == [list(range(M))]
    assert shard.assignment(1, M, W, its, groups=groups) == owners
