"""Shift-sharded nested solve on the GPU: a 2-rank run (gloo process
group, both ranks on cuda:0 -- no kernel waits on another rank) reproduces the
single-rank solutions, iteration counts and L-curve corners bit for bit."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(cfgname, dist_on):
    import torch
    import rsk_synth as S
    from paper_2306_15049_b200 import shard
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = S.CONFIGS[cfgname]
    inp = S.make_inputs(cfg)
    dev = torch.device("cuda", 0)
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"], device=0, check_every=4, dist=shard.Dist(dist_on))
    sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
    outs = sol.run()
    return (sol.final["X_prev"].cpu().numpy(), [o.iters.copy() for o in outs], [o.lstar for o in outs])


def _worker(rank, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        q.put((rank, _run("C1", True)))
    finally:
        dist.destroy_process_group()


def test_two_rank_shift_sharding_is_bitwise_single_rank():
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    X1, it1, ls1 = _run("C1", False)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    for r in (0, 1):
        X2, it2, ls2 = res[r]
        assert ls2 == ls1
        for a, b in zip(it1, it2):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(X1, X2)
