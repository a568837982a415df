"""Shift-sharded nested solve on the GPU: a 2-rank run (gloo process
group, both ranks on cuda:0 -- no kernel waits on another rank) reproduces the
single-rank solutions, iteration counts and L-curve corners bit for bit: with the
cluster-per-shift loop (C1) and with the streaming lockstep loop that C3-C5 run (C2
forced onto it), whose p.w partials and U^T V chunks are batch-composition invariant
(DESIGN.md §4.2)."""
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
    kinds = sorted({int(o.prof[7]) for o in outs if o.prof is not None})
    return (sol.final["X_prev"].cpu().numpy(), [o.iters.copy() for o in outs], [o.lstar for o in outs], kinds)


def _worker(rank, port, q, cfgname, env):
    import torch.distributed as dist
    os.environ.update(env)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        q.put((rank, _run(cfgname, True)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfgname,env", [("C1", {}),
                                         ("C2", {"RSK_CG_NOCLUSTER": "1", "RSK_CG_STREAM": "1"})])
def test_two_rank_shift_sharding_is_bitwise_single_rank(monkeypatch, cfgname, env):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    X1, it1, ls1, k1 = _run(cfgname, False)
    if env:
        assert k1 == [3], k1   # the streaming lockstep loop (cg_stream.cu) ran every inner solve
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, port, q, cfgname, env)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    for r in (0, 1):
        X2, it2, ls2, _ = res[r]
        assert ls2 == ls1
        for a, b in zip(it1, it2):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(X1, X2)
