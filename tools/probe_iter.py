"""Per-lockstep-iteration GPU time of the batched CG loop at 1..32 active shifts
(plain CG on the C2 data, every shift at the same gamma so all stay active)."""
import dataclasses
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import rsk_synth as S
from paper_2306_15049_b200.pipeline import GpuSolver

cfg0 = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
inp = S.make_inputs(cfg0)
dev = torch.device("cuda", 0)
for ns in (1, 2, 4, 8, 16, 32):
    cfg = dataclasses.replace(cfg0, M=ns, maxit=300, tol=1e-30)
    gam = np.full(ns, 1e-5)
    sol = GpuSolver(cfg, inp["psf"], gam, check_every=16)
    sol.reset_weights()
    sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
    X = torch.zeros(ns, cfg.N, dtype=torch.float64, device=dev)
    sol.cg(list(range(ns)), X, [0] * ns)            # warm
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = sol.cg(list(range(ns)), X, [0] * ns)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    it = int(res["iters"].max())
    print(f"{cfg.name} shifts={ns:3d}: {1e6*(t1-t0)/it:8.1f} us per lockstep iteration "
          f"({1e6*(t1-t0)/it/ns:7.2f} us per shift-iteration), iters {it}")
