"""Latency probe: plain batched CG with NS identical shifts for a fixed number of lockstep
iterations (launch-list target for ncu). Usage: probe_one.py CFG NS ITERS"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import rsk_synth as S
from paper_2306_15049_b200.pipeline import GpuSolver

cfg0 = S.CONFIGS[sys.argv[1]]
ns, its = int(sys.argv[2]), int(sys.argv[3])
inp = S.make_inputs(cfg0)
dev = torch.device("cuda", 0)
cfg = dataclasses.replace(cfg0, M=ns, maxit=its, tol=1e-30)
sol = GpuSolver(cfg, inp["psf"], np.full(ns, 1e-5), check_every=8)
sol.reset_weights()
sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
X = torch.zeros(ns, cfg.N, dtype=torch.float64, device=dev)
res = sol.cg(list(range(ns)), X, [0] * ns)
torch.cuda.synchronize()
print("ok", int(res["iters"].max()))
