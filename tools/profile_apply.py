"""Small, repeatable workload for ncu: the fused apply over the C2 batch and a few
lockstep CG iterations (no oracle involved). Usage: python tools/profile_apply.py [C2]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import rsk_synth as S
from paper_2306_15049_b200.pipeline import GpuSolver

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
sol = GpuSolver(cfg, inp["psf"], inp["gamma"], check_every=8)
sol.reset_weights()
X = torch.randn(cfg.M, cfg.N, dtype=torch.float64, device=dev)
Y = torch.empty_like(X)
for _ in range(5):
    sol.h.apply_shifted(X, Y, gamma=sol.gam_dev)
torch.cuda.synchronize()
# a short deflation-free batched CG over all shifts (exercises the CG kernels)
import dataclasses
sol.cfg = dataclasses.replace(cfg, maxit=40)
sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
Xc = torch.zeros(cfg.M, cfg.N, dtype=torch.float64, device=dev)
res = sol.cg(list(range(cfg.M)), Xc, [0] * cfg.M)
torch.cuda.synchronize()
print("ok", int(res["iters"].sum()))
