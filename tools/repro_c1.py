"""Run one C1 nested solve (single rank) -- used for sanitizer / repro runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import rsk_synth as S
from paper_2306_15049_b200 import shard
from paper_2306_15049_b200.pipeline import GpuSolver

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
sol = GpuSolver(cfg, inp["psf"], inp["gamma"], device=0, check_every=4, dist=shard.Dist(False))
sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
outs = sol.run()
torch.cuda.synchronize()
print("ok", [o.iters.tolist() for o in outs])
