"""One C2 outer step k=0 through the GPU pipeline, with host wall time around the
batched CG call -- for launch lists (ncu --metrics gpu__time_duration.sum)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import rsk_synth as S
from paper_2306_15049_b200 import _lib as L
from paper_2306_15049_b200.pipeline import GpuSolver

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
ce = int(sys.argv[2]) if len(sys.argv) > 2 else 8
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
sol = GpuSolver(cfg, inp["psf"], inp["gamma"], check_every=ce)
sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
sol.reset_weights()
lib = L.load()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); l0 = lib.rsk_launch_count()
    o, st = sol.outer_step(0, {})
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"rep {rep}: outer step 0 wall {1e3*(t1-t0):.1f} ms, iters {int(o.iters.sum())}, "
          f"launches {lib.rsk_launch_count()-l0}, cg-loop lockstep max {int(o.iters.max())}")
# the CG alone on all shifts, plain (no deflation), timing
X = torch.zeros(cfg.M, cfg.N, dtype=torch.float64, device=dev)
torch.cuda.synchronize(); t0 = time.perf_counter(); l0 = lib.rsk_launch_count()
res = sol.cg(list(range(cfg.M)), X, [0] * cfg.M)
torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"plain batched CG: wall {1e3*(t1-t0):.1f} ms, iters sum {int(res['iters'].sum())} max {int(res['iters'].max())}, launches {lib.rsk_launch_count()-l0}")
# host launch overhead of a tiny apply
x1 = torch.zeros(1, cfg.N, dtype=torch.float64, device=dev); y1 = torch.empty_like(x1)
g1 = sol.gam_dev[:1].contiguous()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(200):
    sol.h.apply_shifted(x1, y1, gamma=g1)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"200 single-vector applies: host enqueue {1e6*(t1-t0)/200:.1f} us/call, device drain {1e6*(t2-t0)/200:.1f} us/call")
