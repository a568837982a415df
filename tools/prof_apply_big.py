"""ncu target: the standalone fused shifted apply over a config's full batch.
  python tools/prof_apply_big.py [C4] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import rsk_synth as S  # noqa: E402
from paper_2306_15049_b200.pipeline import GpuSolver  # noqa: E402

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
sol = GpuSolver(cfg, inp["psf"], inp["gamma"])
sol.reset_weights()
X = torch.randn(cfg.M, cfg.N, dtype=torch.float64, device=dev)
Y = torch.empty_like(X)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(reps):
    e0.record()
    sol.h.apply_shifted(X, Y, gamma=sol.gam_dev)
    e1.record()
    torch.cuda.synchronize()
    print(f"{cfg.name} apply x{cfg.M}: {e0.elapsed_time(e1):.3f} ms", flush=True)
