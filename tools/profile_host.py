"""Host-side profile of one C2 nested solve (after a warm-up run): cProfile of sol.run(),
top entries by cumulative and by internal time. The device loop kernel's own time shows
up inside rsk_cg_recycled_batch (host-blocking)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import rsk_synth as S  # noqa: E402
from paper_2306_15049_b200.pipeline import GpuSolver  # noqa: E402

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
sol = GpuSolver(cfg, inp["psf"], inp["gamma"])
xt = torch.from_numpy(inp["x_true"]).to(dev)
xi = torch.from_numpy(inp["xi"]).to(dev)
sol.set_data(xt, xi)
sol.run()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
sol.set_data(xt, xi)
sol.run()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(35)
st.sort_stats("tottime").print_stats(25)
