"""Per-phase time of one lockstep iteration of the persistent deflated CG loop inside an
outer step (RSK_PERSIST_PROF: block 0's view, %globaltimer marks).
  python tools/probe_persist_phases.py [C4] [K_out] [M]"""
import ctypes
import dataclasses
import os
import sys
import time

os.environ["RSK_PERSIST_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import rsk_synth as S  # noqa: E402
from paper_2306_15049_b200 import _lib as L  # noqa: E402
from paper_2306_15049_b200.pipeline import GpuSolver  # noqa: E402

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if len(sys.argv) > 3:
    cfg = dataclasses.replace(cfg, M=int(sys.argv[3]))
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
sol = GpuSolver(cfg, inp["psf"], S.gamma_ladder(cfg))
sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
lib = L.load()
lib.rsk_debug_persist_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
a = (ctypes.c_double * 8)()
lib.rsk_debug_persist_prof(a, 1)
t0 = time.perf_counter()
outs = sol.run(K_out=K)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
lib.rsk_debug_persist_prof(a, 0)
its = max(a[5], 1)
names = ["A apply", "barriers", "B update", "B2 scalars", "C combine"]
print(f"{cfg.name} M={cfg.M} K_out={K}: {dt:.1f} s, shift-iterations {sum(int(o.iters.sum()) for o in outs)}, "
      f"lockstep iterations {int(its)}; per lockstep iteration:",
      ", ".join(f"{n} {a[i] / its / 1e3:.1f} us" for i, n in enumerate(names)), flush=True)
