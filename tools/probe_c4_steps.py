"""Per-outer-step anatomy of the persistent lockstep CG loop at C4 (or another config):
per-shift iteration counts, lockstep iterations and the per-phase time (RSK_PERSIST_PROF,
block 0's %globaltimer marks) of outer steps k = 0 .. K-1.
  python tools/probe_c4_steps.py [C4] [K]"""
import ctypes
import json
import os
import sys
import time

os.environ["RSK_PERSIST_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import rsk_synth as S  # noqa: E402
from paper_2306_15049_b200 import _lib as L  # noqa: E402
from paper_2306_15049_b200.pipeline import GpuSolver  # noqa: E402

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 2
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
sol = GpuSolver(cfg, inp["psf"], S.gamma_ladder(cfg))
sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
lib = L.load()
lib.rsk_debug_persist_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
lib.rsk_debug_stream_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
a = (ctypes.c_double * 8)()
b8 = (ctypes.c_double * 8)()
names = ["A apply", "barriers", "B update", "B2 scalars", "C combine"]
sol.reset_weights()
st = {}
for k in range(K):
    lib.rsk_debug_persist_prof(a, 1)
    lib.rsk_debug_stream_prof(b8, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    o, st = sol.outer_step(k, st)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    lib.rsk_debug_persist_prof(a, 0)
    lib.rsk_debug_stream_prof(b8, 0)
    if b8[5] > 0:
        a = b8
    its = max(a[5], 1)
    it = np.asarray(o.iters)
    rec = {"cfg": cfg.name, "k": k, "s": dt, "shift_iterations": int(it.sum()), "lockstep": int(its),
           "mean_active": float(it.sum() / its), "iters": it.tolist(), "lstar": int(o.lstar), "nc": int(o.nc),
           "loop_ms": float(o.prof[5]) if o.prof is not None else None,
           "loop_kind": int(o.prof[7]) if o.prof is not None else None,
           "phase_us": {n: a[i] / its / 1e3 for i, n in enumerate(names)}}
    print(json.dumps(rec), flush=True)
    if k + 1 < K:
        sol.next_weights(st["xstar"])
        st["W_prev"] = sol.w_prev
