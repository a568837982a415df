"""Strip-apply step anatomy (needs librsk built with -DRSK_STRIP_PROF, standalone kernel):
  python tools/probe_strip.py [C4]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import rsk_synth as S  # noqa: E402
from paper_2306_15049_b200 import _lib as L  # noqa: E402
from paper_2306_15049_b200.pipeline import GpuSolver  # noqa: E402

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
inp = S.make_inputs(cfg)
sol = GpuSolver(cfg, inp["psf"], inp["gamma"])
sol.reset_weights()
X = torch.randn(cfg.M, cfg.N, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
lib = L.load()
lib.rsk_debug_strip_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
a = (ctypes.c_double * 8)()
sol.h.apply_shifted(X, Y, gamma=sol.gam_dev)
torch.cuda.synchronize()
lib.rsk_debug_strip_prof(a, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
sol.h.apply_shifted(X, Y, gamma=sol.gam_dev)
e1.record()
torch.cuda.synchronize()
lib.rsk_debug_strip_prof(a, 0)
print(f"{cfg.name} x{cfg.M}: {e0.elapsed_time(e1):.3f} ms; block 0: steps {int(a[1])}, wait {a[0] / a[1] / 1e3:.3f} us/step, "
      f"step-to-step {a[2] / a[1] / 1e3:.3f} us; after x-pass barrier {a[4] / a[1] / 1e3:.3f}, weights issued "
      f"{a[5] / a[1] / 1e3:.3f}, y DMMA done {a[6] / a[1] / 1e3:.3f} us")
