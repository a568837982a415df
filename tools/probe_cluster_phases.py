"""Per-phase time of one iteration of the cluster-per-shift deflated CG loop inside the
C2 nested solve (RSK_CLUSTER_PROF: cluster 0 / rank 0, %globaltimer marks).
  python tools/probe_cluster_phases.py [C2] [K_out]"""
import ctypes
import os
import sys

os.environ["RSK_CLUSTER_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import rsk_synth as S  # noqa: E402
from paper_2306_15049_b200 import _lib as L  # noqa: E402
from paper_2306_15049_b200.pipeline import GpuSolver  # noqa: E402

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 2
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
sol = GpuSolver(cfg, inp["psf"], inp["gamma"])
sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
lib = L.load()
lib.rsk_debug_cluster_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
a = (ctypes.c_double * 8)()
sol.run(K_out=K)
torch.cuda.synchronize()
lib.rsk_debug_cluster_prof(a, 1)
sol.run(K_out=K)
torch.cuda.synchronize()
lib.rsk_debug_cluster_prof(a, 0)
n = max(a[6], 1)
names = ["A apply", "cluster barriers", "alpha", "B rows+reduce", "z+status", "C rows"]
tot = sum(a[i] for i in range(6)) / n / 1e3
print(f"{cfg.name} K_out={K}: cluster 0 rank 0, {int(n)} iterations, {tot:.2f} us per iteration:",
      ", ".join(f"{nm} {a[i] / n / 1e3:.2f} us" for i, nm in enumerate(names)), flush=True)
if os.environ.get("RSK_APPLY_PROF"):
    lib.rsk_debug_apply_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
    b = (ctypes.c_double * 8)()
    lib.rsk_debug_apply_prof(b, 0)
    names = ["issue->wait", "TMA wait", "x-pass+sync", "y-pass+epilogue", "dot+ticket", "end sync", "", "entry"]
    print("apply item phases, block %s, summed over both runs (us):" % os.environ["RSK_APPLY_PROF"],
          ", ".join(f"{nm} {b[i] / 1e3:.1f}" for i, nm in enumerate(names) if nm), flush=True)
    print("per iteration (2 x %d iterations): " % int(n), ", ".join(f"{nm} {b[i] / 1e3 / (2 * n):.2f}" for i, nm in enumerate(names) if nm))
