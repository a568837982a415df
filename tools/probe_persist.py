"""Per-phase timing of the persistent CG loop (RSK_PERSIST_PROF=1): a plain batched CG on
the config's b over nshift shifts, maxit iterations. Usage: probe_persist.py C2 32 300"""
import ctypes
import dataclasses
import os
import sys
import time

os.environ["RSK_PERSIST_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import rsk_synth as S
from paper_2306_15049_b200 import _lib as L
from paper_2306_15049_b200.pipeline import GpuSolver

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 32
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 300
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
sol = GpuSolver(cfg, inp["psf"], inp["gamma"], check_every=8)
sol.reset_weights()
sol.cfg = dataclasses.replace(cfg, maxit=maxit, tol=1e-30)
sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
lib = L.load()
lib.rsk_debug_persist_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
out = (ctypes.c_double * 8)()
idx = [i % cfg.M for i in range(ns)]
for rep in range(2):
    X = torch.zeros(ns, cfg.N, dtype=torch.float64, device=dev)
    lib.rsk_debug_persist_prof(out, 1)
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = sol.cg(idx, X, [0] * ns)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    lib.rsk_debug_persist_prof(out, 0)
    its = int(out[5])
    names = ["A apply", "barriers", "B update", "B2 scalars", "C combine"]
    print(f"{cfg.name} ns={ns} lockstep its={its} wall {dt*1e3:.1f} ms, per iteration:",
          ", ".join(f"{n} {out[i]/max(its,1)/1e3:.1f} us" for i, n in enumerate(names)))
if os.environ.get("RSK_APPLY_PROF"):
    lib.rsk_debug_apply_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
    a = (ctypes.c_double * 8)()
    lib.rsk_debug_apply_prof(a, 0)
    names = ["issue->wait", "TMA wait", "x-pass+sync", "y-pass+epilogue", "dot+ticket", "end sync"]
    its2 = max(its, 300)
    print("apply block %s per iteration (2 runs):" % os.environ["RSK_APPLY_PROF"],
          ", ".join(f"{n} {a[i]/(2*its2)/1e3:.2f} us" for i, n in enumerate(names)))
if os.environ.get("RSK_CLUSTER_PROF"):
    lib.rsk_debug_cluster_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
    a = (ctypes.c_double * 8)()
    lib.rsk_debug_cluster_prof(a, 0)
    n = max(a[6], 1)
    names = ["A apply", "cluster barriers", "alpha", "B rows+reduce", "z+status", "C rows"]
    print("cluster 0 rank 0 per iteration (%d its):" % n, ", ".join(f"{nm} {a[i]/n/1e3:.2f} us" for i, nm in enumerate(names)))
