"""Per-phase timing of block 0 in the standalone apply (RSK_APPLY_PROF=1).
Usage: probe_apply_phases.py C2 1"""
import ctypes
import os
import sys

os.environ["RSK_APPLY_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import rsk_synth as S
from paper_2306_15049_b200 import _lib as L
from paper_2306_15049_b200.rsk import Handle

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 1
inp = S.make_inputs(cfg)
dev = torch.device("cuda", 0)
h = Handle(cfg.n, cfg.n, inp["psf"], 0)
lib = L.load()
lib.rsk_debug_apply_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
out = (ctypes.c_double * 8)()
X = torch.randn(nv, cfg.N, dtype=torch.float64, device=dev)
Y = torch.empty_like(X)
g = torch.full((nv,), 1e-3, dtype=torch.float64, device=dev)
for _ in range(3):
    h.apply_shifted(X, Y, gamma=g)
torch.cuda.synchronize()
lib.rsk_debug_apply_prof(out, 1)
reps = 20
for _ in range(reps):
    h.apply_shifted(X, Y, gamma=g)
torch.cuda.synchronize()
lib.rsk_debug_apply_prof(out, 0)
names = ["issue->wait", "TMA wait", "x-pass+sync", "y-pass+epilogue", "dot", "end sync"]
print(f"{cfg.name} nvec={nv} block0 per launch:", ", ".join(f"{n} {out[i]/reps/1e3:.2f} us" for i, n in enumerate(names)))
