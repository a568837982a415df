"""ncu / timing target: the batched deflated CG loop at a config's grid with M shifts in
two groups, |J| random Ritz-like columns (images by the library's own apply), carried
columns, a fixed number of lockstep iterations.
  python tools/probe_defl.py [C4] [M] [iters] [J]      (PROBE_ONE_GROUP=1: one group)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes  # noqa: E402
import os as _os  # noqa: E402
_os.environ.setdefault("RSK_PERSIST_PROF", "1")
import dataclasses  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import rsk_synth as S  # noqa: E402
from paper_2306_15049_b200 import _lib as L  # noqa: E402
from paper_2306_15049_b200.pipeline import GpuSolver  # noqa: E402

cfg0 = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
M = int(sys.argv[2]) if len(sys.argv) > 2 else 16
its = int(sys.argv[3]) if len(sys.argv) > 3 else 40
J = int(sys.argv[4]) if len(sys.argv) > 4 else cfg0.J
inp = S.make_inputs(cfg0)
dev = torch.device("cuda", 0)
cfg = dataclasses.replace(cfg0, M=M, maxit=its, tol=1e-30)
gam = np.logspace(np.log10(cfg0.gamma_lo), np.log10(cfg0.gamma_hi), M)
sol = GpuSolver(cfg, inp["psf"], gam, check_every=8)
wx, wy = S.random_weights(7, cfg.n, 1.0, 1.0 / cfg.tau)
f = dict(dtype=torch.float64, device=dev)
sol.h.set_weights(torch.from_numpy(wx.ravel()).to(dev), torch.from_numpy(wy.ravel()).to(dev))
sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
N = cfg.N
Ws, AWs, EWs = [], [], []
for g in range(2):
    W = torch.randn(J, N, **f)
    W /= W.norm(dim=1, keepdim=True)
    AW = torch.empty_like(W); EW = torch.empty_like(W)
    sol.h.apply_shifted(W, AW, EY=EW, mode=L.RSK_APPLY_SPLIT)
    Ws.append(W); AWs.append(AW); EWs.append(EW)
grp = np.array([0 if l < M // 2 else 1 for l in range(M)], dtype=np.int32)
if os.environ.get("PROBE_ONE_GROUP"):   # the tail of a C4 step: every active shift in one group
    grp[:] = 0
Gh = torch.randn(M, N, **f)
Gh /= Gh.norm(dim=1, keepdim=True)
ZGh = torch.empty_like(Gh)
sol.h.apply_shifted(Gh, ZGh, gamma=sol.gam_dev)
hg = np.ones(M, dtype=np.int32)
X = torch.zeros(M, N, **f)
lib = L.load()
lib.rsk_debug_stream_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
lib.rsk_debug_persist_prof.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
a8 = (ctypes.c_double * 8)()
b8 = (ctypes.c_double * 8)()
lib.rsk_debug_stream_prof2.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
lib.rsk_debug_stream_prof2(b8, 1)
c8 = (ctypes.c_double * 8)()
lib.rsk_debug_stream_prof3.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
lib.rsk_debug_stream_prof3(c8, 1)
lib.rsk_debug_stream_prof(a8, 1)
lib.rsk_debug_persist_prof(a8, 1)
torch.cuda.synchronize()
res = sol.cg(list(range(M)), X, np.zeros(M, np.int32), groups=dict(W=Ws, AW=AWs, EW=EWs, of_shift=grp),
             ghat=(Gh, ZGh, hg))
torch.cuda.synchronize()
lib.rsk_debug_stream_prof(a8, 0)
lib.rsk_debug_stream_prof2(b8, 0)
lib.rsk_debug_stream_prof3(c8, 0)
if b8[1] > 0:
    print("B issue: expect+bulk us/step", round(c8[0] / b8[1] / 1e3, 3), "expect+bulk+tma", round(c8[1] / b8[1] / 1e3, 3))
if b8[1] > 0:
    print("B: steps", int(b8[1]), "wait us/step", round(b8[0] / b8[1] / 1e3, 3), "step-to-step us", round(b8[4] / b8[1] / 1e3, 3),
          "| C: steps", int(b8[3]), "wait us/step", round(b8[2] / max(b8[3], 1) / 1e3, 3), "step-to-step us",
          round(b8[5] / max(b8[3], 1) / 1e3, 3), "| B issue us/step", round(b8[6] / b8[1] / 1e3, 3),
          "B (a)+sync us/step", round(b8[7] / b8[1] / 1e3, 3))
ct = np.zeros((296, 8))
lib.rsk_debug_stream_cta.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
lib.rsk_debug_stream_cta(ct.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 296)
if ct[:, 0].max() > 0:
    t0 = ct[:, 0].min()
    for j, nm in ((0, "A end"), (2, "B end"), (3, "B2 end"), (4, "C end")):
        v = (ct[:, j] - t0) / 1e3
        print(f"iteration 30 {nm}: min {v.min():.1f} med {np.median(v):.1f} max {v.max():.1f} us; slowest CTAs {np.argsort(-v)[:5].tolist()}")
if a8[5] == 0:
    lib.rsk_debug_persist_prof(a8, 0)
if a8[5] > 0:
    print("phases us per lockstep iteration:", {k: round(a8[i] / a8[5] / 1e3, 1) for i, k in
                                                 enumerate(["A", "barriers", "B", "B2", "C"])})
print("ok", M, "shifts", int(res["iters"].max()), "iterations, loop ms", res["prof"][5], "kind", int(res["prof"][7]),
      "per lockstep iteration us", 1e3 * res["prof"][5] / max(1, int(res["iters"].max())))
