"""Per-iteration cost of rsk_minres_recycled_batch at C2 size for 1, 2 and 32 shifts
(random orthonormal group blocks, |J| = 8, one carried column): maxit iterations with an
unreachable tolerance, wall time / iteration. Run under ncu for the kernel split."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import rsk_synth as S  # noqa: E402
from paper_2306_15049_b200 import _lib as L  # noqa: E402
from paper_2306_15049_b200.rsk import Handle  # noqa: E402


def run(ns, maxit, n=256, J=8, check_every=8):
    dev = torch.device("cuda", 0)
    N = n * n
    h = Handle(n, n, S.gaussian_psf(4, 2.0), 0)
    f = dict(dtype=torch.float64, device=dev)
    b = torch.randn(N, **f)
    X = torch.zeros(ns, N, **f)
    W = torch.linalg.qr(torch.randn(N, J, **f))[0].t().contiguous()
    AW = torch.randn(J, N, **f); EW = torch.randn(J, N, **f)
    Gh = torch.randn(ns, N, **f); ZGh = torch.randn(ns, N, **f)
    gam = np.logspace(-4, 1, ns)
    d = L.CgDesc()
    d.nshift = ns; d.gamma_h = gam.ctypes.data_as(L._hp); d.b = b.data_ptr(); d.X = X.data_ptr(); d.ldx = N
    d.ngroups = 1
    gos = np.zeros(ns, np.int32); hg = np.ones(ns, np.int32)
    d.group_of_shift_h = gos.ctypes.data_as(L.C.POINTER(L.C.c_int))
    d.W[0] = W.data_ptr(); d.AW[0] = AW.data_ptr(); d.EW[0] = EW.data_ptr(); d.J[0] = J; d.ldw = N
    d.Ghat = Gh.data_ptr(); d.ZGhat = ZGh.data_ptr(); d.ldgh = N
    d.has_ghat_h = hg.ctypes.data_as(L.C.POINTER(L.C.c_int))
    d.tol = 1e-300; d.maxit = maxit; d.check_every = check_every
    o = L.CgOut()
    it = np.zeros(ns, np.int32); ap = np.zeros(ns, np.int64); rr = np.zeros(ns); st = np.zeros(ns, np.int32)
    mu = np.zeros(ns, np.int32)
    P = L.C.POINTER
    o.iters = it.ctypes.data_as(P(L.C.c_int)); o.applies = ap.ctypes.data_as(P(L.C.c_int64))
    o.relres_true = rr.ctypes.data_as(L._hp); o.status = st.ctypes.data_as(P(L.C.c_int))
    o.m_used = mu.ctypes.data_as(P(L.C.c_int))
    ws = torch.empty(h.minres_workspace_bytes(ns, J + 1), dtype=torch.uint8, device=dev)
    h.minres_recycled_batch(d, o, ws)        # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.minres_recycled_batch(d, o, ws)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"ns={ns} maxit={maxit} check_every={check_every}: {dt * 1e6 / maxit:.1f} us per lockstep iteration "
          f"({dt * 1e6 / (maxit * ns):.2f} us per shift-iteration), iters {it.min()}..{it.max()}", flush=True)


if __name__ == "__main__":
    maxit = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    for ns in (1, 2, 32):
        for ce in (8, 64):
            run(ns, maxit, check_every=ce)
