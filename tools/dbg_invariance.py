"""Batch-composition invariance of the streaming CG loop: full batch vs a sub-batch after
maxit = 0, 1, 2, ... iterations (max |X_full[sub] - X_sub|)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
os.environ["RSK_CG_NOCLUSTER"] = "1"
os.environ["RSK_CG_STREAM"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import rsk_synth as S  # noqa: E402
import test_gpu_persist as T  # noqa: E402

dev = torch.device("cuda", 0)
n, r, nL, nR = 100, 7, 40, 9
M = nL + nR
sub = [3, 17, 25, 39, 41, 44, 47]
for maxit in [int(a) for a in sys.argv[1:]] or [100, 200, 400, 800, 20000]:
    cfg = dataclasses.replace(S.small_config(n=n, M=M, r=r, sigma=1.0 + 0.3 * r, tol=1e-10), maxit=maxit)
    gam = np.logspace(-4, 1.5, M)
    sol, groups, ghat, X0 = T._setup(torch, dev, cfg, nL, nR, 12, 900 + n, gam)
    X = X0.clone()
    res = sol.cg(list(range(M)), X, T._CTX["has_xp"], groups=groups, ghat=ghat)
    Xs = X0[sub].clone()
    gs = dict(groups, of_shift=np.asarray(groups["of_shift"])[sub])
    Gh, ZGh, hg = ghat
    rs = sol.cg(sub, Xs, T._CTX["has_xp"][sub], groups=gs,
                ghat=(Gh[sub].contiguous(), ZGh[sub].contiguous(), np.asarray(hg)[sub]))
    d = (Xs - X[sub]).abs().max(dim=1).values.cpu().numpy()
    print("maxit", maxit, "kind", int(res["prof"][7]), int(rs["prof"][7]), "iters", res["iters"][sub].tolist(),
          rs["iters"].tolist(), "max|dX| per shift", np.array2string(d, precision=2))
