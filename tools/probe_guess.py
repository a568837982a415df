"""Orthogonal vs oblique principal guesses (§sec:oblique P:870-1005):
for each guess mode, the relative residual of every shift's initial guess
||b - (A + gamma_l E_k) x_0|| / ||b|| and the CG iterations that follow, per outer step.

  python tools/probe_guess.py --config C2 --outer 3 [--rule irn|gazzola]"""
import argparse
import dataclasses
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import rsk_synth as S  # noqa: E402
from paper_2306_15049_b200.pipeline import GpuSolver  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--outer", type=int, default=3)
    ap.add_argument("--rule", default="irn")
    ap.add_argument("--modes", default="orth,oblique,oblique2")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    for mode in a.modes.split(","):
        cfg = dataclasses.replace(S.CONFIGS[a.config], guess=mode, weight_rule=a.rule)
        inp = S.make_inputs(cfg)
        sol = GpuSolver(cfg, inp["psf"], inp["gamma"])
        sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
        grel = {}
        nb = float(torch.linalg.norm(sol.b))

        def hook(k, mine, X, has_xp, sol=sol, grel=grel, nb=nb):
            Y = torch.empty_like(X)
            g = sol.gam_dev[torch.tensor(mine, device=dev)].contiguous()
            sol.h.apply_shifted(X, Y, gamma=g)
            r = torch.linalg.norm(sol.b[None, :] - Y, dim=1) / nb
            grel[k] = r.cpu().numpy()

        sol.guess_hook = hook
        outs = sol.run(K_out=a.outer)
        for o in outs:
            g = grel[o.k]
            print(f"{a.config} rule={a.rule} guess={mode:8s} k={o.k}: guess relres median {np.median(g):.3e} "
                  f"max {g.max():.3e} min {g.min():.3e}; CG its total {int(o.iters.sum())} "
                  f"max {int(o.iters.max())}; l*={o.lstar}; {o.ms * 1e3:.0f} ms", flush=True)


if __name__ == "__main__":
    main()
