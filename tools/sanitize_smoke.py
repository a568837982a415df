"""Small end-to-end exercise of every device loop for compute-sanitizer runs:
cluster CG, persistent CG (RSK_CG_NOCLUSTER), MINRES (cluster loop, even size; lockstep,
odd size), CT apply + MINRES, tensor-core Grams.
  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import rsk_synth as S  # noqa: E402
from paper_2306_15049_b200.pipeline import GpuSolver  # noqa: E402

dev = torch.device("cuda", 0)


def run(cfg):
    inp = S.make_inputs(cfg)
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"], check_every=4)
    xi = inp["xi"].ravel() if cfg.operator == "ct" else inp["xi"]
    sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(np.ascontiguousarray(xi)).to(dev))
    outs = sol.run(K_out=2)
    torch.cuda.synchronize()
    print(cfg.name, cfg.inner, cfg.n, [int(o.iters.sum()) for o in outs], flush=True)


base = S.small_config(n=32, M=6, r=2, sigma=1.0, n_c=16, J=4, K_out=2, tol=1e-8)
run(base)                                                   # cluster CG, TC Grams (k >= 16)
run(dataclasses.replace(base, inner="minres"))              # MINRES cluster loop
run(dataclasses.replace(base, n=33, inner="minres"))        # MINRES lockstep (odd size)
os.environ["RSK_CG_NOCLUSTER"] = "1"
run(dataclasses.replace(base, n=34))                        # persistent lockstep CG
os.environ.pop("RSK_CG_NOCLUSTER")
run(dataclasses.replace(S.CONFIGS["C6"], n=16, n_angles=12, M=4, n_c=8, J=2, idx=(2, 2, 3, 3, 3, 3),
                        gamma_lo=1e-4, gamma_hi=1.0, inner="minres"))   # CT
print("sanitize smoke done")
