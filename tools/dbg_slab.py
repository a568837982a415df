"""Debug: slab CG vs single-domain CG, nranks = 1, 2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import rsk_synth as S
from paper_2306_15049_b200 import _lib as L
from paper_2306_15049_b200.pipeline import GpuSolver
from paper_2306_15049_b200.slab import SlabOps, SlabPlan, run_threads, slab_cg
dev = torch.device("cuda", 0)
cfg = S.small_config(n=64, M=4, r=3, sigma=1.3, tol=1e-10)
inp = S.make_inputs(cfg)
n, N = cfg.n, cfg.N
sol = GpuSolver(cfg, inp["psf"], inp["gamma"], device=0)
wx, wy = S.random_weights(5, n)
wxd, wyd = (torch.from_numpy(np.ascontiguousarray(a.ravel())).to(dev) for a in (wx, wy))
sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
sol.h.set_weights(wxd, wyd)
b = sol.b.clone()
gam = np.asarray(inp["gamma"])[:cfg.M]
X1 = torch.zeros(cfg.M, N, dtype=torch.float64, device=dev)
res1 = sol.cg(list(range(cfg.M)), X1, [0] * cfg.M)
print("single", res1["iters"])
for nr in (1, 2):
    plan = SlabPlan(n, n, cfg.r, nr)
    def rank_fn(k, comm):
        ops = SlabOps(plan, k, comm, inp["psf"], 0)
        ops.set_weights(wxd, wyd)
        be = plan.extend(b, k)
        # check one apply of b
        Bt = be[None].repeat(cfg.M, 1).contiguous()
        Yt = torch.empty_like(Bt)
        ops.apply(Bt, Yt, torch.from_numpy(gam).to(dev))
        Xe = torch.zeros(cfg.M, plan.slabs[k].ext_rows * n, dtype=torch.float64, device=dev)
        res = slab_cg(ops, gam, be, Xe, tol=cfg.tol, maxit=2000)
        torch.cuda.synchronize()
        return res, ops.own(Xe).cpu().numpy(), ops.own(Yt).cpu().numpy()
    outs = run_threads(plan, rank_fn)
    Yref = torch.empty(cfg.M, N, dtype=torch.float64, device=dev)
    sol.h.apply_shifted(b[None].repeat(cfg.M, 1).contiguous(), Yref, gamma=torch.from_numpy(gam).to(dev))
    Ys = np.concatenate([o[2] for o in outs], 1)
    print(nr, "apply err", np.max(np.abs(Ys - Yref.cpu().numpy())) / np.max(np.abs(Ys)))
    print(nr, outs[0][0]["iters"], outs[0][0]["relres_true"])
