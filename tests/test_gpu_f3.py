"""GPU parity of the principal update with V^(new) (eq:delta, eq:tildeUupdate P:633-654;
SURVEY §8(f) f3): the eq:delta correction solve against the oracle's, and the nested
solve with principal="vnew" stepwise against the oracle (reading G28): solutions within
1e-8 (or the tolerance-limited bound), iterations +-2 on 95 % of the solves, same l*."""
import dataclasses

import numpy as np
import pytest

import rsk_synth as S
from paper_2306_15049_b200.indices import shift_indices
from oracle import dense
from oracle import operators as ops
from oracle import pipeline as opipe

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    return torch, torch.device("cuda", 0)


def _t(torch, dev, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def _dev_state(torch, dev, st):
    out = {}
    if st.V_i1 is not None:
        out["V_i1"] = _t(torch, dev, st.V_i1.T)
    if st.X_prev is not None:
        out["X_prev"] = _t(torch, dev, st.X_prev.T)
        out["G_prev"] = _t(torch, dev, st.G_prev.T)
    if st.wx_prev is not None:
        out["W_prev"] = (_t(torch, dev, st.wx_prev.ravel()), _t(torch, dev, st.wy_prev.ravel()))
    return out


@pytest.mark.parametrize("inner", ["cg", "minres"])
def test_vnew_stepwise_handoff(torch_dev, inner):
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = dataclasses.replace(S.CONFIGS["C1"], tol=1e-10, principal="vnew", n_c=40, inner=inner)
    inp = S.make_inputs(cfg)
    ref = opipe.run(cfg, inp, keep_steps=True)
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"], check_every=4)
    sol.set_data(_t(torch, dev, inp["x_true"].ravel()), _t(torch, dev, inp["xi"].ravel()))
    n = cfg.n
    wx, wy = ops.identity_weights(n)
    st = opipe.StepState(0, wx, wy, None, None, None)
    all_d = []
    for k, rs in enumerate(ref["steps"]):
        sol.h.set_weights(_t(torch, dev, st.wx.ravel()), _t(torch, dev, st.wy.ravel()))
        sol.cur_w = (_t(torch, dev, st.wx.ravel()), _t(torch, dev, st.wy.ravel()))
        dst = _dev_state(torch, dev, st)
        if k >= 1:
            # the eq:delta solve itself: V^(new)'s first column vs the oracle's
            Vg, _ = sol.principal_update(dst)
            Vo, _ = opipe.principal_update(cfg, inp["psf"], ref["b"], inp["gamma"], st)
            dxg, dxo = Vg[0].cpu().numpy(), Vo[:, 0]
            # 100 CG steps that stop short of convergence (eq:delta at l_c, IRN weights up
            # to 1/tau): two correct implementations drift apart by rounding amplified along
            # the iteration (reading G27; CG residual norms oscillate before convergence),
            # so compare the iterates to 1e-4 and their residuals in eq:delta to 25 %
            # (MINRES: Lanczos loses orthogonality over the 100 steps, iterates agree to 1e-2)
            assert np.linalg.norm(dxg - dxo) <= (1e-4 if inner == "cg" else 1e-2) * np.linalg.norm(dxo)
            lc = shift_indices(cfg).l_c - 1
            gc = inp["gamma"][lc]
            xp = st.X_prev[:, lc].reshape(n, n)
            q = gc * (ops.apply_E(st.wx, st.wy, xp) - ops.apply_E(st.wx_prev, st.wy_prev, xp)).ravel()
            res = [np.linalg.norm(q - ops.apply_shifted(inp["psf"], st.wx, st.wy, gc, v.reshape(n, n)).ravel())
                   for v in (dxg, dxo)]
            assert 0.8 * res[1] - 1e-12 * np.linalg.norm(q) <= res[0] <= 1.25 * res[1] + 1e-12 * np.linalg.norm(q), res
            assert Vg.shape[0] == Vo.shape[1]
        o, X = sol.outer_step(k, dst)
        assert np.all((o.status == 0) | (o.status == 3)), o.status
        assert o.nc == rs.nc
        Ad = dense.assemble(lambda v: ops.apply_A(inp["psf"], v), n)
        Ed = dense.assemble(lambda v: ops.apply_E(st.wx, st.wy, v), n)
        for l in range(cfg.M):
            xg = X["X_prev"][l].cpu().numpy()
            rel = np.linalg.norm(xg - rs.X[:, l]) / np.linalg.norm(rs.X[:, l])
            if rel > 1e-8:
                ev = np.linalg.eigvalsh(Ad + inp["gamma"][l] * Ed)
                assert rel <= 2.0 * (ev[-1] / ev[0]) * cfg.tol, (k, l, rel)
        d_it = np.abs(o.iters - rs.iters)
        all_d.append(d_it)
        assert np.all(d_it <= np.maximum(2, 0.01 * rs.iters) + 2), (o.iters, rs.iters)
        assert o.lstar == rs.lstar
        xstar = rs.X[:, rs.lstar].reshape(n, n)
        wx, wy = ops.irn_weights(xstar, cfg.tau)
        st = opipe.StepState(k + 1, wx, wy, rs.X, rs.G, rs.V_i1, st.wx, st.wy)
    assert np.mean(np.concatenate(all_d) <= 2) >= 0.95, all_d


def test_vnew_full_run_converges(torch_dev):
    """The free-running nested solve with V^(new) at C2 size: every shift converged."""
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = dataclasses.replace(S.CONFIGS["C2"], principal="vnew", K_out=3)
    inp = S.make_inputs(cfg)
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"])
    sol.set_data(_t(torch, dev, inp["x_true"].ravel()), _t(torch, dev, inp["xi"].ravel()))
    outs = sol.run()
    for o in outs:
        assert np.all(o.status == 0), o.status
        assert np.all(o.relres <= cfg.tol)
