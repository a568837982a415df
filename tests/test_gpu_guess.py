"""GPU parity of the oblique principal guesses (eq:obliqueupdate
P:877-882, two anchors eq:updates P:1000-1005) inside the nested solve: stepwise
handoff from the oracle's state (reading G28), same bars as the orthogonal path --
solutions within 1e-8 (or the tolerance-limited bound), iteration counts +-2 on 95 %
of the run's solves, the same l*."""
import dataclasses

import numpy as np
import pytest

import rsk_synth as S
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


def _state_to_dev(torch, dev, st):
    out = {}
    if st.V_i1 is not None:
        out["V_i1"] = _t(torch, dev, st.V_i1.T)
    if st.X_prev is not None:
        out["X_prev"] = _t(torch, dev, st.X_prev.T)
        out["G_prev"] = _t(torch, dev, st.G_prev.T)
    return out


@pytest.mark.parametrize("mode", ["oblique", "oblique2"])
def test_oblique_guesses_stepwise_handoff(torch_dev, mode):
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = dataclasses.replace(S.CONFIGS["C1"], tol=1e-10, guess=mode)
    inp = S.make_inputs(cfg)
    ref = opipe.run(cfg, inp, keep_steps=True)
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"], check_every=4)
    sol.set_data(_t(torch, dev, inp["x_true"].ravel()), _t(torch, dev, inp["xi"].ravel()))
    n = cfg.n
    wx, wy = ops.identity_weights(n)
    st = opipe.StepState(0, wx, wy, None, None, None)
    guesses = {}
    all_d = []
    sol.guess_hook = lambda k, mine, X, hx: guesses.__setitem__(k, (X.cpu().numpy().copy(), hx.copy()))
    for k, rs in enumerate(ref["steps"]):
        sol.h.set_weights(_t(torch, dev, st.wx.ravel()), _t(torch, dev, st.wy.ravel()))
        o, X = sol.outer_step(k, _state_to_dev(torch, dev, st))
        assert np.all(o.status == 0), o.status
        # the guesses themselves: the coefficients of x_p are ill-conditioned functions of
        # the principal space (which holds the GPU's own seed solves at k = 0, equal to the
        # oracle's only to the CG tolerance), so compare the well-posed quantity, the guess
        # residual ||b - A_g x_p|| / ||b||, within 5 % (or both below 1e-6)
        Xg, hx = guesses[k]
        assert np.all(hx == 1)
        Ad = dense.assemble(lambda v: ops.apply_A(inp["psf"], v), n)
        Ed = dense.assemble(lambda v: ops.apply_E(st.wx, st.wy, v), n)
        b = ref["b"]
        for l in range(cfg.M):
            g = np.linalg.norm(b - (Ad + inp["gamma"][l] * Ed) @ Xg[l]) / np.linalg.norm(b)
            gr = rs.guess_relres[l]
            assert (g <= 1e-6 and gr <= 1e-6) or abs(np.log(g / gr)) <= np.log(1.05), (k, l, g, gr)
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
        st = opipe.StepState(k + 1, wx, wy, rs.X, rs.G, rs.V_i1)
    # reading G27's count bar (+-2 on >= 95 % of shifts) over all the solves of the run
    assert np.mean(np.concatenate(all_d) <= 2) >= 0.95, all_d
