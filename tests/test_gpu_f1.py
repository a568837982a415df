"""GPU parity for SURVEY §8(f) row f1 (the paper's own outer step) through the C-ABI:
isotropic IRN weights (rsk_irn_weights_iso), Gazzola's update (rsk_gazzola_weights and
its max/update halves) chained over several steps, its row-slab form, and the
outer loop with Gazzola's rule and the P:1042 stopping rule.

Bars: every step of both weight rules is one correctly rounded operation in the
oracle's order, so isotropic weights and Gazzola's D / W at p = 2 (an exact square) are
compared bitwise; other p go through pow (<= 2 ulp in CUDA), compared to 4 ulp of 1."""
import dataclasses

import numpy as np
import pytest

import rsk_synth as S
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
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).ravel()).to(dev)


def _img(seed, n):
    cfg = S.small_config(n=n)
    return S.phantom(cfg, S.rng_for(cfg)) + 1e-2 * S.random_vectors(seed, (n, n))


@pytest.mark.parametrize("n", [77, 300])
def test_irn_iso_weights_bitwise(torch_dev, n):
    torch, dev = torch_dev
    from paper_2306_15049_b200.rsk import Handle
    tau = 1e-3
    x = _img(5, n)
    h = Handle(n, n, S.gaussian_psf(2, 1.0), 0)
    hw = S.random_weights(6, n)
    h.set_weights(_t(torch, dev, hw[0]), _t(torch, dev, hw[1]))
    wx = torch.empty(n * n, dtype=torch.float64, device=dev)
    wy = torch.empty_like(wx)
    e2 = torch.empty(1, dtype=torch.float64, device=dev)
    h.irn_weights_iso(_t(torch, dev, x), tau, wx, wy, e2)
    rx, ry = ops.irn_weights_iso(x, tau)
    np.testing.assert_array_equal(wx.cpu().numpy().reshape(n, n), rx)
    np.testing.assert_array_equal(wy.cpu().numpy().reshape(n, n), ry)
    assert float(e2.cpu()[0]) == pytest.approx(ops.seminorm2(hw[0], hw[1], x), rel=1e-13)


@pytest.mark.parametrize("p", [2.0, 1.0, 0.5, 1.5, 3.0])
@pytest.mark.parametrize("n", [150])
def test_gazzola_chain_matches_oracle(torch_dev, n, p):
    """Three chained steps from D_0 = I with a different x each step (D carried on the
    device, in place); D, W and the max compared after every step."""
    torch, dev = torch_dev
    from paper_2306_15049_b200.rsk import Handle
    h = Handle(n, n, S.gaussian_psf(2, 1.0), 0)
    dx, dy = ops.identity_weights(n)
    Dx, Dy = _t(torch, dev, dx), _t(torch, dev, dy)
    wx = torch.empty(n * n, dtype=torch.float64, device=dev)
    wy = torch.empty_like(wx)
    m = torch.empty(1, dtype=torch.float64, device=dev)
    tol = 0.0 if p in (2.0, 1.0) else 4 * np.spacing(1.0)
    for k in range(3):
        x = _img(10 + k, n)
        xd = _t(torch, dev, x)
        h.gazzola_max(xd, Dx, Dy, m)
        qx, qy = ops.grad(x)
        m_ref = max(np.abs(dx[:, :-1] * qx).max(), np.abs(dy[:-1, :] * qy).max())
        if tol == 0.0:
            assert float(m.cpu()[0]) == m_ref
        else:    # D has drifted by ulps through pow in earlier steps
            assert abs(float(m.cpu()[0]) - m_ref) <= 8 * np.spacing(m_ref)
        h.gazzola_weights(xd, p, Dx, Dy, wx, wy)
        (dx, dy), (rwx, rwy) = ops.gazzola_step(dx, dy, x, p)
        for got, ref in ((Dx, dx), (Dy, dy), (wx, rwx), (wy, rwy)):
            g = got.cpu().numpy().reshape(n, n)
            assert np.max(np.abs(g - ref)) <= tol, (k, p, np.max(np.abs(g - ref)))


def test_gazzola_constant_image_and_errors(torch_dev):
    torch, dev = torch_dev
    from paper_2306_15049_b200.rsk import Handle, RskError
    n = 40
    h = Handle(n, n, S.gaussian_psf(1, 1.0), 0)
    dx, dy = S.random_weights(7, n, 0.1, 1.0)
    Dx, Dy = _t(torch, dev, dx), _t(torch, dev, dy)
    wx = torch.empty(n * n, dtype=torch.float64, device=dev)
    wy = torch.empty_like(wx)
    h.gazzola_weights(_t(torch, dev, np.full((n, n), 2.5)), 2.0, Dx, Dy, wx, wy)
    np.testing.assert_array_equal(Dx.cpu().numpy().reshape(n, n), dx)
    np.testing.assert_array_equal(Dy.cpu().numpy().reshape(n, n), dy)
    np.testing.assert_array_equal(wx.cpu().numpy().reshape(n, n), dx * dx)
    x = _t(torch, dev, _img(8, n))
    for bad in (0.0, -1.0, float("nan"), float("inf")):
        with pytest.raises(RskError):
            h.gazzola_weights(x, bad, Dx, Dy, wx, wy)
    with pytest.raises(RskError):
        h.gazzola_weights(x, 2.0, Dx, Dx, wx, wy)
    with pytest.raises(RskError):
        h.gazzola_weights(x, 2.0, Dx, Dy, Dx, wy)


def test_gazzola_split_halves_equal_one_call(torch_dev):
    """rsk_gazzola_max + rsk_gazzola_update with the same m == rsk_gazzola_weights."""
    torch, dev = torch_dev
    from paper_2306_15049_b200.rsk import Handle
    n = 129
    h = Handle(n, n, S.gaussian_psf(2, 1.0), 0)
    d0 = S.random_weights(9, n, 0.1, 1.0)
    x = _t(torch, dev, _img(12, n))
    A = [_t(torch, dev, d0[0]), _t(torch, dev, d0[1])]
    B = [a.clone() for a in A]
    wa = [torch.empty_like(A[0]) for _ in range(2)]
    wb = [torch.empty_like(A[0]) for _ in range(2)]
    h.gazzola_weights(x, 1.7, A[0], A[1], wa[0], wa[1])
    m = torch.empty(1, dtype=torch.float64, device=dev)
    h.gazzola_max(x, B[0], B[1], m)
    h.gazzola_update(x, 1.7, m, B[0], B[1], wb[0], wb[1])
    for a, b in zip(A + wa, B + wb):
        assert torch.equal(a, b)


@pytest.mark.parametrize("n,r,nranks", [(64, 2, 2), (96, 3, 3)])
def test_slab_gazzola_and_iso_match_single_domain(torch_dev, n, r, nranks):
    """Row slabs (emulated ranks on one GPU): the max-reduced Gazzola update over two
    chained steps and the isotropic weights equal the single-domain ones bitwise on
    every owned row."""
    torch, dev = torch_dev
    from paper_2306_15049_b200.rsk import Handle
    from paper_2306_15049_b200.slab import SlabOps, SlabPlan, run_threads
    psf = S.gaussian_psf(r, 1.0 + 0.3 * r)
    xs = [torch.from_numpy(_img(20 + k, n).ravel()).to(dev) for k in range(2)]
    h = Handle(n, n, psf, 0)
    d0 = ops.identity_weights(n)
    Dx, Dy = _t(torch, dev, d0[0]), _t(torch, dev, d0[1])
    wx = torch.empty(n * n, dtype=torch.float64, device=dev)
    wy = torch.empty_like(wx)
    for x in xs:
        h.gazzola_weights(x, 2.0, Dx, Dy, wx, wy)
    ix = torch.empty_like(wx)
    iy = torch.empty_like(wx)
    h.irn_weights_iso(xs[0], 1e-3, ix, iy)
    torch.cuda.synchronize()
    plan = SlabPlan(n, n, r, nranks)

    def rank_fn(k, comm):
        so = SlabOps(plan, k, comm, psf, 0)
        ext = plan.slabs[k].ext_rows * n
        dx = plan.extend(_t(torch, dev, d0[0]), k).contiguous()
        dy = plan.extend(_t(torch, dev, d0[1]), k).contiguous()
        swx = torch.empty(ext, dtype=torch.float64, device=dev)
        swy = torch.empty_like(swx)
        for x in xs:
            xe = torch.zeros(ext, dtype=torch.float64, device=dev)
            so.own(xe).copy_(plan.owned(x, k))
            so.gazzola_weights(xe, 2.0, dx, dy, swx, swy)
        xe = torch.zeros(ext, dtype=torch.float64, device=dev)
        so.own(xe).copy_(plan.owned(xs[0], k))
        jx, jy = so.irn_weights_iso(xe, 1e-3, adopt=False)
        torch.cuda.synchronize()
        return [so.own(t).cpu().numpy() for t in (dx, dy, swx, swy, jx, jy)]

    outs = run_threads(plan, rank_fn)
    for k, got in enumerate(outs):
        for g, ref in zip(got, (Dx, Dy, wx, wy, ix, iy)):
            np.testing.assert_array_equal(g, plan.owned(ref, k).cpu().numpy())


@pytest.mark.parametrize("rule", ["gazzola", "irn_iso"])
def test_outer_steps_stepwise_handoff_f1_rules(torch_dev, rule):
    """Stepwise parity (reading G28) of the nested solve under the f1 weight rules: at
    every step the GPU starts from the oracle's state, runs step k, picks the same l*,
    and its own next_weights from the oracle's x* equal the oracle's W_{k+1} (and D_{k+1})
    bitwise (p = 2)."""
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = dataclasses.replace(S.CONFIGS["C1"], tol=1e-10, weight_rule=rule)
    inp = S.make_inputs(cfg)
    ref = opipe.run(cfg, inp, keep_steps=True)
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"], check_every=4)
    sol.set_data(_t(torch, dev, inp["x_true"]), _t(torch, dev, inp["xi"]))
    sol.reset_weights()
    n = cfg.n
    wx, wy = ops.identity_weights(n)
    D = ops.identity_weights(n)
    st = opipe.StepState(0, wx, wy, None, None, None)
    for k, rs in enumerate(ref["steps"]):
        sol.h.set_weights(_t(torch, dev, st.wx), _t(torch, dev, st.wy))
        o, X = sol.outer_step(k, _state_to_dev(torch, dev, st))
        assert np.all(o.status == 0), o.status
        assert o.lstar == rs.lstar, (k, o.lstar, rs.lstar)
        for l in range(cfg.M):
            xg = X["X_prev"][l].cpu().numpy()
            assert np.linalg.norm(xg - rs.X[:, l]) <= 1e-6 * np.linalg.norm(rs.X[:, l]), (k, l)
        xstar = rs.X[:, rs.lstar].reshape(n, n)
        if rule == "gazzola":
            sol.Dx.copy_(_t(torch, dev, D[0]))
            sol.Dy.copy_(_t(torch, dev, D[1]))
        sol.next_weights(_t(torch, dev, xstar))
        (wx, wy), Dn = opipe.next_weights(cfg, D, xstar)
        np.testing.assert_array_equal(sol.wx.cpu().numpy().reshape(n, n), wx)
        np.testing.assert_array_equal(sol.wy.cpu().numpy().reshape(n, n), wy)
        if rule == "gazzola":
            np.testing.assert_array_equal(sol.Dx.cpu().numpy().reshape(n, n), Dn[0])
            D = Dn
        st = opipe.StepState(k + 1, wx, wy, rs.X, rs.G, rs.V_i1)


def test_run_gazzola_with_lstar3_stop(torch_dev):
    """GpuSolver.run under Gazzola's rule + P:1042: the run ends at the first step that
    completes three equal l* (or K_out); every shift converged to the true residual bar."""
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = dataclasses.replace(S.CONFIGS["C1"], weight_rule="gazzola", stop="lstar3", K_out=8)
    inp = S.make_inputs(cfg)
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"], check_every=4)
    sol.set_data(_t(torch, dev, inp["x_true"]), _t(torch, dev, inp["xi"]))
    outs = sol.run()
    hist = [o.lstar for o in outs]
    for k in range(len(hist) - 1):
        assert not ops.lstar_settled(hist[:k + 1]), hist
    assert len(hist) == cfg.K_out or ops.lstar_settled(hist), hist
    for o in outs:
        assert np.all(o.status == 0)
        assert np.all(o.relres <= cfg.tol * (1 + 1e-6))
    wx = sol.wx.cpu().numpy()
    assert np.all((wx >= 0) & (wx <= 1))


def _state_to_dev(torch, dev, st):
    def m(a):
        return torch.from_numpy(np.ascontiguousarray(a.T, dtype=np.float64)).to(dev)
    out = {}
    if st.V_i1 is not None:
        out["V_i1"] = m(st.V_i1)
    if st.X_prev is not None:
        out["X_prev"] = m(st.X_prev)
        out["G_prev"] = m(st.G_prev)
    return out
