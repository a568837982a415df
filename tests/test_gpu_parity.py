"""GPU parity: every librsk entry point against the oracle, element by element, on
seeded inputs at sizes spanning several tiles and a ragged tail, plus edge cases.
Tolerances: apply / projections <= 1e-13 relative inf-norm;
IRN weights <= 4 ulp; CG solutions (both at relres tol) <= 1e-8 relative 2-norm
(or the tolerance-limited bound 2 kappa tol when larger), iteration counts +-2."""
import math

import numpy as np
import pytest

import rsk_synth as S
from oracle import defcg as dcg
from oracle import operators as ops
from oracle import pipeline as opipe

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    return torch, torch.device("cuda", 0)


def _handle(n, psf):
    from paper_2306_15049_b200.rsk import Handle
    return Handle(n, n, psf, 0)


def _t(torch, dev, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def _rel_inf(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("n,r,sigma", [(37, 1, 0.8), (50, 2, 1.0), (96, 4, 1.5), (130, 4, 2.0),
                                       (75, 7, 3.0), (64, 10, 5.0), (256, 4, 2.0)])
def test_apply_shifted_all_modes(torch_dev, n, r, sigma):
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    psf = S.gaussian_psf(r, sigma)
    h = _handle(n, psf)
    wx, wy = S.random_weights(100 + n, n)
    h.set_weights(_t(torch, dev, wx.ravel()), _t(torch, dev, wy.ravel()))
    X = S.random_vectors(200 + n, (4, n * n))
    gam = np.array([0.0, 1e-5, 0.37, 250.0])
    Xd = _t(torch, dev, X)
    Y = torch.empty_like(Xd); EY = torch.empty_like(Xd); xy = torch.empty(4, dtype=torch.float64, device=dev)
    h.apply_shifted(Xd, Y, gamma=_t(torch, dev, gam), xdoty=xy)
    h.apply_shifted(Xd, EY.clone(), EY=EY, mode=L.RSK_APPLY_SPLIT)  # EY = E X (Y ignored)
    Yc = torch.empty_like(Xd); Yt = torch.empty_like(Xd)
    h.apply_shifted(Xd, Yc, mode=L.RSK_APPLY_C_ONLY)
    h.apply_shifted(Xd, Yt, mode=L.RSK_APPLY_CT_ONLY)
    torch.cuda.synchronize()
    Yh, EYh, Ych, Yth, xyh = (a.cpu().numpy() for a in (Y, EY, Yc, Yt, xy))
    for s in range(4):
        img = X[s].reshape(n, n)
        ref = ops.apply_shifted(psf, wx, wy, gam[s], img).ravel()
        assert _rel_inf(Yh[s], ref) <= 1e-13
        assert abs(xyh[s] - X[s] @ ref) <= 1e-13 * np.abs(X[s]) @ np.abs(ref)
        assert _rel_inf(EYh[s], ops.apply_E(wx, wy, img).ravel()) <= 1e-13
        assert _rel_inf(Ych[s], ops.conv(psf, img).ravel()) <= 1e-13
        assert _rel_inf(Yth[s], ops.conv_t(psf, img).ravel()) <= 1e-13


def test_apply_nonsymmetric_separable_psf(torch_dev):
    """Rank-1 but not point-symmetric PSF: catches flipped taps in C / C^T / B tables."""
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    n, r = 70, 3
    u = S.random_vectors(5, 2 * r + 1, "uniform") + 0.1
    v = S.random_vectors(6, 2 * r + 1, "uniform") + 0.1
    psf = np.outer(u, v)
    h = _handle(n, psf)
    X = S.random_vectors(7, (2, n * n))
    Xd = _t(torch, dev, X)
    Y = torch.empty_like(Xd)
    h.apply_shifted(Xd, Y, gamma=_t(torch, dev, [0.0, 0.0]))
    Yc = torch.empty_like(Xd); Yt = torch.empty_like(Xd)
    h.apply_shifted(Xd, Yc, mode=L.RSK_APPLY_C_ONLY)
    h.apply_shifted(Xd, Yt, mode=L.RSK_APPLY_CT_ONLY)
    for s in range(2):
        img = X[s].reshape(n, n)
        assert _rel_inf(Y[s].cpu().numpy(), ops.apply_A(psf, img).ravel()) <= 1e-13
        assert _rel_inf(Yc[s].cpu().numpy(), ops.conv(psf, img).ravel()) <= 1e-13
        assert _rel_inf(Yt[s].cpu().numpy(), ops.conv_t(psf, img).ravel()) <= 1e-13


def test_apply_invalid_arguments(torch_dev):
    torch, dev = torch_dev
    from paper_2306_15049_b200.rsk import RskError
    n = 40
    h = _handle(n, S.gaussian_psf(2, 1.0))
    X = torch.zeros(2, n * n, dtype=torch.float64, device=dev)
    with pytest.raises(RskError):
        h.apply_shifted(X, X, gamma=torch.zeros(2, dtype=torch.float64, device=dev))  # aliasing
    with pytest.raises(RskError):
        h.irn_weights(X[0], -1.0, eta2=torch.zeros(1, dtype=torch.float64, device=dev))


@pytest.mark.parametrize("N,k,nv", [(5000, 7, 3), (65536, 40, 40), (100003, 17, 1), (4096, 130, 9)])
def test_recycle_project(torch_dev, N, k, nv):
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    h = _handle(64, S.gaussian_psf(1, 1.0))
    U = S.random_vectors(300 + k, (k, N)); V = S.random_vectors(301 + nv, (nv, N))
    Ud, Vd = _t(torch, dev, U), _t(torch, dev, V)
    Cm = torch.empty(nv, k, dtype=torch.float64, device=dev)
    h.recycle_project(L.RSK_PROJ_UTV, Ud, Vd, Cm)
    ref = U @ V.T                                   # k x nv
    scale = np.abs(U) @ np.abs(V).T
    assert np.all(np.abs(Cm.cpu().numpy().T - ref) <= 1e-14 * scale + 1e-300)
    C2 = S.random_vectors(302, (nv, k))
    h.recycle_project(L.RSK_ADD_UC, Ud, Vd, _t(torch, dev, C2))
    V2 = V + C2 @ U
    assert _rel_inf(Vd.cpu().numpy(), V2) <= 1e-13
    h.recycle_project(L.RSK_SUB_UC, Ud, Vd, _t(torch, dev, C2))
    assert _rel_inf(Vd.cpu().numpy(), V) <= 1e-12


def test_irn_weights_and_seminorm(torch_dev):
    torch, dev = torch_dev
    n, tau = 77, 1e-3
    cfg = S.small_config(n=n)
    x = S.phantom(cfg, S.rng_for(cfg)) + 1e-3 * S.random_vectors(9, (n, n))
    h = _handle(n, S.gaussian_psf(2, 1.0))
    hw = S.random_weights(10, n)
    h.set_weights(_t(torch, dev, hw[0].ravel()), _t(torch, dev, hw[1].ravel()))
    wx = torch.empty(n * n, dtype=torch.float64, device=dev); wy = torch.empty_like(wx)
    e2 = torch.empty(1, dtype=torch.float64, device=dev)
    h.irn_weights(_t(torch, dev, x.ravel()), tau, wx, wy, e2)
    rx, ry = ops.irn_weights(x, tau)
    for got, ref in ((wx, rx), (wy, ry)):
        g = got.cpu().numpy().reshape(n, n)
        ulp = np.abs(g - ref) / np.maximum(np.spacing(np.abs(ref)), 1e-300)
        assert np.max(ulp[ref != 0]) <= 4
        assert np.all(g[ref == 0] == 0)
    assert float(e2.cpu()[0]) == pytest.approx(ops.seminorm2(hw[0], hw[1], x), rel=1e-13)


def test_make_rhs_and_qr_tall(torch_dev):
    torch, dev = torch_dev
    cfg = S.CONFIGS["C1"]
    inp = S.make_inputs(cfg)
    n = cfg.n
    h = _handle(n, inp["psf"])
    d = torch.empty(n * n, dtype=torch.float64, device=dev); b = torch.empty_like(d)
    h.make_rhs(_t(torch, dev, inp["x_true"].ravel()), _t(torch, dev, inp["xi"].ravel()), cfg.noise, d, b)
    dr, br = ops.make_data(inp["psf"], inp["x_true"], inp["xi"], cfg.noise)
    assert _rel_inf(d.cpu().numpy(), dr.ravel()) <= 1e-13
    assert _rel_inf(b.cpu().numpy(), br.ravel()) <= 1e-13
    # shifted Cholesky QR3 on an ill-conditioned block
    rng = np.random.default_rng(1)
    Qa, _ = np.linalg.qr(rng.standard_normal((5000, 12)))
    V = (Qa @ np.diag(np.logspace(0, -12, 12)) @ np.linalg.qr(rng.standard_normal((12, 12)))[0]).T
    Vd = _t(torch, dev, V); Q = torch.empty_like(Vd)
    R = h.qr_tall(Vd, Q)
    Qh = Q.cpu().numpy()
    assert np.max(np.abs(Qh @ Qh.T - np.eye(12))) <= 1e-13
    assert np.max(np.abs(Qh.T @ R - V.T)) <= 1e-13 * np.max(np.abs(V))
    assert np.all(np.diag(R) > 0)


def _oracle_cg(cfg, psf, wx, wy, b, gam, **kw):
    n = cfg.n
    A = lambda v: ops.apply_shifted(psf, wx, wy, gam, v.reshape(n, n)).ravel()
    return dcg.defcg(A, b, tol=cfg.tol, maxit=cfg.maxit, **kw)


def _kappa_bound(cfg, iters):
    return 1e-8


# the three implementations of the lockstep loop: cluster per shift (default at these
# sizes), persistent cooperative grid, host-polled kernels
LOOPS = {"cluster": {}, "persistent": {"RSK_CG_NOCLUSTER": "1", "RSK_CG_STREAM": "0"},
         "stream": {"RSK_CG_NOCLUSTER": "1", "RSK_CG_STREAM": "1"}, "hostpolled": {"RSK_CG_LEGACY": "1"}}


@pytest.mark.parametrize("loop", list(LOOPS))
@pytest.mark.parametrize("n", [40, 96])
def test_cg_plain_batch_matches_oracle(torch_dev, n, loop, monkeypatch):
    for k, v in LOOPS[loop].items():
        monkeypatch.setenv(k, v)
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = S.small_config(n=n, M=5, r=2, sigma=1.0, tol=1e-10)
    inp = S.make_inputs(cfg)
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"], check_every=3)
    sol.reset_weights()
    sol.set_data(_t(torch, dev, inp["x_true"]), _t(torch, dev, inp["xi"]))
    b = sol.b.cpu().numpy()
    X = torch.empty(cfg.M, cfg.N, dtype=torch.float64, device=dev)
    store = torch.empty(cfg.M * 100, cfg.N, dtype=torch.float64, device=dev)
    res = sol.cg(list(range(cfg.M)), X, [0] * cfg.M, store=store)
    wx, wy = ops.identity_weights(n)
    for l in range(cfg.M):
        o = _oracle_cg(cfg, inp["psf"], wx, wy, b, inp["gamma"][l], store_cap=100)
        assert res["status"][l] == 0 and o.status == 0
        assert abs(int(res["iters"][l]) - o.iters) <= 2
        assert np.linalg.norm(X[l].cpu().numpy() - o.x) <= 1e-8 * np.linalg.norm(o.x)
        assert res["relres"][l] <= cfg.tol
        cnt = int(res["store_count"][l])
        assert cnt == len(o.store) or abs(cnt - len(o.store)) <= 2
        st = store[l * 100:l * 100 + min(cnt, len(o.store), 10)].cpu().numpy()
        np.testing.assert_allclose(st, np.stack(o.store[:st.shape[0]]), atol=1e-9)


@pytest.mark.parametrize("loop,J", [(lp, 5) for lp in LOOPS] + [("cluster", 12), ("cluster", 16),
                                                                  ("persistent", 16), ("stream", 16)])
def test_cg_deflated_with_guess_and_carried_column(torch_dev, loop, J, monkeypatch):
    """All three loops at |J| = 5; the cluster loop's wide register path (|J| > 8) and the
    maximum local dimension |J| + 1 = 17."""
    for k, v in LOOPS[loop].items():
        monkeypatch.setenv(k, v)
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = S.small_config(n=64, M=4, r=3, sigma=1.3, tol=1e-10)
    inp = S.make_inputs(cfg)
    n, N, M = cfg.n, cfg.N, cfg.M
    psf = inp["psf"]
    sol = GpuSolver(cfg, psf, inp["gamma"], check_every=5)
    wx, wy = S.random_weights(77, n, 1.0, 300.0)
    sol.h.set_weights(_t(torch, dev, wx.ravel()), _t(torch, dev, wy.ravel()))
    sol.set_data(_t(torch, dev, inp["x_true"]), _t(torch, dev, inp["xi"]))
    b = sol.b.cpu().numpy()
    rng = np.random.default_rng(12)
    W, _ = np.linalg.qr(rng.standard_normal((N, J)))
    AW = np.stack([ops.apply_A(psf, W[:, j].reshape(n, n)).ravel() for j in range(J)], 1)
    EW = np.stack([ops.apply_E(wx, wy, W[:, j].reshape(n, n)).ravel() for j in range(J)], 1)
    gh = rng.standard_normal((N, M)); gh -= W @ (W.T @ gh); gh /= np.linalg.norm(gh, axis=0)
    gam = inp["gamma"]
    Zg = np.stack([ops.apply_shifted(psf, wx, wy, gam[l], gh[:, l].reshape(n, n)).ravel() for l in range(M)], 1)
    xp = 0.1 * rng.standard_normal((N, M))
    has_g = np.array([1, 0, 1, 1], dtype=np.int32)
    has_xp = np.array([1, 1, 0, 1], dtype=np.int32)
    X = _t(torch, dev, (xp * has_xp).T)
    G = torch.empty_like(X)
    groups = dict(W=[_t(torch, dev, W.T)], AW=[_t(torch, dev, AW.T)], EW=[_t(torch, dev, EW.T)],
                  of_shift=np.zeros(M, dtype=np.int32))
    res = sol.cg(list(range(M)), X, has_xp, Gout=G, groups=groups,
                 ghat=(_t(torch, dev, gh.T), _t(torch, dev, Zg.T), has_g))
    for l in range(M):
        U = W if not has_g[l] else np.column_stack([W, gh[:, l]])
        Z = AW + gam[l] * EW
        if has_g[l]:
            Z = np.column_stack([Z, Zg[:, l]])
        o = _oracle_cg(cfg, psf, wx, wy, b, gam[l], x_p=xp[:, l] if has_xp[l] else None, U=U, Z=Z,
                       n_carry=int(has_g[l]))
        assert res["status"][l] == 0 and o.status == 0
        assert abs(int(res["iters"][l]) - o.iters) <= 2, (res["iters"][l], o.iters)
        assert int(res["applies"][l]) - int(res["iters"][l]) == o.applies - o.iters
        xg = X[l].cpu().numpy()
        assert np.linalg.norm(xg - o.x) <= 1e-8 * np.linalg.norm(o.x)
        g_ref = o.x - (xp[:, l] if has_xp[l] else 0.0)
        assert np.linalg.norm(G[l].cpu().numpy() - g_ref) <= 1e-8 * np.linalg.norm(o.x)


def test_cg_zero_rhs(torch_dev):
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    from paper_2306_15049_b200 import _lib as L
    cfg = S.small_config(n=32, M=3)
    inp = S.make_inputs(cfg)
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"])
    sol.reset_weights()
    sol.b.zero_()
    X = torch.ones(cfg.M, cfg.N, dtype=torch.float64, device=dev)
    res = sol.cg(list(range(cfg.M)), X, [1] * cfg.M)
    assert np.all(res["status"] == L.RSK_CG_ZERO_RHS) and np.all(res["iters"] == 0)
    assert float(X.abs().max()) == 0.0


def _state_to_dev(torch, dev, st):
    out = {}
    if st.V_i1 is not None:
        out["V_i1"] = _t(torch, dev, st.V_i1.T)
    if st.X_prev is not None:
        out["X_prev"] = _t(torch, dev, st.X_prev.T)
        out["G_prev"] = _t(torch, dev, st.G_prev.T)
    return out


@pytest.mark.parametrize("cfgname", ["C1"])
def test_outer_steps_stepwise_handoff(torch_dev, cfgname):
    """Stepwise parity (reading G28): the oracle runs the IRN loop; at every step k the GPU
    starts from the oracle's state (W_k, X^(k-1), G^(k-1), V_i1) and runs step k itself.
    north_star: converged solutions, both sides at relative residual 1e-10, agree to 1e-8."""
    import dataclasses
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = dataclasses.replace(S.CONFIGS[cfgname], tol=1e-10)
    inp = S.make_inputs(cfg)
    ref = opipe.run(cfg, inp, keep_steps=True)
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"], check_every=4)
    sol.set_data(_t(torch, dev, inp["x_true"]), _t(torch, dev, inp["xi"]))
    n = cfg.n
    wx, wy = ops.identity_weights(n)
    st = opipe.StepState(0, wx, wy, None, None, None)
    total_it_gpu = total_it_ref = 0
    from oracle import dense
    limited = 0
    for k, rs in enumerate(ref["steps"]):
        sol.h.set_weights(_t(torch, dev, st.wx.ravel()), _t(torch, dev, st.wy.ravel()))
        o, X = sol.outer_step(k, _state_to_dev(torch, dev, st))
        assert o.nc == rs.nc
        assert np.all(o.status == 0), o.status
        Ad = dense.assemble(lambda v: ops.apply_A(inp["psf"], v), n)
        Ed = dense.assemble(lambda v: ops.apply_E(st.wx, st.wy, v), n)
        for l in range(cfg.M):
            xg = X["X_prev"][l].cpu().numpy()
            rel = np.linalg.norm(xg - rs.X[:, l]) / np.linalg.norm(rs.X[:, l])
            if rel > 1e-8:
                # reading G27: tolerance-limited when 2 kappa tol exceeds 1e-8 (both sides are
                # correct to their residual tolerance; they differ only in summation order)
                ev = np.linalg.eigvalsh(Ad + inp["gamma"][l] * Ed)
                bound = 2.0 * (ev[-1] / ev[0]) * cfg.tol
                assert rel <= bound, (k, l, rel, bound)
                limited += 1
            assert rel <= 1e-6, (k, l, rel)
        d_it = np.abs(o.iters - rs.iters)
        assert np.mean(d_it <= 2) >= 0.95 and np.all(d_it <= np.maximum(2, 0.01 * rs.iters)), (o.iters, rs.iters)
        assert o.lstar == rs.lstar
        total_it_gpu += int(o.iters.sum()); total_it_ref += int(rs.iters.sum())
        xstar = rs.X[:, rs.lstar].reshape(n, n)
        wx, wy = ops.irn_weights(xstar, cfg.tau)
        st = opipe.StepState(k + 1, wx, wy, rs.X, rs.G, rs.V_i1)
    assert abs(total_it_gpu - total_it_ref) <= 0.02 * total_it_ref + 4
    assert limited <= 0.1 * cfg.M * cfg.K_out, f"{limited} tolerance-limited solutions"


@pytest.mark.parametrize("n,r,sigma", [(50, 2, 1.0), (96, 4, 1.5), (130, 4, 2.0), (64, 10, 5.0),
                                       (200, 7, 3.0), (72, 12, 5.0), (136, 1, 0.8)])
def test_apply_strip_core_shifted_and_split(torch_dev, monkeypatch, n, r, sigma):
    """The streaming strip core (strip_core.cuh; default for N >= 512^2) forced at small,
    ragged sizes: several strips with a partial last strip, several 8-row blocks with a
    ragged last block, the top / bottom / left / right zero-boundary corrections."""
    monkeypatch.setenv("RSK_APPLY_STRIP", "1")
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    psf = S.gaussian_psf(r, sigma)
    h = _handle(n, psf)
    wx, wy = S.random_weights(300 + n, n)
    h.set_weights(_t(torch, dev, wx.ravel()), _t(torch, dev, wy.ravel()))
    nv = 5
    X = S.random_vectors(400 + n, (nv, n * n))
    gam = np.array([0.0, 1e-6, 0.5, 3.0, 700.0])
    Xd = _t(torch, dev, X)
    Y = torch.empty_like(Xd); AY = torch.empty_like(Xd); EY = torch.empty_like(Xd)
    xy = torch.empty(nv, dtype=torch.float64, device=dev)
    h.apply_shifted(Xd, Y, gamma=_t(torch, dev, gam), xdoty=xy)
    h.apply_shifted(Xd, AY, EY=EY, mode=L.RSK_APPLY_SPLIT)
    torch.cuda.synchronize()
    Yh, AYh, EYh, xyh = (a.cpu().numpy() for a in (Y, AY, EY, xy))
    for s in range(nv):
        x = X[s].reshape(n, n)
        ref = ops.apply_shifted(psf, wx, wy, gam[s], x)
        assert _rel_inf(Yh[s].reshape(n, n), ref) <= 1e-13, s
        assert _rel_inf(AYh[s].reshape(n, n), ops.apply_A(psf, x)) <= 1e-13, s
        assert _rel_inf(EYh[s].reshape(n, n), ops.apply_E(wx, wy, x)) <= 1e-13, s
        assert abs(xyh[s] - float(np.sum(x * ref))) <= 1e-13 * float(np.sum(np.abs(x) * np.abs(ref))), s


def test_set_weights_rejects_invalid(torch_dev):
    """rsk_set_weights (include/rsk.h): non-finite / negative weights and non-zero pads
    return RSK_EINVAL and leave the handle's weights (hence E_k) unchanged."""
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    from paper_2306_15049_b200.rsk import RskError
    n = 24
    psf = S.gaussian_psf(2, 1.0)
    h = _handle(n, psf)
    wx, wy = S.random_weights(5, n)
    h.set_weights(_t(torch, dev, wx.ravel()), _t(torch, dev, wy.ravel()))
    X = _t(torch, dev, S.random_vectors(6, (1, n * n)))
    E0 = torch.empty_like(X); A0 = torch.empty_like(X)
    h.apply_shifted(X, A0, EY=E0, mode=L.RSK_APPLY_SPLIT)
    bad = []
    for kind in ("nan", "inf", "neg", "padx", "pady"):
        bx, by = wx.copy(), wy.copy()
        if kind == "nan": bx[3, 4] = np.nan
        if kind == "inf": by[5, 6] = np.inf
        if kind == "neg": bx[7, 1] = -1e-3
        if kind == "padx": bx[2, n - 1] = 1.0
        if kind == "pady": by[n - 1, 3] = 2.0
        with pytest.raises(RskError) as ei:
            h.set_weights(_t(torch, dev, bx.ravel()), _t(torch, dev, by.ravel()))
        assert ei.value.status == L.RSK_EINVAL, kind
        bad.append(kind)
    E1 = torch.empty_like(X); A1 = torch.empty_like(X)
    h.apply_shifted(X, A1, EY=E1, mode=L.RSK_APPLY_SPLIT)
    torch.cuda.synchronize()
    assert torch.equal(E0, E1) and len(bad) == 5


@pytest.mark.parametrize("n", [128, 75])
def test_apply_rank2_psf_all_modes(torch_dev, n):
    """Rank-2 PSF (Example 1's C = sum_i C_i^(1) (x) C_i^(2), config C7): rsk_create finds
    the two separable terms; every apply mode against the oracle's literal 2-D conv."""
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    psf = S.make_inputs(S.CONFIGS["C7"])["psf"]
    h = _handle(n, psf)
    wx, wy = S.random_weights(500 + n, n)
    h.set_weights(_t(torch, dev, wx.ravel()), _t(torch, dev, wy.ravel()))
    nv = 3
    X = S.random_vectors(600 + n, (nv, n * n))
    gam = np.array([0.0, 1e-3, 40.0])
    Xd = _t(torch, dev, X)
    Y = torch.empty_like(Xd); AY = torch.empty_like(Xd); EY = torch.empty_like(Xd)
    Yc = torch.empty_like(Xd); Yt = torch.empty_like(Xd)
    xy = torch.empty(nv, dtype=torch.float64, device=dev)
    h.apply_shifted(Xd, Y, gamma=_t(torch, dev, gam), xdoty=xy)
    h.apply_shifted(Xd, AY, EY=EY, mode=L.RSK_APPLY_SPLIT)
    h.apply_shifted(Xd, Yc, mode=L.RSK_APPLY_C_ONLY)
    h.apply_shifted(Xd, Yt, mode=L.RSK_APPLY_CT_ONLY)
    torch.cuda.synchronize()
    for s in range(nv):
        x = X[s].reshape(n, n)
        ref = ops.apply_shifted(psf, wx, wy, gam[s], x)
        assert _rel_inf(Y[s].cpu().numpy().reshape(n, n), ref) <= 1e-13
        assert _rel_inf(AY[s].cpu().numpy().reshape(n, n), ops.apply_A(psf, x)) <= 1e-13
        assert _rel_inf(EY[s].cpu().numpy().reshape(n, n), ops.apply_E(wx, wy, x)) <= 1e-13
        assert _rel_inf(Yc[s].cpu().numpy().reshape(n, n), ops.conv(psf, x)) <= 1e-13
        assert _rel_inf(Yt[s].cpu().numpy().reshape(n, n), ops.conv_t(psf, x)) <= 1e-13
        assert abs(float(xy[s]) - float(np.sum(x * ref))) <= 1e-13 * float(np.sum(np.abs(x) * np.abs(ref)))


def test_rank3_psf_unsupported_and_rank2_cg_refused(torch_dev):
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    from paper_2306_15049_b200.rsk import RskError
    rng = np.random.default_rng(3)
    h3 = rng.random((7, 7))           # generic: rank 7
    with pytest.raises(RskError):
        _handle(40, h3)
    cfg = S.CONFIGS["C7"]
    import dataclasses
    cfg = dataclasses.replace(cfg, n=48, M=4, inner="cg")
    from paper_2306_15049_b200.pipeline import GpuSolver
    inp = S.make_inputs(S.CONFIGS["C7"])
    sol = GpuSolver(cfg, inp["psf"], np.logspace(-3, 0, 4))
    sol.reset_weights()
    X = torch.zeros(4, cfg.N, dtype=torch.float64, device=dev)
    with pytest.raises(RskError) as ei:
        sol.cg(list(range(4)), X, [0] * 4)
    assert ei.value.status == L.RSK_EUNSUPPORTED
