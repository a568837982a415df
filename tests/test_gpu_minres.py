"""GPU parity of the recycling MINRES batch (rsk_minres_recycled_batch; the paper's inner
solver, eq:localU / eq:minShift / eq:xFinal P:473-534) against
oracle/minres.py on the same seeded inputs: per shift iterations +-2, solutions within
1e-8 relative (or the tolerance-limited bound 2 kappa tol, reading G27), statuses,
apply accounting, g = x - x_p; plus the nested solve with inner="minres" stepwise
against the oracle (reading G28)."""
import dataclasses

import numpy as np
import pytest

import rsk_synth as S
from oracle import dense
from oracle import minres as omr
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


def _setup(n, r, sigma, M, J, seed, ghat=True, xp=True):
    h = S.gaussian_psf(r, sigma)
    wx, wy = S.random_weights(seed, n, 0.5, 30.0)
    b = S.random_vectors(seed + 1, n * n)
    gam = np.logspace(-4, 1, M)
    rng = np.random.Generator(np.random.PCG64(seed + 2))
    # group blocks: W orthonormal, AW, EW their images (oracle operators)
    Wg, AWg, EWg = [], [], []
    for g in range(2):
        W, _ = np.linalg.qr(rng.standard_normal((n * n, J)))
        Wg.append(W)
        AWg.append(np.stack([ops.apply_A(h, W[:, j].reshape(n, n)).ravel() for j in range(J)], 1))
        EWg.append(np.stack([ops.apply_E(wx, wy, W[:, j].reshape(n, n)).ravel() for j in range(J)], 1))
    grp = np.array([0 if l < M // 2 else 1 for l in range(M)], dtype=np.int32)
    Gh = rng.standard_normal((n * n, M))
    Gh /= np.linalg.norm(Gh, axis=0)
    ZGh = np.stack([ops.apply_shifted(h, wx, wy, gam[l], Gh[:, l].reshape(n, n)).ravel() for l in range(M)], 1)
    has_g = np.array([1 if (ghat and l % 3 != 1) else 0 for l in range(M)], dtype=np.int32)
    Xp = 0.05 * rng.standard_normal((n * n, M)) if xp else np.zeros((n * n, M))
    has_xp = np.array([1 if (xp and l % 2 == 0) else 0 for l in range(M)], dtype=np.int32)
    return dict(h=h, wx=wx, wy=wy, b=b, gam=gam, W=Wg, AW=AWg, EW=EWg, grp=grp, Gh=Gh, ZGh=ZGh,
                has_g=has_g, Xp=Xp, has_xp=has_xp, n=n, J=J, M=M)


def _run_gpu(torch, dev, P, tol, maxit=20000, check_every=4, defl=True):
    from paper_2306_15049_b200 import _lib as L
    from paper_2306_15049_b200.rsk import Handle
    n, M, J = P["n"], P["M"], P["J"]
    N = n * n
    hd = Handle(n, n, P["h"], 0)
    hd.set_weights(_t(torch, dev, P["wx"].ravel()), _t(torch, dev, P["wy"].ravel()))
    b = _t(torch, dev, P["b"])
    X = _t(torch, dev, P["Xp"].T)
    G = torch.empty(M, N, dtype=torch.float64, device=dev)
    Wd = [_t(torch, dev, P["W"][g].T) for g in range(2)]
    AWd = [_t(torch, dev, P["AW"][g].T) for g in range(2)]
    EWd = [_t(torch, dev, P["EW"][g].T) for g in range(2)]
    Ghd = _t(torch, dev, P["Gh"].T)
    ZGhd = _t(torch, dev, P["ZGh"].T)
    d = L.CgDesc()
    gam = np.ascontiguousarray(P["gam"])
    hx = np.ascontiguousarray(P["has_xp"], dtype=np.int32)
    gos = np.ascontiguousarray(P["grp"], dtype=np.int32)
    hg = np.ascontiguousarray(P["has_g"], dtype=np.int32)
    d.nshift = M
    d.gamma_h = gam.ctypes.data_as(L._hp)
    d.b = b.data_ptr(); d.X = X.data_ptr(); d.ldx = N
    d.has_xp_h = hx.ctypes.data_as(L.C.POINTER(L.C.c_int))
    d.Gout = G.data_ptr(); d.ldg = N
    if defl:
        d.ngroups = 2
        d.group_of_shift_h = gos.ctypes.data_as(L.C.POINTER(L.C.c_int))
        for g in range(2):
            d.W[g] = Wd[g].data_ptr(); d.AW[g] = AWd[g].data_ptr(); d.EW[g] = EWd[g].data_ptr(); d.J[g] = J
        d.ldw = N
        d.Ghat = Ghd.data_ptr(); d.ZGhat = ZGhd.data_ptr(); d.ldgh = N
        d.has_ghat_h = hg.ctypes.data_as(L.C.POINTER(L.C.c_int))
    else:
        d.ngroups = 0
        d.flags = L.RSK_CG_NO_DEFLATION
    d.tol = tol; d.maxit = maxit; d.check_every = check_every
    out = L.CgOut()
    iters = np.zeros(M, np.int32); apl = np.zeros(M, np.int64); rel = np.zeros(M)
    stt = np.zeros(M, np.int32); mu = np.zeros(M, np.int32)
    P_ = L.C.POINTER
    out.iters = iters.ctypes.data_as(P_(L.C.c_int)); out.applies = apl.ctypes.data_as(P_(L.C.c_int64))
    out.relres_true = rel.ctypes.data_as(L._hp); out.status = stt.ctypes.data_as(P_(L.C.c_int))
    out.m_used = mu.ctypes.data_as(P_(L.C.c_int))
    kmax = (J + 1) if defl else 0   # (J of the call)
    ws = torch.empty(hd.minres_workspace_bytes(M, kmax), dtype=torch.uint8, device=dev)
    hd.get_counters(reset=True)
    hd.minres_recycled_batch(d, out, ws)
    torch.cuda.synchronize()
    cnt = hd.get_counters()
    assert int(cnt[0]) == int(apl.sum()) and int(cnt[1]) == int(apl.sum())
    return dict(X=X.cpu().numpy(), G=G.cpu().numpy(), iters=iters, applies=apl, relres=rel,
                status=stt, m_used=mu)


@pytest.mark.parametrize("n,r,sigma,defl,J", [(24, 2, 1.0, True, 4), (37, 3, 1.3, True, 4), (64, 4, 1.5, True, 4),
                                              (40, 3, 1.2, False, 4), (64, 3, 1.2, True, 16), (48, 2, 1.0, True, 10)])
def test_minres_batch_matches_oracle(torch_dev, n, r, sigma, defl, J):
    """Odd sizes (37: host-polled lockstep kernels), even ones (cluster loop), the local
    dimension at its maximum |J| + 1 = 17 and at the 10 / 11 boundary of the register
    arrays."""
    torch, dev = torch_dev
    tol = 1e-10
    P = _setup(n, r, sigma, M=6, J=J, seed=100 + n)
    res = _run_gpu(torch, dev, P, tol, defl=defl)
    for l in range(P["M"]):
        A = lambda v, g=P["gam"][l]: ops.apply_shifted(P["h"], P["wx"], P["wy"], g, v.reshape(n, n)).ravel()
        g = P["grp"][l]
        Ut = Z = None
        nc = 0
        if defl:
            Ut, Z = P["W"][g], P["AW"][g] + P["gam"][l] * P["EW"][g]
            if P["has_g"][l]:
                Ut = np.column_stack([Ut, P["Gh"][:, l]]); Z = np.column_stack([Z, P["ZGh"][:, l]]); nc = 1
        x0 = P["Xp"][:, l] if P["has_xp"][l] else None
        ref = omr.recycled_minres(A, P["b"], x0=x0, Ut=Ut, Z=Z, tol=tol, n_carry=nc)
        assert res["status"][l] == ref.status, (l, res["status"][l], ref.status)
        # reading G27's bar for every shift: +-max(2, 1 %) (the recursive residual's
        # crossing of tol moves by rounding over hundreds of Lanczos steps)
        assert abs(int(res["iters"][l]) - ref.iters) <= max(2, 0.01 * ref.iters), (l, res["iters"][l], ref.iters)
        assert res["m_used"][l] == ref.m_used
        assert res["relres"][l] <= tol
        rel = np.linalg.norm(res["X"][l] - ref.x) / np.linalg.norm(ref.x)
        if rel > 1e-8:
            Ad = dense.assemble_shifted(P["h"], P["wx"], P["wy"], P["gam"][l], n)
            ev = np.linalg.eigvalsh(Ad)
            assert rel <= 2 * ev[-1] / ev[0] * tol, (l, rel)
        # accounting: iters + r_p apply + confirmations (same rule as the oracle)
        assert res["applies"][l] - res["iters"][l] == ref.applies - ref.iters
        xp = P["Xp"][:, l] if P["has_xp"][l] else 0.0
        assert np.allclose(res["G"][l], res["X"][l] - xp, rtol=0, atol=1e-14 * np.abs(res["X"][l]).max())


def test_minres_zero_rhs_and_independence_of_batch(torch_dev):
    torch, dev = torch_dev
    P = _setup(32, 2, 1.0, M=5, J=3, seed=7)
    a = _run_gpu(torch, dev, P, 1e-9)
    # the same shifts solved in a different check cadence: bitwise the same x
    b2 = _run_gpu(torch, dev, P, 1e-9, check_every=1)
    assert np.array_equal(a["X"], b2["X"]) and np.array_equal(a["iters"], b2["iters"])
    P0 = dict(P); P0["b"] = np.zeros_like(P["b"])
    z = _run_gpu(torch, dev, P0, 1e-9)
    assert np.all(z["status"] == 4) and np.all(z["iters"] == 0) and np.all(z["X"] == 0)


@pytest.mark.parametrize("local", ["d3", "seq"])
def test_nested_solve_minres_stepwise(torch_dev, local):
    """inner="minres" in the whole outer step (C1, tol 1e-10), stepwise handoff; with
    local="seq" the local spaces carry g^(k,l-1) too (Alg. 3/4, wavefront per group)."""
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = dataclasses.replace(S.CONFIGS["C1"], tol=1e-10, inner="minres", local=local)
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
        dst = {}
        if st.V_i1 is not None:
            dst["V_i1"] = _t(torch, dev, st.V_i1.T)
        if st.X_prev is not None:
            dst["X_prev"] = _t(torch, dev, st.X_prev.T)
            dst["G_prev"] = _t(torch, dev, st.G_prev.T)
        o, X = sol.outer_step(k, dst)
        assert np.all((o.status == 0) | (o.status == 3)), o.status
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
        st = opipe.StepState(k + 1, wx, wy, rs.X, rs.G, rs.V_i1)
    assert np.mean(np.concatenate(all_d) <= 2) >= 0.95, all_d


def test_minres_store_spans_the_cg_residual_space_and_error_paths(torch_dev):
    """RSK_CG_STORE_RES with MINRES: the stored normalised Lanczos vectors equal the
    oracle's (up to rounding), span the same Krylov space as the CG's stored residuals,
    and the count is min(cap, iterations); a second carried column is rejected by the CG
    and a CT handle by rsk_cg_recycled_batch."""
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    from paper_2306_15049_b200.pipeline import GpuSolver, STORE_CAP
    from paper_2306_15049_b200.rsk import RskError
    cfg = dataclasses.replace(S.CONFIGS["C1"], tol=1e-10)
    inp = S.make_inputs(cfg)
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"])
    sol.set_data(_t(torch, dev, inp["x_true"].ravel()), _t(torch, dev, inp["xi"].ravel()))
    sol.reset_weights()
    N = cfg.N
    st_m = torch.empty(STORE_CAP, N, dtype=torch.float64, device=dev)
    st_c = torch.empty(STORE_CAP, N, dtype=torch.float64, device=dev)
    Xm = torch.zeros(1, N, dtype=torch.float64, device=dev)
    Xc = torch.zeros(1, N, dtype=torch.float64, device=dev)
    rm = sol.cg([0], Xm, [0], store=st_m, inner="minres")
    rc_ = sol.cg([0], Xc, [0], store=st_c)
    km, kc = int(rm["store_count"][0]), int(rc_["store_count"][0])
    assert km == min(STORE_CAP, int(rm["iters"][0])) and kc == min(STORE_CAP, int(rc_["iters"][0]))
    b = sol.b.cpu().numpy()
    wx, wy = ops.identity_weights(cfg.n)
    A = lambda v: ops.apply_shifted(inp["psf"], wx, wy, inp["gamma"][0], v.reshape(cfg.n, cfg.n)).ravel()
    ref = omr.recycled_minres(A, b, tol=cfg.tol, store_cap=STORE_CAP)
    Vm = st_m[:km].cpu().numpy()
    assert len(ref.store) == km
    for j in range(min(km, 10)):       # early Lanczos vectors: rounding has not grown yet
        assert np.linalg.norm(Vm[j] - ref.store[j]) <= 1e-9, j
    k = min(km, kc, 20)
    Qm, _ = np.linalg.qr(Vm[:k].T)
    Qc, _ = np.linalg.qr(st_c[:k].cpu().numpy().T)
    s = np.linalg.svd(Qm.T @ Qc, compute_uv=False)
    assert s.min() >= 1 - 1e-6            # the same Krylov space K_k(A_g, b)
    # a second carried column is MINRES-only
    G2 = torch.zeros(1, N, dtype=torch.float64, device=dev)
    with pytest.raises(RskError):
        sol.cg([0], Xc, [0], ghat2=(G2, G2, np.ones(1, np.int32)),
               groups=dict(W=[G2], AW=[G2], EW=[G2], of_shift=np.zeros(1, np.int32)))
    # CT handles: the CG device loops embed the stencil apply
    ctcfg = dataclasses.replace(S.CONFIGS["C6"], n=16, n_angles=20, M=2, inner="minres")
    ct = GpuSolver(ctcfg, None, S.gamma_ladder(ctcfg))
    X2 = torch.zeros(1, ctcfg.N, dtype=torch.float64, device=dev)
    with pytest.raises(RskError):
        ct.cg([0], X2, [0])


def test_minres_rank_deficient_local_space_drops_carried(torch_dev):
    """g-hat equal to a W column makes Z_l rank deficient: the carried column is dropped
    (status DEFL_DROPPED, m_used = J) and the solve still converges (as the oracle)."""
    torch, dev = torch_dev
    P = _setup(32, 2, 1.0, M=4, J=3, seed=5)
    for l in range(P["M"]):
        g = P["grp"][l]
        P["Gh"][:, l] = P["W"][g][:, 0]
        P["ZGh"][:, l] = P["AW"][g][:, 0] + P["gam"][l] * P["EW"][g][:, 0]
    P["has_g"][:] = 1
    res = _run_gpu(torch, dev, P, 1e-10)
    assert np.all(res["status"] == 3), res["status"]
    assert np.all(res["m_used"] == 3)
    assert np.all(res["relres"] <= 1e-10)
