"""Row-slab decomposition on one GPU with the ranks emulated as host
threads (ThreadComm: the host moves halo rows between launches, no kernel waits on
another rank): the slab apply equals the single-domain apply on every owned row
(<= 1e-13 relative, the apply bar), and the slab deflated CG reaches the same solutions
as the single-domain rsk_cg_recycled_batch (<= 1e-8 relative at tol 1e-10, iteration
counts +-max(2, 1%)) -- all-reduced sums, so not bitwise."""
import numpy as np
import pytest

import rsk_synth as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    return torch, torch.device("cuda", 0)


@pytest.mark.parametrize("n,r,nranks", [(64, 2, 2), (96, 3, 3), (128, 4, 4)])
def test_slab_apply_matches_single_domain(torch_dev, n, r, nranks):
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    from paper_2306_15049_b200.rsk import Handle
    from paper_2306_15049_b200.slab import SlabOps, SlabPlan, run_threads
    psf = S.gaussian_psf(r, 1.0 + 0.3 * r)
    wx, wy = S.random_weights(7 + n, n)
    wxd, wyd = (torch.from_numpy(np.ascontiguousarray(a.ravel())).to(dev) for a in (wx, wy))
    X = torch.from_numpy(S.random_vectors(11 + n, (3, n * n))).to(dev)
    gam = torch.tensor([0.0, 0.3, 40.0], dtype=torch.float64, device=dev)
    h = Handle(n, n, psf, 0)
    h.set_weights(wxd, wyd)
    Y = torch.empty_like(X)
    h.apply_shifted(X, Y, gamma=gam)
    Yc = torch.empty_like(X)
    h.apply_shifted(X, Yc, mode=L.RSK_APPLY_CT_ONLY)
    torch.cuda.synchronize()
    plan = SlabPlan(n, n, r, nranks)

    def rank_fn(k, comm):
        ops = SlabOps(plan, k, comm, psf, 0)
        ops.set_weights(wxd, wyd)
        Xe = plan.extend(X, k)
        Xe_own = ops.own(Xe).clone()
        Xe.zero_()                       # halo rows must come from the exchange
        ops.own(Xe).copy_(Xe_own)
        Ye = torch.empty_like(Xe)
        ops.apply(Xe, Ye, gam)
        Ze = torch.empty_like(Xe)
        ops.apply(Xe, Ze, mode=L.RSK_APPLY_CT_ONLY)
        torch.cuda.synchronize()
        return ops.own(Ye).cpu().numpy(), ops.own(Ze).cpu().numpy()

    outs = run_threads(plan, rank_fn)
    Yh, Ych = Y.cpu().numpy(), Yc.cpu().numpy()
    for k, (ys, zs) in enumerate(outs):
        sl = plan.slabs[k]
        ref = Yh[:, sl.row0 * n:sl.row1 * n]
        refc = Ych[:, sl.row0 * n:sl.row1 * n]
        assert np.max(np.abs(ys - ref)) <= 1e-13 * np.max(np.abs(Yh))
        assert np.max(np.abs(zs - refc)) <= 1e-13 * np.max(np.abs(Ych))


@pytest.mark.parametrize("nranks,J", [(2, 0), (2, 4), (4, 4)])
def test_slab_cg_matches_single_domain(torch_dev, nranks, J):
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    from paper_2306_15049_b200.pipeline import GpuSolver
    from paper_2306_15049_b200.slab import SlabOps, SlabPlan, run_threads, slab_cg
    cfg = S.small_config(n=64, M=4, r=3, sigma=1.3, tol=1e-10)
    inp = S.make_inputs(cfg)
    n, N = cfg.n, cfg.N
    sol = GpuSolver(cfg, inp["psf"], inp["gamma"], device=0)
    wx, wy = S.random_weights(5, n)
    wxd, wyd = (torch.from_numpy(np.ascontiguousarray(a.ravel())).to(dev) for a in (wx, wy))
    sol.h.set_weights(wxd, wyd)
    sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
    b = sol.b.clone()
    gidx = list(range(cfg.M))
    gam = np.asarray(inp["gamma"])[gidx]
    groups = None
    if J:
        Wr = torch.from_numpy(S.random_vectors(9, (J, N))).to(dev)
        W = torch.empty_like(Wr)
        sol.h.qr_tall(Wr.clone(), W)
        AW, EW = torch.empty_like(W), torch.empty_like(W)
        sol.h.apply_shifted(W, AW, EY=EW, mode=L.RSK_APPLY_SPLIT)
        groups = dict(W=[W], AW=[AW], EW=[EW], J=[J], of_shift=np.zeros(cfg.M, np.int32))
    X1 = torch.zeros(cfg.M, N, dtype=torch.float64, device=dev)
    res1 = sol.cg(gidx, X1, [0] * cfg.M, groups=groups)
    torch.cuda.synchronize()
    plan = SlabPlan(n, n, cfg.r, nranks)

    def rank_fn(k, comm):
        ops = SlabOps(plan, k, comm, inp["psf"], 0)
        ops.set_weights(wxd, wyd)
        be = plan.extend(b, k)
        Xe = torch.zeros(cfg.M, plan.slabs[k].ext_rows * n, dtype=torch.float64, device=dev)
        kw = {}
        if J:
            kw = dict(W=plan.owned(W, k).contiguous(), AW=plan.owned(AW, k).contiguous(),
                      EW=plan.owned(EW, k).contiguous())
        res = slab_cg(ops, gam, be, Xe, tol=cfg.tol, maxit=cfg.maxit, **kw)
        torch.cuda.synchronize()
        return res, ops.own(Xe).cpu().numpy()

    outs = run_threads(plan, rank_fn)
    X1h = X1.cpu().numpy()
    Xs = np.concatenate([o[1] for o in outs], axis=1)
    res = outs[0][0]
    for o in outs[1:]:
        np.testing.assert_array_equal(o[0]["iters"], res["iters"])   # replicated scalars
    # iteration counts: +-max(2, 1%) (reading G27: rounding order changes counts on the
    # slow, ill-conditioned shifts)
    tolit = np.maximum(2, np.ceil(0.01 * res1["iters"]))
    assert np.all(np.abs(res["iters"] - res1["iters"]) <= tolit), (res["iters"], res1["iters"])
    for l in range(cfg.M):
        rel = np.linalg.norm(Xs[l] - X1h[l]) / np.linalg.norm(X1h[l])
        assert rel <= 1e-8, (l, rel)
        assert res["relres_true"][l] <= cfg.tol * 1.0000001


@pytest.mark.parametrize("n,r,nranks", [(64, 2, 2), (96, 3, 3)])
def test_slab_irn_and_lcurve_norms_match_single_domain(torch_dev, n, r, nranks):
    """IRN weights (halo of x*), the L-curve seminorm eta^2 and residual rho^2 in slab mode
    against the single domain: weights bitwise on owned rows, norms <= 1e-13 relative."""
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    from paper_2306_15049_b200.rsk import Handle
    from paper_2306_15049_b200.slab import SlabOps, SlabPlan, run_threads
    psf = S.gaussian_psf(r, 1.0 + 0.3 * r)
    x = torch.from_numpy(S.random_vectors(3 + n, (n * n,))).to(dev)
    X = torch.from_numpy(S.random_vectors(4 + n, (2, n * n))).to(dev)
    d = torch.from_numpy(S.random_vectors(5 + n, (n * n,))).to(dev)
    tau = 1e-3
    h = Handle(n, n, psf, 0)
    wx = torch.empty(n * n, dtype=torch.float64, device=dev)
    wy = torch.empty_like(wx)
    h.irn_weights(x, tau, wx, wy)
    h.set_weights(wx, wy)
    eta = torch.empty(2, dtype=torch.float64, device=dev)
    h.seminorm_rows(X, 0, n, eta)
    Y = torch.empty_like(X)
    h.apply_shifted(X, Y, mode=L.RSK_APPLY_C_ONLY)
    rho2 = ((Y - d) ** 2).sum(1)
    torch.cuda.synchronize()
    plan = SlabPlan(n, n, r, nranks)

    def rank_fn(k, comm):
        so = SlabOps(plan, k, comm, psf, 0)
        xe = torch.zeros(plan.slabs[k].ext_rows * n, dtype=torch.float64, device=dev)
        so.own(xe).copy_(plan.owned(x, k))
        swx, swy = so.irn_weights(xe, tau)
        Xe = torch.zeros(2, plan.slabs[k].ext_rows * n, dtype=torch.float64, device=dev)
        so.own(Xe).copy_(plan.owned(X, k))
        de = plan.extend(d, k)
        e2 = so.seminorm2(Xe)
        r2 = so.resnorm2(Xe, de)
        torch.cuda.synchronize()
        return (so.own(swx).cpu().numpy(), so.own(swy).cpu().numpy(), e2.cpu().numpy(), r2.cpu().numpy())

    outs = run_threads(plan, rank_fn)
    for k, (a, b2, e2, r2) in enumerate(outs):
        np.testing.assert_array_equal(a, plan.owned(wx, k).cpu().numpy())
        np.testing.assert_array_equal(b2, plan.owned(wy, k).cpu().numpy())
        np.testing.assert_allclose(e2, eta.cpu().numpy(), rtol=1e-13)
        np.testing.assert_allclose(r2, rho2.cpu().numpy(), rtol=1e-13)


@pytest.mark.parametrize("nranks", [2, 3])
def test_slab_nested_outer_step_matches_single_domain(torch_dev, nranks):
    """The whole outer step (seeds, Ritz, stabilize, anchoring, guesses, groups, deflated CG,
    L-curve) in slab mode (SlabGpuSolver, ranks as threads) against the single-domain
    GpuSolver: same corner l*, iteration counts +-max(2, 2%), solutions <= 1e-7 relative."""
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    from paper_2306_15049_b200.slab import SlabGpuSolver, SlabPlan, run_threads
    cfg = S.small_config(n=48, M=6, r=3, sigma=1.2, n_c=10, J=3, K_out=1, tol=1e-10)
    inp = S.make_inputs(cfg)
    xt = torch.from_numpy(inp["x_true"]).to(dev)
    xi = torch.from_numpy(inp["xi"]).to(dev)
    ref = GpuSolver(cfg, inp["psf"], inp["gamma"], device=0)
    ref.set_data(xt, xi)
    o_ref = ref.run(K_out=1)[0]
    X_ref = ref.final["X_prev"].cpu().numpy()
    torch.cuda.synchronize()
    plan = SlabPlan(cfg.n, cfg.n, cfg.r, nranks)

    def rank_fn(k, comm):
        sol = SlabGpuSolver(cfg, inp["psf"], inp["gamma"], plan, k, comm, device=0)
        sol.set_data(xt, xi)
        o = sol.run(K_out=1)[0]
        torch.cuda.synchronize()
        return o, sol.o.own(sol.final["X_prev"]).cpu().numpy()

    outs = run_threads(plan, rank_fn)
    o = outs[0][0]
    Xs = np.concatenate([r[1] for r in outs], axis=1)
    assert o.lstar == o_ref.lstar
    tolit = np.maximum(2, np.ceil(0.02 * o_ref.iters))
    assert np.all(np.abs(o.iters - o_ref.iters) <= tolit), (o.iters, o_ref.iters)
    for l in range(cfg.M):
        rel = np.linalg.norm(Xs[l] - X_ref[l]) / np.linalg.norm(X_ref[l])
        assert rel <= 1e-7, (l, rel)


@pytest.mark.parametrize("n,r", [(512, 7), (520, 10)])
def test_apply_shifted_rows_matches_full_apply(torch_dev, n, r):
    """rsk_apply_shifted_rows (the row-slab overlap's interior / boundary applies): rows
    [row0, row1) equal to the whole-image apply (bit for bit when row0 is a multiple of 8,
    the whole apply's output-block grid; to 1e-13 otherwise), the other rows untouched,
    xdoty over the range's rows; and a cover of the image by ragged ranges reproduces the
    whole apply. Below the strip core's size the call declines (RSK_EUNSUPPORTED)."""
    torch, dev = torch_dev
    from paper_2306_15049_b200 import _lib as L
    from paper_2306_15049_b200.rsk import Handle
    psf = S.gaussian_psf(r, 1.0 + 0.3 * r)
    wx, wy = S.random_weights(5 + n, n)
    wxd, wyd = (torch.from_numpy(np.ascontiguousarray(a.ravel())).to(dev) for a in (wx, wy))
    X = torch.from_numpy(S.random_vectors(3 + n, (3, n * n))).to(dev)
    gam = torch.tensor([0.0, 0.7, 25.0], dtype=torch.float64, device=dev)
    h = Handle(n, n, psf, 0)
    h.set_weights(wxd, wyd)
    Y = torch.empty_like(X)
    h.apply_shifted(X, Y, gamma=gam)
    for row0, row1 in [(40, 301), (0, 8), (n - 24, n), (37, 301), (n - 21, n)]:
        Yr = torch.full_like(X, float("nan"))
        xd = torch.zeros(3, dtype=torch.float64, device=dev)
        assert h.apply_shifted_rows(X, Yr, row0, row1, gamma=gam, xdoty=xd)
        a, b = row0 * n, row1 * n
        if row0 % 8 == 0:   # the same 8-row output blocks as the whole apply: same bits
            assert torch.equal(Yr[:, a:b], Y[:, a:b]), (row0, row1)
        else:               # another grouping of the y-pass k-steps: the apply bar (1e-13)
            err = ((Yr[:, a:b] - Y[:, a:b]).abs().max(dim=1).values / Y[:, a:b].abs().max(dim=1).values)
            assert float(err.max()) <= 1e-13, (row0, row1, err)
        assert torch.isnan(Yr[:, :a]).all() and torch.isnan(Yr[:, b:]).all()
        ref = (X[:, a:b] * Y[:, a:b]).sum(dim=1)
        assert torch.allclose(xd, ref, rtol=1e-13, atol=0), (xd, ref)
    Ys = torch.full_like(X, float("nan"))
    EYs = torch.full_like(X, float("nan"))
    for row0, row1 in [(0, 16), (16, 248), (248, n)]:
        assert h.apply_shifted_rows(X, Ys, row0, row1, EY=EYs, mode=L.RSK_APPLY_SPLIT)
    Ya = torch.empty_like(X)
    EYa = torch.empty_like(X)
    h.apply_shifted(X, Ya, EY=EYa, mode=L.RSK_APPLY_SPLIT)
    assert torch.equal(Ys, Ya) and torch.equal(EYs, EYa)
    small = Handle(64, 64, psf, 0)
    Z = torch.zeros(1, 64 * 64, dtype=torch.float64, device=dev)
    assert not small.apply_shifted_rows(Z, torch.empty_like(Z), 8, 40, gamma=gam)
