"""Solver parity at BASELINE.json's full sizes, in the launch configurations the bench
and the nested solve use (the oracle runs its per-shift solves in forked processes, one
per host core -- its only parallelism, across shifts):

* C4 (1024 x 1024, 15 x 15 PSF, all 128 shifts, two groups of |J| = 12, carried columns,
  principal guesses) and C3 (512 x 512, 64 shifts, |J| = 10): the persistent lockstep loop
  over the whole ladder for a fixed 30 iterations; nine sampled shifts (C4: l = 1, 17,
  ..., 113, 128) are recomputed by the oracle
  one by one and compared element by element (the iterates of 30 CG steps agree to
  rounding: 1e-10 relative 2-norm) with the same apply accounting.
* C2 (256 x 256, 32 shifts): outer steps k = 0 and k = 1 stepwise (reading G28: the
  oracle's state after step 0 seeds the GPU's step 1), both sides at relres 1e-10:
  n_c and l* equal, iterations +-2 on >= 95 % of the shifts and +-max(2, 1 %) on all,
  solutions 1e-8 relative (north_star) -- a shift beyond 1e-8 must have a GPU solution
  whose true residual, recomputed by the oracle, meets the tolerance (reading G27:
  tolerance-limited), and at most 10 % of them may be.
"""
import dataclasses
import multiprocessing as mp
import os

import numpy as np
import pytest

import rsk_synth as S
from oracle import defcg as dcg
from oracle import operators as ops
from oracle import pipeline as opipe

pytestmark = pytest.mark.gpu
_CTX = {}
WORKERS = max(1, min(16, os.cpu_count() or 1))


def _t(torch, dev, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def _one_thread(fn, x):
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):   # one BLAS thread per worker: the workers are the parallelism
        return fn(x)


def _pmap(fn, items):
    import functools
    with mp.get_context("fork").Pool(min(len(items), WORKERS)) as pool:
        return pool.map(functools.partial(_one_thread, fn), items, chunksize=1)


def _img_A(v):
    n = _CTX["n"]
    return ops.apply_A(_CTX["psf"], v.reshape(n, n)).ravel()


def _img_E(v):
    n = _CTX["n"]
    return ops.apply_E(_CTX["wx"], _CTX["wy"], v.reshape(n, n)).ravel()


def _img_shift(a):
    v, g = a
    n = _CTX["n"]
    return ops.apply_shifted(_CTX["psf"], _CTX["wx"], _CTX["wy"], g, v.reshape(n, n)).ravel()


def _c4_oracle(l):
    c = _CTX
    n, g = c["n"], c["gam"][l]
    A = lambda v: ops.apply_shifted(c["psf"], c["wx"], c["wy"], g, v.reshape(n, n)).ravel()
    grp = c["grp"][l]
    U, Z = c["W"][grp], c["AW"][grp] + g * c["EW"][grp]
    nc = 0
    if l in c["gidx"]:
        j = c["gidx"].index(l)
        U = np.column_stack([U, c["gh"][:, j]]); Z = np.column_stack([Z, c["Zg"][:, j]]); nc = 1
    xp = c["xp"][:, l] if c["has_xp"][l] else None
    r = dcg.defcg(A, c["b"], x_p=xp, U=U, Z=Z, tol=c["tol"], maxit=c["maxit"], n_carry=nc)
    return r.x, r.iters, r.applies, r.status


@pytest.fixture(scope="module")
def torch_dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    return torch, torch.device("cuda", 0)


@pytest.mark.parametrize("cfgname", ["C3", "C4", "C5"])
def test_c4_full_ladder_fixed_iterations(torch_dev, cfgname):
    """C4 (and C3: 512^2, 64 shifts, |J| = 10, the same streaming loop at another
    geometry) -- the whole ladder for 30 lockstep iterations, sampled shifts by the oracle.
    C5 (4096^2, r = 10, 16 shifts, |J| = 8): the oracle's 21 x 21 convolution takes ~50 s
    per apply at this size, so 2 lockstep iterations and the two largest shifts (the
    survey's d4 plan for C5)."""
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    its = 2 if cfgname == "C5" else 30
    cfg = dataclasses.replace(S.CONFIGS[cfgname], tol=1e-30, maxit=its)
    inp = S.make_inputs(cfg)
    n, N, M, J = cfg.n, cfg.N, cfg.M, cfg.J
    psf, gam = inp["psf"], inp["gamma"]
    wx, wy = S.random_weights(4104, n, 1.0, 1.0 / cfg.tau)     # IRN-shaped: up to 1/tau
    rng = np.random.default_rng(4104)
    Wall, _ = np.linalg.qr(rng.standard_normal((N, 2 * J)))
    Ws = [Wall[:, :J], Wall[:, J:]]
    _CTX.clear()
    _CTX.update(n=n, psf=psf, wx=wx, wy=wy)
    cols = [Wall[:, j] for j in range(2 * J)]
    AWall = np.stack(_pmap(_img_A, cols), 1)
    EWall = np.stack(_pmap(_img_E, cols), 1)
    AWs, EWs = [AWall[:, :J], AWall[:, J:]], [EWall[:, :J], EWall[:, J:]]
    nL = int(round(0.75 * M))
    grp = np.array([0 if l < nL else 1 for l in range(M)], dtype=np.int32)
    sample = sorted(set([0] + [int(round(f * (M - 1))) for f in np.linspace(0.125, 1.0, 8)]))
    if cfgname == "C5":
        sample = [M - 2, M - 1]
    gidx = sorted(set(sample[::2] + [int(M * f) for f in (0.04, 0.31, 0.78, 0.94)]))   # carried columns
    gh = rng.standard_normal((N, len(gidx)))
    for j, l in enumerate(gidx):
        W = Ws[grp[l]]
        gh[:, j] -= W @ (W.T @ gh[:, j])
        gh[:, j] /= np.linalg.norm(gh[:, j])
    Zg = np.stack(_pmap(_img_shift, [(gh[:, j], gam[l]) for j, l in enumerate(gidx)]), 1)
    has_xp = (np.arange(M) % 3 != 0).astype(np.int32)
    xp = 0.01 * rng.standard_normal((N, M)) * has_xp

    sol = GpuSolver(cfg, psf, gam, check_every=8)
    sol.h.set_weights(_t(torch, dev, wx.ravel()), _t(torch, dev, wy.ravel()))
    sol.set_data(_t(torch, dev, inp["x_true"]), _t(torch, dev, inp["xi"]))
    b = sol.b.cpu().numpy()
    ghf = np.zeros((M, N)); zgf = np.zeros((M, N)); hg = np.zeros(M, dtype=np.int32)
    for j, l in enumerate(gidx):
        ghf[l], zgf[l], hg[l] = gh[:, j], Zg[:, j], 1
    groups = dict(W=[_t(torch, dev, W.T) for W in Ws], AW=[_t(torch, dev, A.T) for A in AWs],
                  EW=[_t(torch, dev, E.T) for E in EWs], of_shift=grp)
    X = _t(torch, dev, xp.T)
    res = sol.cg(list(range(M)), X, has_xp, groups=groups, ghat=(_t(torch, dev, ghf), _t(torch, dev, zgf), hg))
    assert int(res["prof"][7]) == 3, "the streaming lockstep loop (cg_stream.cu) must have run"
    Xs = X[sample].cpu().numpy()
    del X, groups, sol
    torch.cuda.empty_cache()
    _CTX.update(gam=gam, grp=grp, W=Ws, AW=AWs, EW=EWs, gidx=gidx, gh=gh, Zg=Zg, has_xp=has_xp, xp=xp,
                b=b, tol=cfg.tol, maxit=cfg.maxit)
    ref = _pmap(_c4_oracle, sample)
    for i, l in enumerate(sample):
        x, it, ap, st = ref[i]
        assert int(res["iters"][l]) == it == cfg.maxit, (l, res["iters"][l], it)
        assert int(res["applies"][l]) == ap, (l, res["applies"][l], ap)
        assert int(res["status"][l]) == st, (l, res["status"][l], st)
        rel = np.linalg.norm(Xs[i] - x) / np.linalg.norm(x)
        assert rel <= 1e-10, (l, rel)


def _c2_true_res(a):
    v, g = a
    return np.linalg.norm(_CTX["b"] - _img_shift((v, g))) / np.linalg.norm(_CTX["b"])


def test_c2_stepwise_k0_k1(torch_dev):
    torch, dev = torch_dev
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = dataclasses.replace(S.CONFIGS["C2"], tol=1e-10)
    inp = S.make_inputs(cfg)
    n, M = cfg.n, cfg.M
    h = inp["psf"]
    d, b2 = ops.make_data(h, inp["x_true"], inp["xi"], cfg.noise)
    b = b2.ravel()
    wx, wy = ops.identity_weights(n)
    st = opipe.StepState(0, wx, wy, None, None, None)
    sol = GpuSolver(cfg, h, inp["gamma"], check_every=8)
    sol.set_data(_t(torch, dev, inp["x_true"]), _t(torch, dev, inp["xi"]))
    limited = 0
    for k in range(2):
        rs = opipe.outer_step(cfg, h, b, d, inp["gamma"], st, workers=WORKERS)
        sol.h.set_weights(_t(torch, dev, st.wx.ravel()), _t(torch, dev, st.wy.ravel()))
        dst = {}
        if st.V_i1 is not None:
            dst = {"V_i1": _t(torch, dev, st.V_i1.T), "X_prev": _t(torch, dev, st.X_prev.T),
                   "G_prev": _t(torch, dev, st.G_prev.T)}
        o, X = sol.outer_step(k, dst)
        assert o.nc == rs.nc, (k, o.nc, rs.nc)
        assert np.all(o.status == 0) and np.all(rs.status == 0), (o.status, rs.status)
        assert o.lstar == rs.lstar, (k, o.lstar, rs.lstar)
        d_it = np.abs(o.iters - rs.iters)
        assert np.mean(d_it <= 2) >= 0.95 and np.all(d_it <= np.maximum(2, 0.01 * rs.iters)), (k, o.iters, rs.iters)
        Xg = X["X_prev"].cpu().numpy()
        rel = np.array([np.linalg.norm(Xg[l] - rs.X[:, l]) / np.linalg.norm(rs.X[:, l]) for l in range(M)])
        bad = [l for l in range(M) if rel[l] > 1e-8]
        if bad:
            _CTX.clear(); _CTX.update(n=n, psf=h, wx=st.wx, wy=st.wy, b=b)
            tr = _pmap(_c2_true_res, [(Xg[l], inp["gamma"][l]) for l in bad])
            for l, t in zip(bad, tr):
                assert t <= 1.01 * cfg.tol and rel[l] <= 1e-5, (k, l, rel[l], t)
            limited += len(bad)
        xstar = rs.X[:, rs.lstar].reshape(n, n)
        nwx, nwy = ops.irn_weights(xstar, cfg.tau)
        st = opipe.StepState(k + 1, nwx, nwy, rs.X, rs.G, rs.V_i1)
    assert limited <= 0.1 * 2 * M, f"{limited} tolerance-limited solutions"


def test_checkpoint_resume_is_bitwise(tmp_path):
    """SURVEY §5 (checkpoint / hand-off): the nested solve resumed from the on-disk state
    written after outer step 1 finishes with the same bits as the uninterrupted run (the
    state is everything step k+1 reads: W_{k+1}, W_k, X^(k), G^(k), V_i1, x*)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_2306_15049_b200.pipeline import GpuSolver
    cfg = S.CONFIGS["C1"]
    inp = S.make_inputs(cfg)
    dev = torch.device("cuda", 0)
    xt, xi = torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev)
    ck = str(tmp_path / "state.pt")

    sol = GpuSolver(cfg, inp["psf"], inp["gamma"])
    sol.set_data(xt, xi)
    full = sol.run(K_out=3)
    X_full = sol.final["X_prev"].clone()

    sol_a = GpuSolver(cfg, inp["psf"], inp["gamma"])
    sol_a.set_data(xt, xi)
    first = sol_a.run(K_out=2, checkpoint=ck)      # writes the state step 1 starts from
    assert len(first) == 2
    del sol_a
    sol_b = GpuSolver(cfg, inp["psf"], inp["gamma"])
    sol_b.set_data(xt, xi)
    k_next, _, lst = sol_b.load_state(ck)
    assert k_next == 1 and lst == [int(full[0].lstar)]
    rest = sol_b.run(K_out=3, resume=ck)
    assert [o.k for o in rest] == [1, 2]
    for o, ref in zip(rest, full[1:]):
        np.testing.assert_array_equal(o.iters, ref.iters)
        np.testing.assert_array_equal(o.applies, ref.applies)
        assert o.lstar == ref.lstar and o.nc == ref.nc
    assert torch.equal(sol_b.final["X_prev"], X_full)
    other = GpuSolver(S.CONFIGS["C2"], S.make_inputs(S.CONFIGS["C2"])["psf"], S.make_inputs(S.CONFIGS["C2"])["gamma"])
    with pytest.raises(ValueError):
        other.load_state(ck)
