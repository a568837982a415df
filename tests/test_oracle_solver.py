"""Pins for oracle/defcg.py (O4), oracle/recycle.py (O5) and oracle/pipeline.py (O6)
against closed forms, dense solves, dense least squares and invariants."""
import math

import numpy as np
import pytest
import scipy.linalg
import scipy.sparse.linalg as spla

import rsk_synth as S
from oracle import defcg as dcg
from oracle import dense
from oracle import operators as ops
from oracle import pipeline
from oracle import recycle as rc


def _problem(n=8, r=2, sigma=1.0, seed=30, wlo=0.5, whi=20.0):
    h = S.gaussian_psf(r, sigma)
    wx, wy = S.random_weights(seed, n, wlo, whi)
    b = S.random_vectors(seed + 1, n * n)
    return h, wx, wy, b


def _Ag(h, wx, wy, g, n):
    return lambda v: ops.apply_shifted(h, wx, wy, g, v.reshape(n, n)).ravel()


@pytest.mark.parametrize("n,g", [(4, 0.5), (8, 0.05), (8, 3.0)])
def test_plain_cg_matches_dense_cholesky(n, g):
    h, wx, wy, b = _problem(n)
    Ad = dense.assemble_shifted(h, wx, wy, g, n)
    kappa = np.linalg.cond(Ad)
    x_ref = scipy.linalg.cho_solve(scipy.linalg.cho_factor(Ad), b)
    res = dcg.defcg(_Ag(h, wx, wy, g, n), b, tol=1e-12)
    assert res.status == dcg.CONVERGED
    err = np.linalg.norm(res.x - x_ref) / np.linalg.norm(x_ref)
    assert err <= 2 * kappa * 1e-12
    assert res.relres_true <= 1e-12


def test_plain_cg_agrees_with_scipy_cg():
    n, g = 8, 0.2
    h, wx, wy, b = _problem(n)
    op = spla.LinearOperator((n * n, n * n), matvec=_Ag(h, wx, wy, g, n), dtype=np.float64)
    xs, info = spla.cg(op, b, rtol=1e-13, atol=0.0, maxiter=5000)
    assert info == 0
    res = dcg.defcg(_Ag(h, wx, wy, g, n), b, tol=1e-13)
    assert np.linalg.norm(res.x - xs) <= 1e-9 * np.linalg.norm(xs)


@pytest.mark.parametrize("n", [4, 8])
def test_cg_finishes_within_N_steps_on_tiny_spd(n):
    h, wx, wy, b = _problem(n, r=1, sigma=0.7, wlo=1.0, whi=3.0)
    g = 1.0
    Ad = dense.assemble_shifted(h, wx, wy, g, n)
    assert np.linalg.cond(Ad) < 1e3
    res = dcg.defcg(_Ag(h, wx, wy, g, n), b, tol=1e-10)
    assert res.status == dcg.CONVERGED and res.iters <= n * n


def test_deflation_invariant_and_exact_eigvec_speedup():
    """U = eigenvectors of m isolated small eigenvalues: U^T r stays ~0, the count obeys the
    CG bound at kappa_eff = lambda_max / lambda_(m+1), and it drops by >= 25 % against
    U = empty (SPEC acceptance 3 analogue)."""
    rng = np.random.Generator(np.random.PCG64(31))
    N, m = 200, 4
    Q, _ = np.linalg.qr(rng.standard_normal((N, N)))
    lam = np.concatenate([[1e-5, 3e-5, 1e-4, 4e-4], np.linspace(1.0, 50.0, N - m)])
    Ad = (Q * lam) @ Q.T
    Ad = 0.5 * (Ad + Ad.T)
    b = rng.standard_normal(N)
    U = Q[:, :m]
    Z = Ad @ U
    tol = 1e-10
    plain = dcg.defcg(lambda v: Ad @ v, b, tol=tol)
    defl = dcg.defcg(lambda v: Ad @ v, b, U=U, Z=Z, tol=tol)
    assert plain.status == dcg.CONVERGED and defl.status == dcg.CONVERGED
    assert defl.iters <= 0.75 * plain.iters
    keff = lam[-1] / lam[m]
    assert defl.iters <= math.ceil(0.5 * math.sqrt(keff) * math.log(2.0 / tol)) + 2
    assert defl.utr_max <= 1e-12
    x_ref = np.linalg.solve(Ad, b)
    assert np.linalg.norm(defl.x - x_ref) <= 2 * np.linalg.cond(Ad) * tol * np.linalg.norm(x_ref)


def test_deflated_cg_with_initial_guess_and_random_space():
    n, g = 8, 0.01
    h, wx, wy, b = _problem(n)
    Ad = dense.assemble_shifted(h, wx, wy, g, n)
    U, _ = np.linalg.qr(S.random_vectors(40, (n * n, 5)))
    xp = S.random_vectors(41, n * n)
    res = dcg.defcg(_Ag(h, wx, wy, g, n), b, x_p=xp, U=U, Z=Ad @ U, tol=1e-11)
    assert res.status == dcg.CONVERGED
    assert res.utr_max <= 1e-12
    x_ref = np.linalg.solve(Ad, b)
    assert np.linalg.norm(res.x - x_ref) <= 2 * np.linalg.cond(Ad) * 1e-11 * np.linalg.norm(x_ref)


def test_zero_rhs_and_exact_guess():
    n, g = 6, 0.3
    h, wx, wy, b = _problem(n)
    res = dcg.defcg(_Ag(h, wx, wy, g, n), np.zeros(n * n))
    assert res.status == dcg.ZERO_RHS and res.iters == 0 and np.all(res.x == 0)
    Ad = dense.assemble_shifted(h, wx, wy, g, n)
    xs = np.linalg.solve(Ad, b)
    res = dcg.defcg(_Ag(h, wx, wy, g, n), b, x_p=xs, tol=1e-8)
    assert res.iters == 0 and res.status == dcg.CONVERGED and res.applies == 2


def test_non_spd_local_gram_drops_carried_column():
    n, g = 6, 0.3
    h, wx, wy, b = _problem(n)
    Ad = dense.assemble_shifted(h, wx, wy, g, n)
    U, _ = np.linalg.qr(S.random_vectors(42, (n * n, 3)))
    U = np.column_stack([U, U[:, 0]])          # duplicated column => G singular
    res = dcg.defcg(_Ag(h, wx, wy, g, n), b, U=U, Z=Ad @ U, tol=1e-10, n_carry=1)
    assert res.status == dcg.DEFL_DROPPED and res.m_used == 3


def test_store_holds_normalised_cg_residuals():
    n, g = 8, 0.01
    h, wx, wy, b = _problem(n)
    res = dcg.defcg(_Ag(h, wx, wy, g, n), b, tol=1e-10, store_cap=7)
    R = np.stack(res.store, 1)
    assert R.shape[1] == 7
    np.testing.assert_allclose(np.linalg.norm(R, axis=0), 1.0, rtol=1e-14)
    np.testing.assert_allclose(R[:, 0], b / np.linalg.norm(b), rtol=0, atol=1e-15)
    Gm = R.T @ R                               # CG residuals are mutually orthogonal
    assert np.max(np.abs(Gm - np.eye(7))) < 1e-8


# ---------------------------------------------------------------- shift family (§3.1)

def _pencil():
    n = 5
    h = S.gaussian_psf(1, 0.5)                 # 3x3, sigma 0.5 => A well conditioned (G26)
    wx, wy = S.random_weights(50, n, 0.5, 5.0)
    Ad = dense.assemble(lambda v: ops.apply_A(h, v), n)
    Ed = dense.assemble(lambda v: ops.apply_E(wx, wy, v), n)
    b = S.random_vectors(51, n * n)
    return Ad, Ed, b


def test_x_gamma_generalized_eigen_formula():
    """eq:x_gamma: x_gamma = sum_j v_j d~_j / (1 + gamma mu_j),
    E V = A V M, V^T A V = I, d~ = V^T b (= coefficients of d in the C V basis)."""
    Ad, Ed, b = _pencil()
    mu, V = scipy.linalg.eigh(Ed, Ad)          # E v = mu A v, V^T A V = I
    np.testing.assert_allclose(V.T @ Ad @ V, np.eye(len(b)), atol=1e-10)
    dt = V.T @ b
    assert np.min(np.abs(mu)) < 1e-10          # mu_N = 0 (null space of L)
    for g in (0.0, 1e-4, 1.0, 1e4):
        xg = V @ (dt / (1.0 + g * mu))
        xs = np.linalg.solve(Ad + g * Ed, b)
        assert np.linalg.norm(xg - xs) <= 1e-8 * np.linalg.norm(xs)


def test_shift_difference_identity():
    """eq:compare."""
    Ad, Ed, b = _pencil()
    mu, V = scipy.linalg.eigh(Ed, Ad)
    dt = V.T @ b
    ga, gb = 0.01, 3.0
    diff = np.linalg.solve(Ad + ga * Ed, b) - np.linalg.solve(Ad + gb * Ed, b)
    coef = (gb - ga) * mu / ((1 + gb * mu) * (1 + ga * mu))
    assert np.linalg.norm(diff - V @ (coef * dt)) <= 1e-9 * np.linalg.norm(diff)


# ---------------------------------------------------------------- recycle machinery

def test_stabilize_known_svd_cut():
    """A 30 x 10 block with sigma log-spaced 1..1e-18 keeps exactly the sigma_1/sigma_i < 1e10
    directions."""
    rng = np.random.Generator(np.random.PCG64(7))
    Qa, _ = np.linalg.qr(rng.standard_normal((30, 10)))
    Qb, _ = np.linalg.qr(rng.standard_normal((10, 10)))
    s = np.logspace(0, -18, 10)
    X = Qa @ np.diag(s) @ Qb.T
    # stabilize normalises columns first; undo by giving it already-normalised columns
    Xn = X / np.linalg.norm(X, axis=0)
    U = rc.stabilize(Xn)
    sv = np.linalg.svd(Xn, compute_uv=False)
    assert U.shape[1] == int(np.sum(sv[0] / sv < 1e10))
    np.testing.assert_allclose(U.T @ U, np.eye(U.shape[1]), atol=1e-13)
    assert rc.stabilize(Xn, cap=3).shape[1] == 3
    dup = np.column_stack([Xn[:, 0], Xn[:, 0], 2 * Xn[:, 0]])
    assert rc.stabilize(dup).shape[1] == 1      # duplicated column leaves one direction


def _anchor_problem(gamma_star=0.05, nc=7):
    n = 8
    h, wx, wy, b = _problem(n, r=2, sigma=1.0)
    Ut, _ = np.linalg.qr(S.random_vectors(60, (n * n, nc)))
    return n, h, wx, wy, b, Ut, rc.anchor(h, wx, wy, Ut, b, gamma_star, n)


def test_anchor_factors():
    n, h, wx, wy, b, Ut, an = _anchor_problem()
    Y = an.ZA + an.gamma_star * an.ZE
    np.testing.assert_allclose(an.K @ an.R, Y, atol=1e-13 * np.max(np.abs(Y)))
    np.testing.assert_allclose(an.K.T @ an.K, np.eye(Ut.shape[1]), atol=1e-13)
    assert np.all(np.diag(an.R) > 0) and np.allclose(an.R, np.triu(an.R))
    for j in range(Ut.shape[1]):
        img = Ut[:, j].reshape(n, n)
        np.testing.assert_allclose(an.ZE[:, j], ops.apply_E(wx, wy, img).ravel(), rtol=0, atol=1e-12)


@pytest.mark.parametrize("gamma", [0.0, 1e-4, 0.05, 0.3, 5.0, 100.0])
def test_orthupdate_guess_is_dense_least_squares_minimum(gamma):
    """eq:orthupdate gives the minimum-residual x_0 over Range(U~)."""
    n, h, wx, wy, b, Ut, an = _anchor_problem()
    Ag = dense.assemble_shifted(h, wx, wy, gamma, n)
    coef, *_ = np.linalg.lstsq(Ag @ Ut, b, rcond=None)
    x_ls = Ut @ coef
    x0 = rc.principal_guess(an, gamma)
    r_ls = np.linalg.norm(b - Ag @ x_ls); r0 = np.linalg.norm(b - Ag @ x0)
    assert abs(r0 - r_ls) <= 1e-9 * np.linalg.norm(b)
    assert np.linalg.norm(x0 - x_ls) <= 1e-7 * np.linalg.norm(x_ls)


def test_orthupdate_delta_zero_is_initX():
    """delta = 0 reduces to eq:initX: x_0 = U K^T b, r_0 = (I - K K^T) b."""
    n, h, wx, wy, b, Ut, an = _anchor_problem()
    c = rc.guess_coeffs(an, an.gamma_star)
    q = an.R @ c
    np.testing.assert_allclose(q, an.K.T @ b, rtol=1e-12, atol=1e-14)
    Ag = dense.assemble_shifted(h, wx, wy, an.gamma_star, n)
    r0 = b - Ag @ (Ut @ c)
    np.testing.assert_allclose(r0, b - an.K @ (an.K.T @ b), atol=1e-12)


def test_orthogonal_beats_oblique_and_cs_identity():
    """§7.1: ||r_1|| <= ||r_2|| and ||r_2||^2 = ||r_1||^2 + ||Omega^-1 Sigma Y_c^T b||^2."""
    n, h, wx, wy, b, Ut, an = _anchor_problem()
    gamma = 2.0
    d = gamma - an.gamma_star
    EU = dense.tri_inv_t_apply(an.R, an.ZE.T).T            # E U = Z_E R^-1
    Yfull = an.K + d * EU
    Y, Sm = np.linalg.qr(Yfull)
    r1 = b - Y @ (Y.T @ b)
    q2 = np.linalg.solve(an.K.T @ Y, an.K.T @ b)
    r2 = b - Y @ q2
    assert np.linalg.norm(r1) <= np.linalg.norm(r2) + 1e-14
    Phi, om, PsiT = np.linalg.svd(Y.T @ an.K)
    sig = np.sqrt(np.clip(1 - om ** 2, 0, None))
    KPsi = an.K @ PsiT.T
    Yc = KPsi - Y @ (Phi * om)
    with np.errstate(divide="ignore", invalid="ignore"):
        Yc = np.where(sig[None, :] > 1e-14, Yc / sig[None, :], 0.0)
    extra = np.linalg.norm((sig / om) * (Yc.T @ b)) ** 2
    assert abs(np.linalg.norm(r2) ** 2 - (np.linalg.norm(r1) ** 2 + extra)) <= 1e-10 * np.linalg.norm(b) ** 2
    # and the oracle's orthogonal guess residual equals ||r_1||
    Ag = dense.assemble_shifted(h, wx, wy, gamma, n)
    x0 = rc.principal_guess(an, gamma)
    assert np.linalg.norm(b - Ag @ x0) == pytest.approx(np.linalg.norm(r1), rel=1e-9)


@pytest.mark.parametrize("gamma", [1e-4, 0.05, 0.3, 2.0, 100.0])
def test_oblique_guess_petrov_galerkin_and_analysis(gamma):
    """eq:obliqueupdate: the oracle's oblique x_0 satisfies K^T r_0 = 0 with
    r_0 from the dense operator, and its residual is the r_2 of §7.1's analysis
    (q_2 = (K^T Y)^-1 K^T b with Y S = qr(K + delta E U))."""
    n, h, wx, wy, b, Ut, an = _anchor_problem()
    Ag = dense.assemble_shifted(h, wx, wy, gamma, n)
    x0 = rc.oblique_guess(an, gamma)
    r0 = b - Ag @ x0
    assert np.linalg.norm(an.K.T @ r0) <= 1e-11 * np.linalg.norm(b)
    d = gamma - an.gamma_star
    EU = dense.tri_inv_t_apply(an.R, an.ZE.T).T
    Y, _ = np.linalg.qr(an.K + d * EU)
    r2 = b - Y @ np.linalg.solve(an.K.T @ Y, an.K.T @ b)
    assert np.linalg.norm(r0) == pytest.approx(np.linalg.norm(r2), rel=1e-8)
    assert np.linalg.norm(r0) >= np.linalg.norm(b - Ag @ rc.principal_guess(an, gamma)) * (1 - 1e-12)


def test_oblique_guess_delta_zero_and_exact_range():
    """delta = 0: oblique == orthogonal == eq:initX. b in Range((A + gamma E) U~):
    both projections reproduce the exact solution (r_2 = r_1 = 0)."""
    n, h, wx, wy, b, Ut, an = _anchor_problem()
    c_o = rc.oblique_coeffs(an, an.gamma_star)
    np.testing.assert_allclose(c_o, rc.guess_coeffs(an, an.gamma_star), rtol=1e-12, atol=1e-14)
    gamma = 0.7
    Ag = dense.assemble_shifted(h, wx, wy, gamma, n)
    z = S.random_vectors(61, (Ut.shape[1],))
    bb = Ag @ (Ut @ z)
    an2 = rc.anchor(h, wx, wy, Ut, bb, an.gamma_star, n)
    for x0 in (rc.oblique_guess(an2, gamma), rc.principal_guess(an2, gamma)):
        np.testing.assert_allclose(x0, Ut @ z, rtol=0, atol=1e-9 * np.linalg.norm(Ut @ z))


def test_two_anchor_oblique_groups():
    """eq:updates: each group's guess is the oblique guess of its own anchor
    (K_L or K_R), so K_g^T r_0 = 0 per group; at the right anchor's own shift it is
    eq:initX for K_R."""
    n, h, wx, wy, b, Ut, an = _anchor_problem(gamma_star=0.01)
    gR = 3.0
    anR = rc.anchor(h, wx, wy, Ut, b, gR, n)
    for gamma, a in ((0.003, an), (0.02, an), (1.5, anR), (10.0, anR)):
        Ag = dense.assemble_shifted(h, wx, wy, gamma, n)
        r0 = b - Ag @ rc.oblique_guess(a, gamma)
        assert np.linalg.norm(a.K.T @ r0) <= 1e-11 * np.linalg.norm(b)
    AgR = dense.assemble_shifted(h, wx, wy, gR, n)
    r0 = b - AgR @ rc.oblique_guess(anR, gR)
    np.testing.assert_allclose(r0, b - anR.K @ (anR.K.T @ b), atol=1e-11 * np.linalg.norm(b))


def test_group_ritz_smallest_eigenpairs():
    n, h, wx, wy, b, Ut, an = _anchor_problem(nc=9)
    gJ = 0.7
    W, AW, EW, theta, Wt = rc.group_ritz(an, gJ, 3)
    Hd = Ut.T @ dense.assemble_shifted(h, wx, wy, gJ, n) @ Ut
    np.testing.assert_allclose(theta, np.linalg.eigvalsh(dense.sym(Hd))[:3], rtol=1e-12)
    np.testing.assert_allclose(W.T @ W, np.eye(3), atol=1e-13)
    Ad = dense.assemble(lambda v: ops.apply_A(h, v), n)
    np.testing.assert_allclose(AW, Ad @ W, atol=1e-12)


def test_carried_direction_orthogonal_and_duplicate_drop():
    rng = np.random.Generator(np.random.PCG64(8))
    W, _ = np.linalg.qr(rng.standard_normal((50, 4)))
    g = rng.standard_normal(50)
    gh = rc.carried_direction(W, g)
    assert np.linalg.norm(W.T @ gh) <= 1e-14 and abs(np.linalg.norm(gh) - 1) < 1e-14
    assert rc.carried_direction(W, W @ np.ones(4) + 1e-3 * g) is None
    assert rc.carried_direction(W, np.zeros(50)) is None


def test_ritz_space_on_diagonal_operator():
    """Diagonal operator: Ritz values from a Krylov store equal diagonal entries."""
    d = np.array([1.0, 2.0, 3.0, 5.0, 8.0, 13.0])
    b = np.ones(6)
    res = dcg.defcg(lambda v: d * v, b, tol=1e-14, store_cap=100)
    V, theta, _ = rc.ritz_space(lambda v: d * v, res.store, 3)
    np.testing.assert_allclose(theta, d[:3], rtol=1e-10)


# ---------------------------------------------------------------- L-curve / pipeline

def test_lcurve_corner_synthetic_L():
    """Two straight arms meeting at index 6: vertical arm then horizontal arm."""
    M = 12
    lr = np.array([0.0] * 6 + [0.0 + 0.5 * k for k in range(1, 7)])
    le = np.array([5.0 - 0.8 * k for k in range(6)] + [1.0] * 6)
    best, kappa = pipeline.lcurve_corner(np.exp(lr), np.exp(le))
    assert best in (5, 6)
    assert kappa[best] > 0


@pytest.mark.slow
def test_pipeline_tiny_matches_dense_every_step():
    cfg = S.small_config(n=10, M=6, r=2, sigma=1.0, n_c=8, J=2, K_out=3, tol=1e-10)
    inp = S.make_inputs(cfg)
    out = pipeline.run(cfg, inp, keep_steps=True)
    h = inp["psf"]; b = out["b"]; n = cfg.n
    wx, wy = ops.identity_weights(n)
    for k, st in enumerate(out["steps"]):
        assert np.all(st.status == dcg.CONVERGED)
        for l in range(cfg.M):
            Ad = dense.assemble_shifted(h, wx, wy, inp["gamma"][l], n)
            xs = np.linalg.solve(Ad, b)
            kap = np.linalg.cond(Ad)
            assert np.linalg.norm(st.X[:, l] - xs) <= max(2 * kap * cfg.tol, 1e-12) * np.linalg.norm(xs)
        xstar = st.X[:, st.lstar].reshape(n, n)
        wx, wy = ops.irn_weights(xstar, cfg.tau)

