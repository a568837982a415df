"""Pins for oracle/minres.py (recycling MINRES, eq:minShift / eq:xFinal, P:454-534;
SURVEY §8(f) f2(ii)) against things other than itself: dense minimum-residual problems
over explicitly built bases, scipy's MINRES, dense solves, and the invariants the paper's
construction implies (K^T r = 0 after eq:xFinal, monotone LS residuals)."""
import numpy as np
import pytest
import scipy.linalg

from oracle.indices import of as _ixof
import scipy.sparse.linalg as spla

import rsk_synth as S
from oracle import dense
from oracle import minres as mr
from oracle import operators as ops


def _problem(n=8, r=2, sigma=1.0, seed=40, wlo=0.5, whi=20.0):
    h = S.gaussian_psf(r, sigma)
    wx, wy = S.random_weights(seed, n, wlo, whi)
    b = S.random_vectors(seed + 1, n * n)
    return h, wx, wy, b


def _Ag(h, wx, wy, g, n):
    return lambda v: ops.apply_shifted(h, wx, wy, g, v.reshape(n, n)).ravel()


def _krylov_basis(op, v, m):
    """Orthonormal basis of span{v, op v, ..., op^(m-1) v} built from explicit powers
    (independent of any Lanczos recurrence; small m only)."""
    cols = [v / np.linalg.norm(v)]
    for _ in range(m - 1):
        cols.append(op(cols[-1]))
        cols[-1] = cols[-1] / np.linalg.norm(cols[-1])
    Q, _ = np.linalg.qr(np.stack(cols, 1))
    return Q


@pytest.mark.parametrize("m", [1, 3, 6])
def test_plain_minres_iterate_is_the_krylov_min_residual(m):
    """U = empty: the m-th iterate minimises ||b - A_g x|| over x in K_m(A_g, b)."""
    n, g = 8, 0.3
    h, wx, wy, b = _problem(n)
    Ad = dense.assemble_shifted(h, wx, wy, g, n)
    res = mr.recycled_minres(lambda v: Ad @ v, b, tol=1e-300, maxit=m)
    assert res.iters == m and res.status == mr.MAXIT
    Q = _krylov_basis(lambda v: Ad @ v, b, m)
    c = np.linalg.lstsq(Ad @ Q, b, rcond=None)[0]
    x_ref = Q @ c
    assert np.linalg.norm(res.x - x_ref) <= 1e-10 * np.linalg.norm(x_ref)
    assert abs(res.res_hist[-1] - np.linalg.norm(b - Ad @ x_ref)) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("m", [1, 4])
def test_recycled_iterate_is_min_residual_over_U_plus_projected_krylov(m):
    """eq:minShift: x_0 + g with g the minimiser of ||r - A_g g|| over
    Range([U, V_m]), V_m spanning K_m((I - KK^T) A_g, (I - KK^T) r)."""
    n, g = 8, 0.1
    h, wx, wy, b = _problem(n, seed=41)
    Ad = dense.assemble_shifted(h, wx, wy, g, n)
    rng = np.random.Generator(np.random.PCG64(7))
    Ut = rng.standard_normal((n * n, 3))
    x0 = 0.01 * rng.standard_normal(n * n)
    Z = Ad @ Ut
    res = mr.recycled_minres(lambda v: Ad @ v, b, x0=x0, Ut=Ut, Z=Z, tol=1e-300, maxit=m)
    r = b - Ad @ x0
    Kq, _ = np.linalg.qr(Z)
    P = np.eye(n * n) - Kq @ Kq.T
    V = _krylov_basis(lambda v: P @ (Ad @ v), P @ r, m)
    B = np.concatenate([Ut, V], 1)
    c = np.linalg.lstsq(Ad @ B, r, rcond=None)[0]
    x_ref = x0 + B @ c
    assert np.linalg.norm(res.x - x_ref) <= 1e-9 * np.linalg.norm(x_ref)
    # eq:xFinal makes the final residual orthogonal to K_l = Range(A_g U~)
    assert np.linalg.norm(Kq.T @ (b - Ad @ res.x)) <= 1e-11 * np.linalg.norm(b)


def test_minres_agrees_with_scipy_minres_and_dense_solve():
    n, g = 8, 0.2
    h, wx, wy, b = _problem(n)
    Ad = dense.assemble_shifted(h, wx, wy, g, n)
    x_ref = scipy.linalg.cho_solve(scipy.linalg.cho_factor(Ad), b)
    kappa = np.linalg.cond(Ad)
    op = spla.LinearOperator((n * n, n * n), matvec=lambda v: Ad @ v, dtype=np.float64)
    xs, info = spla.minres(op, b, rtol=1e-12, maxiter=5000)
    res = mr.recycled_minres(lambda v: Ad @ v, b, tol=1e-12)
    assert res.status == mr.CONVERGED and res.relres_true <= 1e-12
    assert np.linalg.norm(res.x - x_ref) <= 2 * kappa * 1e-12 * np.linalg.norm(x_ref)
    assert np.linalg.norm(res.x - xs) <= 4 * kappa * 1e-12 * np.linalg.norm(x_ref)


def test_ls_residuals_nonincreasing_and_equal_true_residual():
    n, g = 8, 1e-3
    h, wx, wy, b = _problem(n, seed=43)
    A = _Ag(h, wx, wy, g, n)
    res = mr.recycled_minres(A, b, tol=1e-10)
    hst = np.asarray(res.res_hist)
    assert np.all(np.diff(hst) <= 1e-12 * np.linalg.norm(b))
    assert res.status == mr.CONVERGED
    assert abs(res.relres_true - hst[-1] / np.linalg.norm(b)) <= 1e-9


@pytest.mark.parametrize("n", [4, 6])
def test_tiny_spd_converges_within_N_minus_k_steps(n):
    h, wx, wy, b = _problem(n, r=1, sigma=0.7, wlo=1.0, whi=3.0)
    g = 1.0
    Ad = dense.assemble_shifted(h, wx, wy, g, n)
    rng = np.random.Generator(np.random.PCG64(9))
    Ut = rng.standard_normal((n * n, 2))
    res = mr.recycled_minres(lambda v: Ad @ v, b, Ut=Ut, Z=Ad @ Ut, tol=1e-10)
    assert res.status == mr.CONVERGED
    assert res.iters <= n * n - 2 + 1
    x_ref = np.linalg.solve(Ad, b)
    assert np.linalg.norm(res.x - x_ref) <= 2 * np.linalg.cond(Ad) * 1e-10 * np.linalg.norm(x_ref)


def test_exact_eigenvectors_deflate_the_small_eigenvalues():
    """U = eigenvectors of isolated small eigenvalues: the count drops by >= 25 %
    against U = empty and obeys the MINRES bound at kappa_eff = lam_max / lam_(m+1)."""
    rng = np.random.Generator(np.random.PCG64(31))
    N, m = 200, 4
    Q, _ = np.linalg.qr(rng.standard_normal((N, N)))
    lam = np.concatenate([[1e-5, 3e-5, 1e-4, 4e-4], np.linspace(1.0, 50.0, N - m)])
    Ad = (Q * lam) @ Q.T
    Ad = 0.5 * (Ad + Ad.T)
    b = rng.standard_normal(N)
    U = Q[:, :m]
    tol = 1e-10
    plain = mr.recycled_minres(lambda v: Ad @ v, b, tol=tol)
    defl = mr.recycled_minres(lambda v: Ad @ v, b, Ut=U, Z=Ad @ U, tol=tol)
    assert plain.status == mr.CONVERGED and defl.status == mr.CONVERGED
    assert defl.iters <= 0.75 * plain.iters
    keff = lam[-1] / lam[m]
    # MINRES residual bound 2((sqrt(k)-1)/(sqrt(k)+1))^j (j even steps of a CG-type bound)
    q = (np.sqrt(keff) - 1) / (np.sqrt(keff) + 1)
    bound = int(np.ceil(np.log(tol / 2) / np.log(q))) + 2
    assert defl.iters <= bound


def test_block_ls_decouples_as_the_paper_states():
    """The first block row of eq:minShift is solved exactly: with K = A_g U
    (eq:localU) the residual of x = x_0 + y_m + U K^T (r - A_g y_m) (eq:xFinal) is
    (I - KK^T)(r - A_g y_m), so the LS residual of the y-block alone (res_hist) is the
    true residual, and K^T (b - A_g x) = 0."""
    n, g = 6, 0.05
    h, wx, wy, b = _problem(n, seed=44)
    Ad = dense.assemble_shifted(h, wx, wy, g, n)
    rng = np.random.Generator(np.random.PCG64(3))
    Ut = rng.standard_normal((n * n, 2))
    Z = Ad @ Ut
    res = mr.recycled_minres(lambda v: Ad @ v, b, Ut=Ut, Z=Z, tol=1e-300, maxit=5)
    K, R = mr.local_factor(Z)
    U = Ut @ np.linalg.inv(R)
    assert np.allclose(Ad @ U, K, atol=1e-12)      # eq:localU: A_g U = K
    rt = b - Ad @ res.x
    assert np.linalg.norm(K.T @ rt) <= 1e-12 * np.linalg.norm(b)
    assert abs(np.linalg.norm(rt) - res.res_hist[-1]) <= 1e-11 * np.linalg.norm(b)


def test_zero_rhs_and_carried_column_drop():
    n = 4
    h, wx, wy, _ = _problem(n)
    A = _Ag(h, wx, wy, 0.5, n)
    res = mr.recycled_minres(A, np.zeros(n * n))
    assert res.status == mr.ZERO_RHS and res.iters == 0 and np.all(res.x == 0)
    b = S.random_vectors(5, n * n)
    Ut = S.random_vectors(6, (n * n, 2))
    Ut = np.concatenate([Ut, Ut[:, :1]], 1)          # duplicated carried column: R_l singular
    Z = np.stack([A(Ut[:, i]) for i in range(3)], 1)
    res = mr.recycled_minres(A, b, Ut=Ut, Z=Z, n_carry=1, tol=1e-10)
    assert res.status == mr.DEFL_DROPPED and res.m_used == 2 and res.relres_true <= 1e-10


@pytest.mark.parametrize("local", ["d3", "seq"])
def test_pipeline_minres_tiny_matches_dense_every_step(local):
    """The nested solve with the paper's inner solver (inner="minres") and with its
    sequential local spaces [W, g^(k-1,l), g^(k,l-1)] (Alg. 3/4, local="seq"): every
    (k, l) solution within 2 kappa tol of the dense solve of eq:seqsys."""
    import dataclasses
    from oracle import pipeline
    cfg = dataclasses.replace(S.small_config(n=10, M=6, r=2, sigma=1.0, n_c=8, J=2, K_out=3, tol=1e-10),
                              inner="minres", local=local)
    inp = S.make_inputs(cfg)
    out = pipeline.run(cfg, inp, keep_steps=True)
    h = inp["psf"]; b = out["b"]; n = cfg.n
    wx, wy = ops.identity_weights(n)
    for k, st in enumerate(out["steps"]):
        assert np.all((st.status == mr.CONVERGED) | (st.status == mr.DEFL_DROPPED))
        for l in range(cfg.M):
            Ad = dense.assemble_shifted(h, wx, wy, inp["gamma"][l], n)
            xs = np.linalg.solve(Ad, b)
            kap = np.linalg.cond(Ad)
            assert np.linalg.norm(st.X[:, l] - xs) <= max(2 * kap * cfg.tol, 1e-12) * np.linalg.norm(xs)
        xstar = st.X[:, st.lstar].reshape(n, n)
        wx, wy = ops.irn_weights(xstar, cfg.tau)


def test_sequential_local_space_columns():
    """Alg. 3's second correction: orthogonal to [W, g-hat] and of unit norm; a
    duplicate of g-hat's direction is dropped (footnote P:691)."""
    from oracle import recycle as rc
    rng = np.random.Generator(np.random.PCG64(12))
    W, _ = np.linalg.qr(rng.standard_normal((200, 4)))
    g1 = rng.standard_normal(200)
    gh1 = rc.carried_direction(W, g1)
    B = np.column_stack([W, gh1])
    g2 = rng.standard_normal(200)
    gh2 = rc.carried_direction(B, g2)
    assert np.linalg.norm(B.T @ gh2) <= 1e-14 and abs(np.linalg.norm(gh2) - 1) <= 1e-14
    assert rc.carried_direction(B, 3.0 * g1 + 1e-6 * g2) is None


def test_principal_update_vnew_solves_eq_delta():
    """eq:delta: the first column of V^(new) approximates
    dx = x^(k-1,l_c) - x^(k,l_c), i.e. it solves (A + g E_k) dx = g (E_k - E_{k-1}) x^(k-1,l_c)
    (checked against a dense solve); the rest are orthonormal Krylov vectors whose span
    holds the rhs; the k >= 1 nested solve with principal="vnew" still matches dense
    solves at every (k, l)."""
    import dataclasses
    from oracle import pipeline
    cfg = dataclasses.replace(S.small_config(n=10, M=6, r=2, sigma=1.0, n_c=12, J=2, K_out=3, tol=1e-10),
                              principal="vnew")
    inp = S.make_inputs(cfg)
    out = pipeline.run(cfg, inp, keep_steps=True)
    h = inp["psf"]; b = out["b"]; n = cfg.n
    wx0, wy0 = ops.identity_weights(n)
    st0 = out["steps"][0]
    wx1, wy1 = ops.irn_weights(st0.X[:, st0.lstar].reshape(n, n), cfg.tau)
    st = pipeline.StepState(1, wx1, wy1, st0.X, st0.G, st0.V_i1, wx0, wy0)
    V, _ = pipeline.principal_update(cfg, h, b, inp["gamma"], st)
    lc = _ixof(cfg).l_c - 1
    g = inp["gamma"][lc]
    Ak = dense.assemble_shifted(h, wx1, wy1, g, n)
    E1 = dense.assemble_shifted(h, wx1, wy1, 1.0, n) - dense.assemble_shifted(h, wx1, wy1, 0.0, n)
    E0 = dense.assemble_shifted(h, wx0, wy0, 1.0, n) - dense.assemble_shifted(h, wx0, wy0, 0.0, n)
    q = g * (E1 - E0) @ st0.X[:, lc]
    K = V[:, 1:]
    assert np.allclose(np.linalg.norm(K, axis=0), 1.0)
    # the first column is the 100-step CG iterate on eq:delta from 0 (scipy's CG as the
    # independent reference), the first Krylov vector is the normalised rhs
    op = spla.LinearOperator(Ak.shape, matvec=lambda v: Ak @ v, dtype=np.float64)
    xs, _ = spla.cg(op, q, rtol=cfg.tol, atol=0.0, maxiter=100)
    assert np.linalg.norm(V[:, 0] - xs) <= 1e-6 * np.linalg.norm(xs)
    assert np.allclose(K[:, 0], q / np.linalg.norm(q), atol=1e-14)
    dx = np.linalg.solve(Ak, q)
    assert np.linalg.norm(V[:, 0] - dx) <= 1e-3 * np.linalg.norm(dx)
    wx, wy = wx0, wy0
    for k, sk in enumerate(out["steps"]):
        for l in range(cfg.M):
            Ad = dense.assemble_shifted(h, wx, wy, inp["gamma"][l], n)
            xs = np.linalg.solve(Ad, b)
            assert np.linalg.norm(sk.X[:, l] - xs) <= max(2 * np.linalg.cond(Ad) * cfg.tol, 1e-12) * np.linalg.norm(xs)
        wx, wy = ops.irn_weights(sk.X[:, sk.lstar].reshape(n, n), cfg.tau)
