"""O4: deflated (recycled) CG for one shifted system (oracle, test-only).

The paper's inner solver is recycling MINRES over Range([U_l, V_m]) with the
projector (I - K_l K_l^T) (eq:minShift P:511-526, eq:xFinal P:528-534).
north_star fixes "preconditioner-free recycled CG"; A + gamma E is SPD
(P:298-305), so the build uses the Galerkin (energy-norm) analogue on
the same augmented space x_0 + Range(U_l) + K_m: deflated CG
(reading G1 / D1 in DESIGN.md). Steps, in order:

 setup   Z = A_gamma U, G = sym(U^T Z), Cholesky; on failure drop the carried
         correction column, then all of U (DEFL_DROPPED)
 start   r_p = b - A_gamma x_p (eq:corr_g P:462-468; one fresh apply, G15)
         c = G^-1 U^T r_p ; x_0 = x_p + U c ; r_0 = r_p - Z c
         mu_0 = G^-1 Z^T r_0 ; p_0 = r_0 - U mu_0
 loop    w = A_gamma p ; pi = p.w ; alpha = rho/pi ; x += alpha p ; r -= alpha w
         rho' = r.r ; stop if sqrt(rho') <= tol ||b||
         beta = rho'/rho ; mu = G^-1 Z^T r ; p = r + beta p - U mu
 confirm true residual r_t = b - A_gamma x (stopping rule P:164-170, §8.1
         P:1021 on the true residual, reading G14); if it fails, restart from r_t.
The iteration count is the number of w = A_gamma p applies in the loop.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import dense

CONVERGED, MAXIT, BREAKDOWN, DEFL_DROPPED, ZERO_RHS = 0, 1, 2, 3, 4


@dataclasses.dataclass
class CGResult:
    x: np.ndarray
    iters: int
    applies: int          # A_gamma applies (each = 1 A + 1 E matvec)
    relres_true: float
    status: int
    m_used: int           # recycle columns actually used
    store: list = dataclasses.field(default_factory=list)
    utr_max: float = 0.0  # max_j ||U^T r_j|| / ||b|| (invariant check, reading G29)
    rho_hist: list = dataclasses.field(default_factory=list)


def defcg(apply_gamma, b, x_p=None, U=None, Z=None, tol=1e-8, maxit=20000,
          store_cap=0, n_carry=0) -> CGResult:
    """Deflated CG on A_gamma x = b. apply_gamma maps a flat vector to A_gamma times it.

    U, Z: N x m arrays (Z = A_gamma U), or None for plain CG (U = empty).
    store_cap > 0 stores the first residuals, normalised (seed solves, S1).
    n_carry: number of trailing columns of U that are carried corrections (g-hat);
    they are dropped first when G is not SPD, then all of U.
    """
    N = b.shape[0]
    nb = float(np.linalg.norm(b))
    applies = 0
    if nb == 0.0:
        return CGResult(np.zeros(N), 0, 0, 0.0, ZERO_RHS, 0)

    # ---- setup: G = sym(U^T Z) and its Cholesky factor
    status_setup = CONVERGED
    Lg = None
    if U is not None and U.shape[1] > 0:
        m = U.shape[1]
        while m > 0:
            G = dense.sym(U[:, :m].T @ Z[:, :m])
            Lg = dense.cholesky_or_none(G)
            if Lg is not None:
                break
            status_setup = DEFL_DROPPED
            m = m - n_carry if (n_carry > 0 and m == U.shape[1]) else 0
        if m > 0:
            U, Z = U[:, :m], Z[:, :m]
        else:
            U = Z = None
    m_used = 0 if U is None else U.shape[1]

    def gsolve(z):
        return dense.chol_solve(Lg, z)

    # ---- start
    if x_p is None:
        x = np.zeros(N)
        r = b.copy()
    else:
        x = x_p.copy()
        r = b - apply_gamma(x)
        applies += 1
    if U is not None:
        c = gsolve(U.T @ r)
        x = x + U @ c
        r = r - Z @ c
    res = CGResult(x, 0, applies, 0.0, CONVERGED, m_used)

    def track(rv):
        if U is not None:
            res.utr_max = max(res.utr_max, float(np.linalg.norm(U.T @ rv)) / nb)

    rho = float(r @ r)
    res.rho_hist.append(rho)
    track(r)
    iters = 0
    nrt = None
    while True:
        converged = np.sqrt(rho) <= tol * nb
        if not converged:
            if store_cap > 0 and len(res.store) < store_cap:
                res.store.append(r / np.sqrt(rho))
            p = r - U @ gsolve(Z.T @ r) if U is not None else r.copy()
            while iters < maxit:
                w = apply_gamma(p)
                applies += 1
                iters += 1
                pi = float(p @ w)
                if not (pi > 0.0) or not np.isfinite(pi):
                    res.status = BREAKDOWN
                    break
                alpha = rho / pi
                x = x + alpha * p
                r = r - alpha * w
                rho_new = float(r @ r)
                res.rho_hist.append(rho_new)
                track(r)
                if np.sqrt(rho_new) <= tol * nb:
                    rho = rho_new
                    converged = True
                    break
                if store_cap > 0 and len(res.store) < store_cap:
                    res.store.append(r / np.sqrt(rho_new))
                beta = rho_new / rho
                rho = rho_new
                if U is not None:
                    p = r + beta * p - U @ gsolve(Z.T @ r)
                else:
                    p = r + beta * p
            if res.status == BREAKDOWN:
                break
            if not converged:
                res.status = MAXIT
                break
        # ---- confirm on the true residual
        rt = b - apply_gamma(x)
        applies += 1
        nrt = float(np.linalg.norm(rt))
        if nrt <= tol * nb:
            res.status = CONVERGED
            break
        if iters >= maxit:
            res.status = MAXIT
            break
        r = rt
        rho = float(r @ r)
    res.x = x
    res.iters = iters
    res.applies = applies
    if nrt is None or res.status != CONVERGED:
        nrt = float(np.linalg.norm(b - apply_gamma(x)))
    res.relres_true = nrt / nb
    if res.status == CONVERGED and status_setup == DEFL_DROPPED:
        res.status = DEFL_DROPPED
    return res
