"""Recycling MINRES for one shifted system -- the paper's own inner solver
(oracle, TEST INFRASTRUCTURE ONLY).

Follows §"Shift Specific Recycling" step by step, in its
notation:

 eq:corr_g  r = b - (A + gamma E) x_0 ; solve only for g = x - x_0
 eq:localU      (A + gamma E) U~_l = K_l R_l , K_l^T K_l = I , U_l = U~_l R_l^-1
 S_l  Range([U_l, V_m]), V_m a Lanczos basis of the Krylov space of
                         (I - K K^T)(A + gamma E) from
                         v_1 = (I - K K^T) r / ||(I - K K^T) r||
 Lanczos  (I - K K^T) A_g V_m = V_{m+1} T_m  (T_m (m+1) x m tridiagonal)
 eq:minShift  min_{y,z} || [K^T r ; xi e_1] - [[I, K^T A_g V_m],[0, T_m]] [z; y] ||
 eq:xFinal  g = V_m y + U_l z ,  x = x_0 + g

The stopping rule is the one of the deflated CG (reading G14): the least-squares
residual of eq:minShift (= ||b - A_g x|| in exact arithmetic) <= tol ||b||,
confirmed on the true residual b - A_g x; if the confirmation fails, the solve
restarts from x (x_0 <- x). The iteration count is the number of Lanczos
applies A_g v_j.

Literal and slow: K from numpy's Householder QR (diag(R) > 0, reading G16), the
basis V_m and the images A_g V_m stored, the LS residual min ||xi e_1 - T_m y||
solved by numpy.linalg.lstsq at every iteration, and the full block LS of
eq:minShift solved once at the end.  Pinned in tests/test_oracle_minres.py
(dense minimum-residual problems over explicit bases, scipy MINRES, K^T r = 0,
monotone residuals, tiny SPD systems vs dense solves).
"""
from __future__ import annotations

import dataclasses

import numpy as np

CONVERGED, MAXIT, BREAKDOWN, DEFL_DROPPED, ZERO_RHS = 0, 1, 2, 3, 4


@dataclasses.dataclass
class MinresResult:
    x: np.ndarray
    iters: int            # Lanczos applies A_g v_j
    applies: int          # all A_g applies (iters + residuals of x_0 + confirmations)
    relres_true: float
    status: int
    m_used: int           # columns of U~_l used
    res_hist: list = dataclasses.field(default_factory=list)   # LS residual per iteration
    ktr_max: float = 0.0  # ||K^T (b - A_g x)|| / ||b|| at exit (eq:xFinal makes it 0)


def local_factor(Z):
    """eq:localU: (A + gamma E) U~ = Z = K R with K^T K = I and diag(R) > 0."""
    K, R = np.linalg.qr(Z)
    sg = np.sign(np.diag(R))
    sg[sg == 0] = 1.0
    return K * sg, (R.T * sg).T


def recycled_minres(apply_gamma, b, x0=None, Ut=None, Z=None, tol=1e-8, maxit=20000,
                    n_carry=0) -> MinresResult:
    """Recycling MINRES on (A + gamma E) x = b from x0 over Range([U_l, V_m]).

    apply_gamma: flat vector -> (A + gamma E) times it.
    Ut: N x m local recycle matrix U~_l (columns W_g and the carried g-hat), or None.
    Z:  N x m, (A + gamma E) U~_l (reused, no applies).
    n_carry: trailing carried columns of U~, dropped first if Z is rank deficient
    (R_l singular), then all of U~ (DEFL_DROPPED) -- the same fallback as O4.
    """
    N = b.shape[0]
    nb = float(np.linalg.norm(b))
    if nb == 0.0:
        return MinresResult(np.zeros(N), 0, 0, 0.0, ZERO_RHS, 0)
    x = np.zeros(N) if x0 is None else np.array(x0, dtype=np.float64)
    status_setup = CONVERGED
    K = R = None
    if Ut is not None and Ut.shape[1] > 0:
        m = Ut.shape[1]
        while m > 0:
            Kc, Rc = local_factor(Z[:, :m])
            d = np.abs(np.diag(Rc))
            if d.min() > 1e-14 * d.max():
                K, R, Ut = Kc, Rc, Ut[:, :m]
                break
            status_setup = DEFL_DROPPED
            m = m - n_carry if (n_carry > 0 and m == Ut.shape[1]) else 0
    m_used = 0 if K is None else K.shape[1]

    def proj(v):                      # (I - K K^T) v
        return v if K is None else v - K @ (K.T @ v)

    applies = 0
    iters = 0
    it_restart = -1
    hist = []
    if x0 is None:
        r = b.copy()
    else:
        r = b - apply_gamma(x)
        applies += 1
    while True:
        # ---- v_1 = (I - K K^T) r / xi
        rh = proj(r)
        xi = float(np.linalg.norm(rh))
        V = [rh / xi] if xi > 0 else []
        AV = []
        alphas, betas = [], []       # T_m: diag alpha_j, sub-diagonal beta_{j+1}
        status = MAXIT
        y = np.zeros(0)
        # an initial residual already small enough needs no update beyond the
        # z-block (m = 0 in eq:minShift, whose least-squares residual is xi)
        while xi > tol * nb and iters < maxit:
            j = len(V) - 1
            w = apply_gamma(V[j])
            iters += 1
            applies += 1
            AV.append(w)
            p = proj(w)                                   # (I - K K^T) A_g v_j
            a = float(V[j] @ p)
            p = p - a * V[j] - (betas[-1] * V[j - 1] if j > 0 else 0.0)
            bn = float(np.linalg.norm(p))
            alphas.append(a)
            betas.append(bn)
            mm = len(alphas)
            T = np.zeros((mm + 1, mm))
            for i in range(mm):
                T[i, i] = alphas[i]
                T[i + 1, i] = betas[i]
                if i + 1 < mm:
                    T[i, i + 1] = betas[i]
            e1 = np.zeros(mm + 1)
            e1[0] = xi
            y = np.linalg.lstsq(T, e1, rcond=None)[0]
            res = float(np.linalg.norm(e1 - T @ y))
            hist.append(res)
            if res <= tol * nb or bn == 0.0:
                status = CONVERGED
                break
            V.append(p / bn)
        # ---- eq:minShift (full block least squares) and eq:xFinal
        mm = len(AV)
        if mm > 0:
            Vm = np.stack(V[:mm], 1)
            AVm = np.stack(AV, 1)
            T = np.zeros((mm + 1, mm))
            for i in range(mm):
                T[i, i] = alphas[i]
                T[i + 1, i] = betas[i]
                if i + 1 < mm:
                    T[i, i + 1] = betas[i]
            k = m_used
            Mb = np.zeros((k + mm + 1, k + mm))
            rhs = np.zeros(k + mm + 1)
            if k:
                Mb[:k, :k] = np.eye(k)
                Mb[:k, k:] = K.T @ AVm
                rhs[:k] = K.T @ r
            Mb[k:, k:] = T
            rhs[k] = xi
            sol = np.linalg.lstsq(Mb, rhs, rcond=None)[0]
            z, y = sol[:k], sol[k:]
            g = Vm @ y
            if k:
                g = g + Ut @ np.linalg.solve(R, z)      # U_l z = U~_l R_l^-1 z
            x = x + g
        elif m_used:
            x = x + Ut @ np.linalg.solve(R, K.T @ r)    # m = 0: g = U_l K^T r
        # ---- confirm on the true residual
        r = b - apply_gamma(x)
        applies += 1
        rt = float(np.linalg.norm(r))
        if rt <= tol * nb:
            status = CONVERGED
            break
        if iters >= maxit or iters == it_restart:
            status = MAXIT            # maxit, or a restart that made no Lanczos step (G37)
            break
        it_restart = iters
    if status == CONVERGED and status_setup == DEFL_DROPPED:
        status = DEFL_DROPPED
    ktr = 0.0 if K is None else float(np.linalg.norm(K.T @ r)) / nb
    return MinresResult(x, iters, applies, rt / nb, status, m_used, hist, ktr)
