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

Plain and slow: K from numpy's Householder QR (diag(R) > 0, reading G16), the
basis V_m and the images A_g V_m stored; the y-block min ||xi e_1 - T_m y|| by the
textbook Givens QR of T_m (Paige-Saunders), its residual |phibar| checked after every
step; at the end y from the triangular factor and the first block row of eq:minShift
solved exactly (z = K^T r - K^T A_g V_m y).  Pinned in tests/test_oracle_minres.py
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
    store: list = dataclasses.field(default_factory=list)    # normalised Lanczos vectors


def local_factor(Z):
    """eq:localU: (A + gamma E) U~ = Z = K R with K^T K = I and diag(R) > 0."""
    K, R = np.linalg.qr(Z)
    sg = np.sign(np.diag(R))
    sg[sg == 0] = 1.0
    return K * sg, (R.T * sg).T


def recycled_minres(apply_gamma, b, x0=None, Ut=None, Z=None, tol=1e-8, maxit=20000,
                    n_carry=0, store_cap=0) -> MinresResult:
    """Recycling MINRES on (A + gamma E) x = b from x0 over Range([U_l, V_m]).

    apply_gamma: flat vector -> (A + gamma E) times it.
    Ut: N x m local recycle matrix U~_l (columns W_g and the carried g-hat), or None.
    Z:  N x m, (A + gamma E) U~_l (reused, no applies).
    n_carry: trailing carried columns of U~, dropped first if Z is rank deficient
    (R_l singular), then all of U~ (DEFL_DROPPED) -- the same fallback as O4.
    store_cap > 0 keeps the first Lanczos vectors v_1, v_2, ... of the solve (the seed
    solves' Krylov basis, S1; the span of CG's normalised residuals).
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
    store = []
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
        betas = []                   # beta_{j+1} (sub-diagonal of T_m)
        # QR of T_m by Givens rotations (Paige-Saunders): R_m has three diagonals
        # (rd = diagonal, r1 = first, r2 = second super-diagonal), Q_m^T (xi e_1) = (t, phibar)
        rd, r1, r2, tvec = [], [], [], []
        cs_prev, sn_prev = 1.0, 0.0      # rotation j-1
        cs_pp, sn_pp = 1.0, 0.0          # rotation j-2
        phibar = xi
        status = MAXIT
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
            bprev = betas[-1] if j > 0 else 0.0
            p = p - a * V[j] - (bprev * V[j - 1] if j > 0 else 0.0)
            bn = float(np.linalg.norm(p))
            betas.append(bn)
            # new column of T_m: (.., bprev, a, bn) in rows j-1, j, j+1
            e2 = sn_pp * bprev                     # row j-2 after rotation j-2
            tmp = cs_pp * bprev
            e1 = cs_prev * tmp + sn_prev * a       # row j-1 after rotation j-1
            dj = -sn_prev * tmp + cs_prev * a      # row j before the new rotation
            gm = float(np.hypot(dj, bn))
            c_new, s_new = (dj / gm, bn / gm) if gm > 0 else (1.0, 0.0)
            rd.append(gm); r1.append(e1); r2.append(e2)
            tvec.append(c_new * phibar)
            phibar = -s_new * phibar
            cs_pp, sn_pp, cs_prev, sn_prev = cs_prev, sn_prev, c_new, s_new
            res = abs(phibar)
            hist.append(res)
            if res <= tol * nb or bn == 0.0:
                status = CONVERGED
                break
            V.append(p / bn)
        store.extend(V[:max(0, store_cap - len(store))][:max(len(AV), 0)])
        # ---- eq:minShift: y from R_m y = t (back substitution), the first block row solved
        # exactly, z = K^T r - K^T A_g V_m y; eq:xFinal
        mm = len(AV)
        if mm > 0:
            y = np.zeros(mm)
            for i in range(mm - 1, -1, -1):
                v = tvec[i]
                if i + 1 < mm:
                    v -= r1[i + 1] * y[i + 1]
                if i + 2 < mm:
                    v -= r2[i + 2] * y[i + 2]
                y[i] = v / rd[i]
            Vm = np.stack(V[:mm], 1)
            g = Vm @ y
            if m_used:
                AVm = np.stack(AV, 1)
                z = K.T @ r - K.T @ (AVm @ y)
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
    return MinresResult(x, iters, applies, rt / nb, status, m_used, hist, ktr, store)
