"""O6: L-curve and the outer IRN loop (Alg. 5) -- oracle, test-only.

One outer step k (reading D3: all shifts of a step are independent):
  1. k = 0: seed solves at gamma_i1, gamma_i2 (plain CG, residual store) and
     Ritz spaces V_i1, V_i2;  U~ = [x^(0,i1), x^(0,i2), V_i1, V_i2]
     k >= 1: U~ = [V_i1, x^(k-1,1), ..., x^(k-1,M)]      (eq:tildeUupdate, G10)
  2. U~ <- stabilize(U~, cap n_c)                         (Alg. 1)
  3. anchor at gamma_* = gamma_{i*}                       (eq:establishU)
  4. x_0^(k,l) = U q_l from eq:orthupdate
     [f2(iii): oblique eq:obliqueupdate P:877-882 / two anchors eq:updates P:1000-1005]
  5. groups L = {l <= I}, R = {l > I}; W from gamma_{J_L}, gamma_{J_R} (Alg. 4)
  6. per shift: U_l = [W_g(l), g-hat^(k-1,l)] and deflated CG (O4)
  7. L-curve corner l* (P:138-140), x* = x^(k,l*)
  8. W_{k+1} = IRN weights of x* (north_star; reading G2), or the f1 rules:
     isotropic IRN / Gazzola's D_{k+1} = diag(1 - w.^p) D_k
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import defcg as dcg
from . import indices as _ix
from . import minres as mr
from . import operators as ops
from . import recycle as rc


def lcurve_corner(rho: np.ndarray, eta: np.ndarray) -> tuple[int, np.ndarray]:
    """Corner of the discrete L-curve (log rho_l, log eta_l): maximum curvature
     with centred differences on the uniform t = log10 lambda
    grid, endpoints excluded, ties to the smallest index (reading G25).
    kappa = (rho' eta'' - rho'' eta') / (rho'^2 + eta'^2)^(3/2). Returns 0-based l*."""
    M = len(rho)
    lr = np.log(np.asarray(rho, dtype=np.float64))
    le = np.log(np.asarray(eta, dtype=np.float64))
    kappa = np.full(M, -np.inf)
    for l in range(1, M - 1):
        r1 = (lr[l + 1] - lr[l - 1]) / 2.0
        e1 = (le[l + 1] - le[l - 1]) / 2.0
        r2 = lr[l + 1] - 2.0 * lr[l] + lr[l - 1]
        e2 = le[l + 1] - 2.0 * le[l] + le[l - 1]
        den = (r1 * r1 + e1 * e1) ** 1.5
        kappa[l] = (r1 * e2 - r2 * e1) / den if den > 0 else -np.inf
    if M < 3:
        return 0, kappa
    best = 1 + int(np.argmax(kappa[1:M - 1]))   # np.argmax: first maximum -> smallest l
    return best, kappa


@dataclasses.dataclass
class StepState:
    """Everything outer step k needs from step k-1 (the stepwise parity handoff, G28)."""
    k: int
    wx: np.ndarray
    wy: np.ndarray
    X_prev: np.ndarray | None      # N x M solutions of step k-1
    G_prev: np.ndarray | None      # N x M corrections g^(k-1,l)
    V_i1: np.ndarray | None        # Ritz block kept from k = 0
    wx_prev: np.ndarray | None = None   # W_{k-1} (only for cfg.principal == "vnew", eq:delta)
    wy_prev: np.ndarray | None = None


@dataclasses.dataclass
class StepResult:
    X: np.ndarray
    G: np.ndarray
    Xp: np.ndarray
    iters: np.ndarray
    applies: np.ndarray
    status: np.ndarray
    relres: np.ndarray
    guess_relres: np.ndarray
    nc: int
    lstar: int
    rho: np.ndarray
    eta: np.ndarray
    overhead_applies: int          # seeds + Ritz + anchoring + g-hat images
    V_i1: np.ndarray | None
    Ut: np.ndarray | None = None
    anchor: rc.Anchor | None = None


_SHIFT_SOLVE = None


def _run_shift(l):
    """Pool trampoline (fork start method: the closure is inherited, never pickled). One
    BLAS thread per worker process: the workers are the parallelism."""
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:   # pragma: no cover
        return _SHIFT_SOLVE(l)
    with threadpool_limits(1):
        return _SHIFT_SOLVE(l)


def outer_step(cfg, h, b, d, gamma, st: StepState, shifts=None, workers: int = 1) -> StepResult:
    """One outer step (Alg. 5 body) under the readings listed above.
    `shifts` optionally restricts the CG solves to a subset of 0-based indices
    (the others are left at zero) -- used for bounded-cost samples.
    `workers` > 1 runs the per-shift solves (independent under reading D3) in that many
    forked processes -- the only parallelism of the oracle (across shifts)."""
    n, M, N = cfg.n, cfg.M, cfg.N
    wx, wy = st.wx, st.wy
    ix = _ix.of(cfg)

    def A_g(g):
        return lambda v: ops.apply_shifted(h, wx, wy, g, v.reshape(n, n)).ravel()

    overhead = 0
    i1, i2 = ix.i1 - 1, ix.i2 - 1
    V_i1 = st.V_i1
    if st.k == 0:
        n1 = math.ceil(2 * (cfg.n_c - 2) / 3)
        n2 = cfg.n_c - 2 - n1
        s1 = _seed_solver(cfg)(A_g(gamma[i1]), b, tol=cfg.tol, maxit=cfg.maxit, store_cap=100)
        s2 = _seed_solver(cfg)(A_g(gamma[i2]), b, tol=cfg.tol, maxit=cfg.maxit, store_cap=100)
        V_i1, _, a1 = rc.ritz_space(A_g(gamma[i1]), s1.store, n1)
        V_i2, _, a2 = rc.ritz_space(A_g(gamma[i2]), s2.store, n2)
        overhead += s1.applies + s2.applies + a1 + a2
        raw = np.column_stack([s1.x, s2.x, V_i1, V_i2])
    elif getattr(cfg, "principal", "g10") == "vnew" and st.wx_prev is not None:
        V_new, a_new = principal_update(cfg, h, b, gamma, st)
        overhead += a_new
        raw = np.column_stack([V_i1, V_new, st.X_prev])
    else:
        raw = np.column_stack([V_i1, st.X_prev])
    Ut = rc.stabilize(raw, cfg.n_c)
    gstar = gamma[ix.istar - 1]
    an = rc.anchor(h, wx, wy, Ut, b, gstar, n)
    overhead += Ut.shape[1]
    mode = getattr(cfg, "guess", "orth")
    if mode == "orth":
        def guess(l):
            return rc.principal_guess(an, gamma[l])
    elif mode == "oblique":
        def guess(l):
            return rc.oblique_guess(an, gamma[l])
    elif mode == "oblique2":
        # eq:updates: anchors gamma_{I_L} (left group) and gamma_{I_R} (right group); the
        # images Z_A, Z_E are shared (no extra applies), only K, R differ (reading G34)
        anL = an if ix.I_L == ix.istar else rc.anchor(h, wx, wy, Ut, b, gamma[ix.I_L - 1], n)
        anR = rc.anchor(h, wx, wy, Ut, b, gamma[ix.I_R - 1], n)

        def guess(l):
            return rc.oblique_guess(anL if (l + 1) <= ix.I else anR, gamma[l])
    else:
        raise ValueError(f"unknown guess mode {mode!r}")

    groups = {}
    for gname, jidx in (("L", ix.J_L - 1), ("R", ix.J_R - 1)):
        W, AW, EW, _, _ = rc.group_ritz(an, gamma[jidx], cfg.J)
        groups[gname] = (W, AW, EW)

    X = np.zeros((N, M)); G = np.zeros((N, M)); Xp = np.zeros((N, M))
    iters = np.zeros(M, dtype=np.int64); applies = np.zeros(M, dtype=np.int64)
    status = np.zeros(M, dtype=np.int64); relres = np.zeros(M); grel = np.zeros(M)
    nb = np.linalg.norm(b)
    todo = list(range(M)) if shifts is None else list(shifts)
    seq = getattr(cfg, "local", "d3") == "seq"

    def solve(l):
        """Shift l: principal guess, local space [W_g, g-hat (, g^(k,l-1))], inner solve.
        Returns (x, x_p, iters, applies, status, relres_true, guess relres, overhead)."""
        W, AW, EW = groups["L" if (l + 1) <= ix.I else "R"]
        xp = guess(l)
        cols_U = [W]
        cols_Z = [AW + gamma[l] * EW]
        n_carry = 0
        ov = 0
        if st.k >= 1 and st.G_prev is not None:
            gh = rc.carried_direction(W, st.G_prev[:, l])
            if gh is not None:
                img = gh.reshape(n, n)
                zg = (ops.apply_A(h, img) + gamma[l] * ops.apply_E(wx, wy, img)).ravel()
                ov += 1
                cols_U.append(gh[:, None]); cols_Z.append(zg[:, None]); n_carry = 1
        if seq and l >= 1 and _same_group(cfg, l - 1, l) and (l - 1) in todo:
            # Alg. 3 / Alg. 4: U~_l = [W, g^(k-1,l), g^(k,l-1)], the second
            # correction orthogonalised against [W, g-hat] and dropped when nearly
            # redundant (footnote P:691; reading G35)
            gh2 = rc.carried_direction(np.column_stack(cols_U), G[:, l - 1])
            if gh2 is not None:
                img = gh2.reshape(n, n)
                zg = (ops.apply_A(h, img) + gamma[l] * ops.apply_E(wx, wy, img)).ravel()
                ov += 1
                cols_U.append(gh2[:, None]); cols_Z.append(zg[:, None]); n_carry += 1
        U = np.column_stack(cols_U); Z = np.column_stack(cols_Z)
        if getattr(cfg, "inner", "cg") == "minres":    # the paper's inner solver (f2(ii))
            res = mr.recycled_minres(A_g(gamma[l]), b, x0=xp, Ut=U, Z=Z, tol=cfg.tol,
                                     maxit=cfg.maxit, n_carry=n_carry)
        else:
            res = dcg.defcg(A_g(gamma[l]), b, x_p=xp, U=U, Z=Z, tol=cfg.tol,
                            maxit=cfg.maxit, n_carry=n_carry)
        xpv = np.zeros(N) if xp is None else xp
        gr = (np.linalg.norm(b - A_g(gamma[l])(xpv)) / nb) if xp is not None else 1.0
        return res.x, xpv, res.iters, res.applies, res.status, res.relres_true, gr, ov

    def store(l, r):
        nonlocal overhead
        X[:, l], Xp[:, l] = r[0], r[1]
        G[:, l] = r[0] - r[1]
        iters[l], applies[l], status[l], relres[l], grel[l] = r[2], r[3], r[4], r[5], r[6]
        overhead += r[7]

    if workers > 1 and not seq and len(todo) > 1:
        import multiprocessing as mp
        global _SHIFT_SOLVE
        _SHIFT_SOLVE = solve
        try:
            with mp.get_context("fork").Pool(min(workers, len(todo))) as pool:
                for l, r in zip(todo, pool.map(_run_shift, todo, chunksize=1)):
                    store(l, r)
        finally:
            _SHIFT_SOLVE = None
    else:
        for l in todo:
            store(l, solve(l))

    rho = np.zeros(M); eta = np.zeros(M)
    for l in range(M):
        img = X[:, l].reshape(n, n)
        rho[l] = np.linalg.norm(ops.conv(h, img) - d)
        eta[l] = math.sqrt(ops.seminorm2(wx, wy, img))
    lstar = lcurve_corner(rho, eta)[0] if shifts is None else -1
    return StepResult(X, G, Xp, iters, applies, status, relres, grel, Ut.shape[1], lstar,
                      rho, eta, overhead, V_i1, Ut, an)


def principal_update(cfg, h, b, gamma, st):
    """eq:delta (reading G36): for l_c = round(0.9 M) solve
    (A + gamma_c E_k) dx = gamma_c (E_k - E_{k-1}) x^(k-1,l_c) (eq:delta times gamma_c)
    by at most 100 CG steps from 0, storing the normalised residuals (the Krylov vectors,
    the same span as MINRES's Lanczos vectors); V^(new) = [dx, stored residuals]
    (<= 101 columns). Returns (V_new, applies: the two E images + CG)."""
    n = cfg.n
    lc = _ix.of(cfg).l_c - 1
    gc = gamma[lc]
    x = st.X_prev[:, lc].reshape(n, n)
    q = gc * (ops.apply_E(st.wx, st.wy, x) - ops.apply_E(st.wx_prev, st.wy_prev, x)).ravel()
    A = lambda v: ops.apply_shifted(h, st.wx, st.wy, gc, v.reshape(n, n)).ravel()
    res = _seed_solver(cfg)(A, q, tol=cfg.tol, maxit=100, store_cap=100)
    cols = [res.x] + list(res.store)
    return np.column_stack(cols), res.applies + 2


def _seed_solver(cfg):
    """Plain solves with a Krylov store (seeds S1, eq:delta): the configured inner solver
    (CG residuals or MINRES Lanczos vectors: the same Krylov space)."""
    if getattr(cfg, "inner", "cg") == "minres":
        return mr.recycled_minres
    return dcg.defcg


def operator_of(cfg, inputs):
    """C of the configuration: the PSF array (blur, O1) or the explicit CT matrix (f4)."""
    if getattr(cfg, "operator", "blur") == "ct":
        from .ct import CTOperator
        return CTOperator(cfg.n, inputs["angles"], cfg.ndet)
    return inputs["psf"]


def _same_group(cfg, a, b):
    """Shifts a, b (0-based) in the same group (left: l <= I, right: l > I; Alg. 4)."""
    return ((a + 1) <= _ix.of(cfg).I) == ((b + 1) <= _ix.of(cfg).I)


def next_weights(cfg, st_w, xstar):
    """W_{k+1} from x* by cfg.weight_rule: "irn" (north_star, reading G2), "irn_iso"
    (isotropic IRN) or "gazzola" (st_w carries D_k). Returns
    ((wx, wy), D_{k+1} or None)."""
    rule = getattr(cfg, "weight_rule", "irn")
    if rule == "irn":
        return ops.irn_weights(xstar, cfg.tau), None
    if rule == "irn_iso":
        return ops.irn_weights_iso(xstar, cfg.tau), None
    if rule == "gazzola":
        D, W = ops.gazzola_step(st_w[0], st_w[1], xstar, getattr(cfg, "p", 2.0))
        return W, D
    raise ValueError(f"unknown weight rule {rule!r}")


def run(cfg, inputs, K_out=None, keep_steps=False):
    """The outer loop: up to K_out outer steps (configs fix the count, reading of A28);
    cfg.stop == "lstar3" also stops once l* is the same for 3 consecutive steps."""
    n = cfg.n
    h = operator_of(cfg, inputs)
    d, b2 = ops.make_data(h, inputs["x_true"], inputs["xi"], cfg.noise)
    b = b2.ravel(); dd = d
    gamma = inputs["gamma"]
    wx, wy = ops.identity_weights(n)
    D = ops.identity_weights(n)            # D_0 = I (Gazzola's rule only)
    st = StepState(0, wx, wy, None, None, None)
    steps = []
    hist = []
    for k in range(K_out or cfg.K_out):
        st.k = k
        res = outer_step(cfg, h, b, dd, gamma, st)
        steps.append(res if keep_steps else dataclasses.replace(res, Ut=None, anchor=None))
        hist.append(res.lstar)
        xstar = res.X[:, res.lstar].reshape(n, n)
        (wx, wy), D = next_weights(cfg, D, xstar)
        st = StepState(k + 1, wx, wy, res.X, res.G, res.V_i1, st.wx, st.wy)
        if getattr(cfg, "stop", "fixed") == "lstar3" and ops.lstar_settled(hist):
            break
    return {"b": b, "d": dd, "steps": steps, "final_weights": (wx, wy), "lstar": hist}
