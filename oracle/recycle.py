"""O5: recycle-space machinery for one outer step k (oracle, test-only).

PAPER.md passages followed, in the order Alg. 5 uses them:
  seed solves + Ritz spaces V_i1, V_i2      §5.1
  U~ = [x^(0,i1), x^(0,i2), V_i1, V_i2]     eq:widetildeU P:575
  U~ = [V_i1, x^(k-1,1..M)]  (k >= 1)       eq:tildeUupdate P:654 (no V^(new), reading G10)
  stabilize (Alg. 1)
  anchor (A + gamma_* E) U = K, K^T K = I   eq:establishU P:386-391, implicit R^-1 P:851-853
  initial guess per shift                   eq:orthupdate P:410-430
    (or oblique: eq:obliqueupdate P:877-882, two anchors eq:updates P:1000-1005)
  projected pencil A^, E^                   eq:hq P:677
  group Ritz block W (Alg. 2, Alg. 4)       P:681-687, groups §5.4
  local space [W, g^(k-1,l)]                Alg. 3 P:700-704 without g^(k,l-1) (reading D3),
                                            near-duplicate test footnote P:691 (reading G12)
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import dense
from . import operators as ops

COND_CAP = 1e10          # Alg. 1: sigma_1 / sigma_i < 1e10
DUP_SIN = math.sqrt(1.0 - 0.999 ** 2)   # reading G12: cos > 0.999 is "nearly redundant"


def stabilize(raw: np.ndarray, cap: int | None = None, condcap: float = COND_CAP) -> np.ndarray:
    """Alg. 1: thin SVD raw = Q S W^T, keep the leading columns with
    sigma_1/sigma_i < condcap (strict), then at most `cap` of them (reading G6).
    Columns are first scaled to unit 2-norm (the paper is silent on scaling, G6);
    zero columns are discarded."""
    norms = np.linalg.norm(raw, axis=0)
    keep = norms > 0
    X = raw[:, keep] / norms[keep][None, :]
    if X.shape[1] == 0:
        return np.zeros((raw.shape[0], 0))
    Q, s, _ = np.linalg.svd(X, full_matrices=False)
    nk = int(np.sum(s[0] / s < condcap))
    if cap is not None:
        nk = min(nk, cap)
    return Q[:, :nk].copy()


def ritz_space(apply_gamma, store: list, n_keep: int):
    """Rayleigh-Ritz on the stored (normalised) residuals of a seed solve:
    Q = stabilize(store), H = Q^T A_gamma Q (one apply per column),
    ascending eig, keep the n_keep smallest Ritz vectors (reading G9).
    Returns (V, theta, applies)."""
    if n_keep <= 0 or len(store) == 0:
        return np.zeros((store[0].shape[0] if store else 0, 0)), np.zeros(0), 0
    Q = stabilize(np.stack(store, axis=1))
    AQ = np.stack([apply_gamma(Q[:, j]) for j in range(Q.shape[1])], axis=1)
    H = dense.sym(Q.T @ AQ)
    theta, Zr = np.linalg.eigh(H)
    k = min(n_keep, Q.shape[1])
    return Q @ Zr[:, :k], theta[:k], Q.shape[1]


@dataclasses.dataclass
class Anchor:
    Ut: np.ndarray     # U~ (N x nc), orthonormal
    ZA: np.ndarray     # A U~
    ZE: np.ndarray     # E_k U~
    K: np.ndarray      # (A + gamma_* E) U~ = K R
    R: np.ndarray
    P: np.ndarray      # K^T E U          = K^T Z_E R^-1
    Q2: np.ndarray     # (E U)^T (E U)    = R^-T Z_E^T Z_E R^-1
    u: np.ndarray      # U^T E b          = R^-T Z_E^T b
    v: np.ndarray      # K^T b
    Ahat: np.ndarray   # U~^T A U~        (eq:hq)
    Ehat: np.ndarray   # U~^T E U~
    gamma_star: float


def anchor(h, wx, wy, Ut: np.ndarray, b: np.ndarray, gamma_star: float, n: int) -> Anchor:
    """eq:establishU and the n_c x n_c quantities of eq:orthupdate,
    formed from E U~ without forming U = U~ R^-1. n_c apply pairs."""
    nc = Ut.shape[1]
    ZA = np.zeros_like(Ut)
    ZE = np.zeros_like(Ut)
    for j in range(nc):
        img = Ut[:, j].reshape(n, n)
        ZA[:, j] = ops.apply_A(h, img).ravel()
        ZE[:, j] = ops.apply_E(wx, wy, img).ravel()
    K, R = dense.qr_pos(ZA + gamma_star * ZE)
    P = dense.tri_inv_t_apply(R, (K.T @ ZE).T).T          # K^T Z_E R^-1
    Q2 = dense.tri_inv_t_apply(R, dense.tri_inv_t_apply(R, ZE.T @ ZE).T)  # R^-T (.) R^-1
    Q2 = dense.sym(Q2)
    u = dense.tri_inv_t_apply(R, ZE.T @ b)
    v = K.T @ b
    Ahat = dense.sym(Ut.T @ ZA)
    Ehat = dense.sym(Ut.T @ ZE)
    return Anchor(Ut, ZA, ZE, K, R, P, Q2, u, v, Ahat, Ehat, gamma_star)


def guess_coeffs(an: Anchor, gamma: float):
    """eq:orthupdate for delta = gamma - gamma_*:
    (I + delta (K^T E U) + delta (K^T E U)^T + delta^2 U^T E^2 U) q = K^T b + delta U^T E b,
    solved by Cholesky; returns c = R^-1 q (so x_0 = U~ c), or None when
    the Cholesky factorisation fails (x_0 = 0, status NOT_SPD)."""
    nc = an.P.shape[0]
    d = gamma - an.gamma_star
    G = np.eye(nc) + d * (an.P + an.P.T) + d * d * an.Q2
    L = dense.cholesky_or_none(G)
    if L is None:
        return None
    q = dense.chol_solve(L, an.v + d * an.u)
    return dense.tri_inv_apply(an.R, q)


def oblique_coeffs(an: Anchor, gamma: float):
    """eq:obliqueupdate: x_0 = U q with the oblique condition K^T r_0 = 0,
    r_0 = b - (A + gamma E) U q = b - K q - delta E U q (since (A + gamma_a E) U = K):
        (I + delta K^T E U) q = K^T b,   delta = gamma - gamma_a,
    with K^T E U = K^T Z_E R^-1 = an.P. Solved by LU (numpy); returns c = R^-1 q, or
    None when the system is singular (x_0 = 0)."""
    nc = an.P.shape[0]
    d = gamma - an.gamma_star
    try:
        q = np.linalg.solve(np.eye(nc) + d * an.P, an.v)
    except np.linalg.LinAlgError:
        return None
    if not np.all(np.isfinite(q)):
        return None
    return dense.tri_inv_apply(an.R, q)


def oblique_guess(an: Anchor, gamma: float):
    c = oblique_coeffs(an, gamma)
    return None if c is None else an.Ut @ c


def principal_guess(an: Anchor, gamma: float):
    c = guess_coeffs(an, gamma)
    return None if c is None else an.Ut @ c


def group_ritz(an: Anchor, gamma_J: float, J: int):
    """Alg. 2: H = A^ + gamma E^, eigenvectors ascending, keep the J
    smallest; W = U~ W~, with images A W = Z_A W~, E W = Z_E W~ (no new applies)."""
    H = dense.sym(an.Ahat + gamma_J * an.Ehat)
    theta, Wt = np.linalg.eigh(H)
    k = min(J, Wt.shape[1])
    Wt = Wt[:, :k]
    return an.Ut @ Wt, an.ZA @ Wt, an.ZE @ Wt, theta[:k], Wt


def carried_direction(W: np.ndarray, g: np.ndarray | None):
    """Alg. 3 local update with the carried correction g^(k-1,l) (reading D3):
    two passes of classical Gram-Schmidt against W; dropped when
    ||(I - W W^T) g|| / ||g|| < sin(acos 0.999) (footnote P:691, reading G12)."""
    if g is None:
        return None
    ng = float(np.linalg.norm(g))
    if ng == 0.0:
        return None
    gh = g - W @ (W.T @ g)
    gh = gh - W @ (W.T @ gh)
    nh = float(np.linalg.norm(gh))
    if nh / ng < DUP_SIN:
        return None
    return gh / nh
