"""O2/O3: dense assembly and small dense tools (oracle, test-only).

numpy.linalg routines serve as the library primitives (QR, SVD, symmetric
eig, Cholesky); this module only states how the paper uses them.
"""
from __future__ import annotations

import numpy as np

from . import operators as ops


def assemble(apply, n: int) -> np.ndarray:
    """Dense N x N matrix of a linear image operator, column by column
    (the footnote construction of P:1085)."""
    N = n * n
    M = np.zeros((N, N))
    e = np.zeros((n, n))
    for k in range(N):
        e.flat[k] = 1.0
        M[:, k] = apply(e).ravel()
        e.flat[k] = 0.0
    return M


def assemble_shifted(h, wx, wy, gamma, n):
    return assemble(lambda v: ops.apply_shifted(h, wx, wy, gamma, v), n)


def sym(M: np.ndarray) -> np.ndarray:
    return 0.5 * (M + M.T)


def qr_pos(Y: np.ndarray):
    """Economy QR, Y = K R with diag(R) > 0 so the factors are unique (reading G16)."""
    K, R = np.linalg.qr(Y, mode="reduced")
    s = np.sign(np.diag(R))
    s[s == 0] = 1.0
    return K * s[None, :], R * s[:, None]


def tri_inv_apply(R: np.ndarray, B: np.ndarray) -> np.ndarray:
    """R^{-1} B for upper-triangular R (the implicit U = U~ R^{-1} of P:851)."""
    import scipy.linalg
    return scipy.linalg.solve_triangular(R, B, lower=False)


def tri_inv_t_apply(R: np.ndarray, B: np.ndarray) -> np.ndarray:
    """R^{-T} B."""
    import scipy.linalg
    return scipy.linalg.solve_triangular(R, B, lower=False, trans="T")


def cholesky_or_none(G: np.ndarray):
    try:
        return np.linalg.cholesky(G)
    except np.linalg.LinAlgError:
        return None


def chol_solve(L: np.ndarray, z: np.ndarray) -> np.ndarray:
    import scipy.linalg
    return scipy.linalg.cho_solve((L, True), z)
