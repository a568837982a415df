"""O1: the operators of the shifted family, written out literally (oracle, test-only).

Images are n x n arrays, row index i (y), column index j (x); a vector x of
length N = n^2 is the row-major flattening (pixel (i, j) at i*n + j).

PAPER.md:
  * forward model d = C x + e                         eq:forward
  * normal equations (C^T C + lambda^2 L^T D^2 L) x = C^T d   eq:blkeqn P:126-128
  * A = C^T C, E_0 = L^T L, b = C^T d, gamma = lambda^2
  * E_k = L^T D_k^2 L                                 P:147, eq:shift P:365
  * L = [Delta_x; Delta_y], discrete derivatives
  * C: symmetric Gaussian blur, zero boundary
North-star (BASELINE.json): E_k = L^T W_k L with the IRN weights
  w_i = ((L x)_i^2 + tau^2)^(-1/2), W_0 = I            (reading G2/G3)
SURVEY §8(f) f1 (the paper's own outer step): Gazzola's rule P:144-152, isotropic
  IRN, the 3-consecutive-lambda* stopping rule P:1042.
"""
from __future__ import annotations

import numpy as np


def _psf_r(h: np.ndarray) -> int:
    ph, pw = h.shape
    if ph != pw or ph % 2 != 1:
        raise ValueError("PSF must be square with odd size")
    return ph // 2


def conv(h: np.ndarray, x: np.ndarray) -> np.ndarray:
    """C x: 'same'-size 2-D convolution with zero boundary (reading G20).

    y[i, j] = sum_{a, b = -r..r} h[a+r, b+r] * x[i-a, j-b], summed over the
    in-range pixels (i-a, j-b) only.
    """
    if hasattr(h, "forward"):          # an explicit operator (CT, oracle/ct.py)
        return h.forward(x)
    r = _psf_r(h)
    n0, n1 = x.shape
    xp = np.zeros((n0 + 2 * r, n1 + 2 * r))
    xp[r:r + n0, r:r + n1] = x
    y = np.zeros((n0, n1))
    for a in range(-r, r + 1):
        for b in range(-r, r + 1):
            # x[i-a, j-b] = xp[r+i-a, r+j-b]
            y += h[a + r, b + r] * xp[r - a:r - a + n0, r - b:r - b + n1]
    return y


def conv_t(h: np.ndarray, y: np.ndarray) -> np.ndarray:
    """C^T y: the literal scatter adjoint of `conv`.

    For every (i, j) and (a, b) with (i-a, j-b) in range:
        out[i-a, j-b] += h[a+r, b+r] * y[i, j].
    """
    if hasattr(h, "adjoint"):          # an explicit operator (CT, oracle/ct.py)
        return h.adjoint(y)
    r = _psf_r(h)
    n0, n1 = y.shape
    op = np.zeros((n0 + 2 * r, n1 + 2 * r))
    for a in range(-r, r + 1):
        for b in range(-r, r + 1):
            op[r - a:r - a + n0, r - b:r - b + n1] += h[a + r, b + r] * y
    return op[r:r + n0, r:r + n1].copy()


def apply_A(h: np.ndarray, x: np.ndarray) -> np.ndarray:
    """A x = C^T (C x)."""
    return conv_t(h, conv(h, x))


def grad(x: np.ndarray):
    """L x = (Dx x, Dy x), forward differences without boundary rows (reading G4):
    (Dx x)[i, j] = x[i, j+1] - x[i, j] for j <= n-2; (Dy x)[i, j] = x[i+1, j] - x[i, j]
    for i <= n-2. Shapes (n, n-1) and (n-1, n)."""
    return x[:, 1:] - x[:, :-1], x[1:, :] - x[:-1, :]


def grad_t(qx: np.ndarray, qy: np.ndarray) -> np.ndarray:
    """L^T (qx, qy): the literal scatter adjoint of `grad`."""
    n = qx.shape[0]
    out = np.zeros((n, n))
    for j in range(n - 1):
        out[:, j + 1] += qx[:, j]
        out[:, j] -= qx[:, j]
    for i in range(n - 1):
        out[i + 1, :] += qy[i, :]
        out[i, :] -= qy[i, :]
    return out


def identity_weights(n: int):
    """W_0 = I on the n(n-1) rows of each derivative; padded layout (n, n) with
    wx[:, n-1] = 0 and wy[n-1, :] = 0 (SURVEY §8.0 data layout)."""
    wx = np.ones((n, n))
    wy = np.ones((n, n))
    wx[:, n - 1] = 0.0
    wy[n - 1, :] = 0.0
    return wx, wy


def apply_E(wx: np.ndarray, wy: np.ndarray, x: np.ndarray) -> np.ndarray:
    """E x = L^T (W (L x)) with W = diag(wx, wy) (P:147 with W_k = D_k^2)."""
    qx, qy = grad(x)
    return grad_t(wx[:, :-1] * qx, wy[:-1, :] * qy)


def apply_shifted(h, wx, wy, gamma: float, x: np.ndarray) -> np.ndarray:
    """(A + gamma E_k) x  (eq:seqsys P:47, eq:shift P:361-365)."""
    return apply_A(h, x) + gamma * apply_E(wx, wy, x)


def irn_weights(x: np.ndarray, tau: float):
    """IRN weights w_i = ((L x)_i^2 + tau^2)^(-1/2) (north_star; IRN family P:60),
    one weight per row of L (anisotropic, reading G3), pads = 0."""
    n = x.shape[0]
    qx, qy = grad(x)
    wx = np.zeros((n, n))
    wy = np.zeros((n, n))
    wx[:, :-1] = 1.0 / np.sqrt(qx * qx + tau * tau)
    wy[:-1, :] = 1.0 / np.sqrt(qy * qy + tau * tau)
    return wx, wy


def irn_weights_iso(x: np.ndarray, tau: float):
    """Isotropic IRN weights (the isotropic TV term of P:117 with
    beta = tau^2): one weight per PIXEL p,
        w_p = ((Dx x)_p^2 + (Dy x)_p^2 + tau^2)^(-1/2),
    a difference that does not exist at p (last column / last row) counting 0
    (reading G32), placed on both rows of L at p; pads = 0."""
    n = x.shape[0]
    qx, qy = grad(x)
    gx = np.zeros((n, n))
    gy = np.zeros((n, n))
    gx[:, :-1] = qx
    gy[:-1, :] = qy
    w = 1.0 / np.sqrt(gx * gx + gy * gy + tau * tau)
    wx = w.copy()
    wy = w.copy()
    wx[:, n - 1] = 0.0
    wy[n - 1, :] = 0.0
    return wx, wy


def gazzola_step(dx: np.ndarray, dy: np.ndarray, x: np.ndarray, p: float):
    """Gazzola's edge-preserving update of the paper's own outer loop:
        q = L x,   w = |D_k q| / ||D_k q||_inf,   w <- 1 - w.^p,   D_{k+1} = diag(w) D_k,
    E_{k+1} = L^T D_{k+1}^2 L. D_k is diagonal over the 2 n(n-1) rows of L and is
    held in the padded layout of the weights (dx on the Dx rows, dy on the Dy rows,
    pads 0); D_0 = I (E_0 = L^T L). p is never given by the paper (default 2,
    SPEC S:421). ||D_k q||_inf = 0 (x constant along every row with D_k > 0): w = 0,
    so D_{k+1} = D_k (reading G31).
    Returns (dx', dy') = D_{k+1} and (wx', wy') = D_{k+1}^2, the weights E uses."""
    qx, qy = grad(x)
    tx = np.abs(dx[:, :-1] * qx)
    ty = np.abs(dy[:-1, :] * qy)
    m = max(float(tx.max(initial=0.0)), float(ty.max(initial=0.0)))
    if m > 0.0:
        wxr = tx / m
        wyr = ty / m
    else:
        wxr = np.zeros_like(tx)
        wyr = np.zeros_like(ty)
    wxr = 1.0 - wxr ** p
    wyr = 1.0 - wyr ** p
    ndx = np.zeros_like(dx)
    ndy = np.zeros_like(dy)
    ndx[:, :-1] = wxr * dx[:, :-1]
    ndy[:-1, :] = wyr * dy[:-1, :]
    return (ndx, ndy), (ndx * ndx, ndy * ndy)


def lstar_settled(history, count: int = 3) -> bool:
    """The paper's outer stopping rule: stop 'once the selected lambda is the
    same for three consecutive iterations' -- the last `count` L-curve choices are one
    shift index (the shift grid is fixed, so equal lambda = equal index)."""
    return len(history) >= count and len(set(history[-count:])) == 1


def seminorm2(wx, wy, x) -> float:
    """||W^(1/2) L x||^2 = sum wx (Dx x)^2 + sum wy (Dy x)^2, the L-curve's
    vertical coordinate under the current E_k (reading G25)."""
    qx, qy = grad(x)
    return float(np.sum(wx[:, :-1] * qx * qx) + np.sum(wy[:-1, :] * qy * qy))


def make_data(h, x_true, xi, nu):
    """d = C x_true + e with ||e|| = nu ||C x_true|| and e parallel to xi (eq:forward P:107,
    reading G21); b = C^T d."""
    cx = conv(h, x_true)
    e = nu * np.linalg.norm(cx) * xi / np.linalg.norm(xi)
    d = cx + e
    return d, conv_t(h, d)
