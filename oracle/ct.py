"""Parallel-beam CT operator of Example 2.
ORACLE, TEST INFRASTRUCTURE ONLY.

C is "the discrete Radon transform matrix for parallel beam CT corresponding to taking
measurements angles from 1 to 135 degrees in increments of 1 degree", "normalized
so that C has unit Frobenius norm". Reading G38: the line-integral
model -- entry (ray, pixel) = length of the ray's segment inside the pixel square.

Geometry: pixel (i, j) (row i from the top, column j) is the unit square
x in [j - n/2, j + 1 - n/2], y in [n/2 - i - 1, n/2 - i]; ray (theta, s) is the line
{x cos(theta) + y sin(theta) = s}; detector d sits at s_d = d - (ndet - 1)/2 (unit bins,
ndet = 2 ceil(n/sqrt 2) + 2); rows of C are ordered (angle, detector).

Literal and slow: every entry is the clipped length of the line in the pixel square
(Liang-Barsky clipping of the parametric line p(t) = s (cos, sin) + t (-sin, cos) against
the square, |d p / d t| = 1; a line lying on a pixel face counts for the pixel on its
high side only), evaluated for all pixels of a ray at once. The operator is
assembled as a dense (m x N) matrix (n = 82: 15930 x 6724). Pinned in
tests/test_oracle_ct.py (chord lengths through the image square, axis-aligned rays,
single-pixel diagonals, unit Frobenius norm).
"""
from __future__ import annotations

import numpy as np


def clipped_lengths(theta: float, s: float, n: int) -> np.ndarray:
    """Length of the ray (theta [rad], s) inside each pixel square, as an (n, n) array."""
    c, sn = np.cos(theta), np.sin(theta)
    p0 = np.array([s * c, s * sn])
    u = np.array([-sn, c])
    jj, ii = np.meshgrid(np.arange(n), np.arange(n))
    x0 = jj - n / 2.0
    x1 = x0 + 1.0
    y1 = n / 2.0 - ii
    y0 = y1 - 1.0
    lo = np.full((n, n), -np.inf)
    hi = np.full((n, n), np.inf)
    inside = np.ones((n, n), dtype=bool)
    for comp, a, b in ((0, x0, x1), (1, y0, y1)):
        if abs(u[comp]) < 1e-15:
            # line parallel to this pair of faces: inside iff the coordinate lies in the
            # half-open [a, b) (a line on a shared face belongs to one pixel, not both)
            inside &= (p0[comp] >= a) & (p0[comp] < b)
            continue
        t_a = (a - p0[comp]) / u[comp]
        t_b = (b - p0[comp]) / u[comp]
        lo = np.maximum(lo, np.minimum(t_a, t_b))
        hi = np.minimum(hi, np.maximum(t_a, t_b))
    out = np.where(inside, np.maximum(hi - lo, 0.0), 0.0)
    out[~np.isfinite(out)] = 0.0
    return out


class CTOperator:
    """C (m x N) as a dense matrix, rows (angle, detector); forward = C x, adjoint = C^T y."""

    def __init__(self, n: int, angles_deg, ndet: int, normalize: bool = True):
        self.n, self.ndet = n, ndet
        self.angles = np.asarray(angles_deg, dtype=np.float64)
        m = len(self.angles) * ndet
        C = np.zeros((m, n * n))
        row = 0
        for a in self.angles:
            th = np.deg2rad(a)
            for d in range(ndet):
                s = d - (ndet - 1) / 2.0
                C[row] = clipped_lengths(th, s, n).ravel()
                row += 1
        self.fro_unscaled = float(np.linalg.norm(C))
        if normalize:
            C /= self.fro_unscaled
        self.C = C

    @property
    def m(self) -> int:
        return self.C.shape[0]

    def forward(self, x: np.ndarray) -> np.ndarray:
        return self.C @ np.asarray(x).ravel()

    def adjoint(self, y: np.ndarray) -> np.ndarray:
        return (self.C.T @ np.asarray(y).ravel()).reshape(self.n, self.n)
