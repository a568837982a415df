"""Pins of the Example-1-shaped workload (config C7, reading G40): the oracle's blur with
the rank-2 PSF is exactly the paper's C = sum_{i=1,2} C_i^(1) (x) C_i^(2) built from
explicit Toeplitz matrices (§8.2; Regtools' blur: T = toeplitz(z),
z_k = exp(-k^2 / (2 sigma^2)) for k < bandwidth), up to the normalisation sum h = 1."""
import numpy as np
import scipy.linalg

import rsk_synth as S
from oracle import dense
from oracle import operators as ops


def _toeplitz(n, band, sigma):
    z = np.zeros(n)
    k = np.arange(min(band, n))
    z[:len(k)] = np.exp(-k ** 2 / (2.0 * sigma * sigma))
    return scipy.linalg.toeplitz(z)


def test_c7_blur_is_the_kronecker_sum():
    cfg = S.CONFIGS["C7"]
    h = S.make_inputs(cfg)["psf"]
    n = 30
    # row-major image x[i, j] (i: y, j: x): (T_y (x) T_x) vec_row(X) = vec_row(T_y X T_x^T)
    Cd = dense.assemble(lambda v: ops.conv(h, v), n)
    K = np.zeros((n * n, n * n))
    for bx, sx, by, sy in cfg.psf_terms:
        K += np.kron(_toeplitz(n, by, sy), _toeplitz(n, bx, sx))
    K /= sum(np.outer(np.where(np.abs(np.arange(-11, 12)) <= by - 1, np.exp(-np.arange(-11, 12) ** 2 / (2 * sy * sy)), 0),
                      np.where(np.abs(np.arange(-11, 12)) <= bx - 1, np.exp(-np.arange(-11, 12) ** 2 / (2 * sx * sx)), 0)).sum()
             for bx, sx, by, sy in cfg.psf_terms)
    assert np.max(np.abs(Cd - K)) <= 1e-15 * np.max(np.abs(K))


def test_c7_psf_rank_two_and_paper_indices():
    cfg = S.CONFIGS["C7"]
    h = S.make_inputs(cfg)["psf"]
    s = np.linalg.svd(h, compute_uv=False)
    assert h.shape == (23, 23) and abs(h.sum() - 1.0) < 1e-15
    assert s[1] > 1e-6 * s[0] and s[2] < 1e-15 * s[0]
    from oracle.indices import of
    ix = of(cfg)
    assert (ix.i1, ix.i2, ix.istar, ix.I, ix.J_L, ix.J_R, ix.l_c) == (1, 10, 10, 15, 15, 19, 18)
    lam = np.sqrt(S.make_inputs(cfg)["gamma"])
    np.testing.assert_allclose(lam, np.logspace(-4, 2.5, 20), rtol=1e-13)
