"""Pins for oracle/operators.py (O1) and oracle/dense.py against things other than itself:
library routines that compute the same definition, adjoint identities, closed-form
impulse responses, null spaces and the golden fixture in tests/golden/."""
import json
import os

import numpy as np
import pytest
import scipy.signal

import rsk_synth as S
from oracle import dense
from oracle import operators as ops

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand_psf(seed, r):
    # deliberately NOT point-symmetric so a flipped tap or a transposed operand shows
    return S.random_vectors(seed, (2 * r + 1, 2 * r + 1), "uniform") + 0.1


@pytest.mark.parametrize("n,r", [(7, 1), (12, 2), (16, 4), (9, 4)])
def test_conv_is_scipy_convolve2d_same(n, r):
    h = _rand_psf(1 + n, r)
    x = S.random_vectors(2 + n, (n, n))
    ref = scipy.signal.convolve2d(x, h, mode="same", boundary="fill", fillvalue=0.0)
    np.testing.assert_allclose(ops.conv(h, x), ref, rtol=0, atol=1e-13)


@pytest.mark.parametrize("n,r", [(7, 1), (12, 2), (16, 4)])
def test_conv_t_is_scipy_correlate2d_same(n, r):
    h = _rand_psf(3 + n, r)
    y = S.random_vectors(4 + n, (n, n))
    ref = scipy.signal.correlate2d(y, h, mode="same", boundary="fill", fillvalue=0.0)
    np.testing.assert_allclose(ops.conv_t(h, y), ref, rtol=0, atol=1e-13)


def test_conv_adjoint_identity():
    n, r = 11, 3
    h = _rand_psf(5, r)
    x = S.random_vectors(6, (n, n)); y = S.random_vectors(7, (n, n))
    lhs = np.sum(ops.conv(h, x) * y)
    rhs = np.sum(x * ops.conv_t(h, y))
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)


def test_conv_delta_and_shift_psf():
    n = 8
    x = S.random_vectors(8, (n, n))
    d = np.zeros((3, 3)); d[1, 1] = 1.0
    np.testing.assert_array_equal(ops.conv(d, x), x)
    s = np.zeros((3, 3)); s[1, 2] = 1.0          # h[a+r, b+r] with (a, b) = (0, 1): y[i,j] = x[i, j-1]
    y = ops.conv(s, x)
    np.testing.assert_array_equal(y[:, 1:], x[:, :-1])
    np.testing.assert_array_equal(y[:, 0], 0.0)


def test_A_impulse_interior_is_psf_autocorrelation():
    """Interior column of A = C^T C equals the full autocorrelation of h (closed form)."""
    n, r = 21, 3
    h = _rand_psf(9, r)
    e = np.zeros((n, n)); c = n // 2; e[c, c] = 1.0
    col = ops.apply_A(h, e)
    ac = np.zeros((4 * r + 1, 4 * r + 1))
    for da in range(-2 * r, 2 * r + 1):
        for db in range(-2 * r, 2 * r + 1):
            s = 0.0
            for a in range(-r, r + 1):
                for b in range(-r, r + 1):
                    if -r <= a + da <= r and -r <= b + db <= r:
                        s += h[a + r, b + r] * h[a + da + r, b + db + r]
            ac[da + 2 * r, db + 2 * r] = s
    np.testing.assert_allclose(col[c - 2 * r:c + 2 * r + 1, c - 2 * r:c + 2 * r + 1], ac,
                               rtol=1e-13, atol=1e-16)
    mask = np.ones((n, n), bool); mask[c - 2 * r:c + 2 * r + 1, c - 2 * r:c + 2 * r + 1] = False
    assert np.all(col[mask] == 0.0)


def test_E_null_space_and_zero_weights():
    n = 10
    wx, wy = S.random_weights(11, n)
    one = np.ones((n, n))
    assert np.max(np.abs(ops.apply_E(wx, wy, one))) <= 1e-12 * np.max(wx)
    z = np.zeros((n, n))
    x = S.random_vectors(12, (n, n))
    assert np.all(ops.apply_E(z, z, x) == 0.0)


def test_E_impulse_is_weighted_five_point():
    """E e_(i,j) in the interior = 5-point pattern with the four incident weights."""
    n = 9
    wx, wy = S.random_weights(13, n)
    i, j = 4, 5
    e = np.zeros((n, n)); e[i, j] = 1.0
    col = ops.apply_E(wx, wy, e)
    ref = np.zeros((n, n))
    ref[i, j] = wx[i, j - 1] + wx[i, j] + wy[i - 1, j] + wy[i, j]
    ref[i, j - 1] = -wx[i, j - 1]
    ref[i, j + 1] = -wx[i, j]
    ref[i - 1, j] = -wy[i - 1, j]
    ref[i + 1, j] = -wy[i, j]
    np.testing.assert_allclose(col, ref, rtol=1e-15, atol=0)
    # corner pixel: only the two existing differences contribute
    e = np.zeros((n, n)); e[0, 0] = 1.0
    col = ops.apply_E(wx, wy, e)
    assert col[0, 0] == pytest.approx(wx[0, 0] + wy[0, 0], rel=1e-15)


def test_E_is_LT_W_L_via_dense_difference_matrices():
    """Build L explicitly as a sparse-free dense matrix from its row definition."""
    n = 5; N = n * n
    wx, wy = S.random_weights(14, n)
    rows, wts = [], []
    for i in range(n):
        for j in range(n - 1):
            v = np.zeros(N); v[i * n + j + 1] = 1; v[i * n + j] = -1
            rows.append(v); wts.append(wx[i, j])
    for i in range(n - 1):
        for j in range(n):
            v = np.zeros(N); v[(i + 1) * n + j] = 1; v[i * n + j] = -1
            rows.append(v); wts.append(wy[i, j])
    Lm = np.array(rows)
    assert Lm.shape[0] == 2 * n * (n - 1)          # 2n(n-1) rows
    Em = Lm.T @ np.diag(wts) @ Lm
    x = S.random_vectors(15, (n, n))
    np.testing.assert_allclose(ops.apply_E(wx, wy, x).ravel(), Em @ x.ravel(), rtol=1e-13, atol=1e-12)


def test_shifted_dense_symmetric_pd_and_linear():
    n = 6
    h = S.gaussian_psf(2, 1.0)
    wx, wy = S.random_weights(16, n, 0.5, 50.0)
    for g in (0.0, 1e-4, 1.0, 30.0):
        Ag = dense.assemble_shifted(h, wx, wy, g, n)
        assert np.max(np.abs(Ag - Ag.T)) <= 1e-13 * np.max(np.abs(Ag))
        if g > 0:
            assert np.linalg.eigvalsh(Ag).min() > 0
    x = S.random_vectors(17, (n, n)); y = S.random_vectors(18, (n, n))
    g = 0.37
    ax = ops.apply_shifted(h, wx, wy, g, x); ay = ops.apply_shifted(h, wx, wy, g, y)
    s1 = np.sum(ax * y); s2 = np.sum(ay * x)
    assert abs(s1 - s2) <= 1e-13 * abs(s1)
    lin = ops.apply_shifted(h, wx, wy, g, 2.5 * x - 0.5 * y)
    np.testing.assert_allclose(lin, 2.5 * ax - 0.5 * ay, rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(ops.apply_shifted(h, wx, wy, 0.0, x), ops.apply_A(h, x), rtol=0, atol=0)


def test_irn_weights_closed_forms():
    n = 6; tau = 1e-3
    x = np.full((n, n), 0.3)
    wx, wy = ops.irn_weights(x, tau)
    assert np.all(wx[:, :-1] == 1.0 / tau) and np.all(wx[:, -1] == 0.0)
    assert np.all(wy[:-1, :] == 1.0 / tau) and np.all(wy[-1, :] == 0.0)
    x = np.zeros((n, n)); x[:, 3:] = 0.5                 # one vertical edge of height 0.5
    wx, wy = ops.irn_weights(x, tau)
    assert np.all(wx[:, 2] == 1.0 / np.sqrt(0.25 + tau * tau))
    assert np.all(wx[:, [0, 1, 3, 4]] == 1.0 / tau)
    assert np.all(wy[:-1, :] == 1.0 / tau)


def test_seminorm_matches_E_quadratic_form():
    n = 7
    wx, wy = S.random_weights(19, n)
    x = S.random_vectors(20, (n, n))
    assert ops.seminorm2(wx, wy, x) == pytest.approx(float(np.sum(x * ops.apply_E(wx, wy, x))), rel=1e-13)


def test_make_data_noise_level():
    cfg = S.small_config(n=12)
    inp = S.make_inputs(cfg)
    d, b = ops.make_data(inp["psf"], inp["x_true"], inp["xi"], 0.02)
    cx = ops.conv(inp["psf"], inp["x_true"])
    assert np.linalg.norm(d - cx) == pytest.approx(0.02 * np.linalg.norm(cx), rel=1e-13)
    np.testing.assert_allclose(b, ops.conv_t(inp["psf"], d), rtol=0, atol=0)


def test_golden_hand_computed_apply():
    """tests/golden/apply_3x3.json: a 3x3 image worked by hand (see the fixture's note)."""
    with open(os.path.join(GOLDEN, "apply_3x3.json")) as f:
        gdat = json.load(f)
    h = np.array(gdat["psf"]); x = np.array(gdat["x"])
    np.testing.assert_allclose(ops.conv(h, x), np.array(gdat["Cx"]), rtol=0, atol=1e-15)
    wx = np.array(gdat["wx"]); wy = np.array(gdat["wy"])
    np.testing.assert_allclose(ops.apply_E(wx, wy, x), np.array(gdat["Ex"]), rtol=0, atol=1e-15)
