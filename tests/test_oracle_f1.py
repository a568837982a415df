"""Pins for the f1 outer-step rules of the oracle:
Gazzola's weight update, isotropic IRN weights and the
3-consecutive-lambda* stopping rule -- against closed forms on step/ramp
images, a dense L built row by row from its definition, and invariants the paper
states (weights bounded by 1 and non-increasing in k)."""
import numpy as np
import pytest

import rsk_synth as S
from oracle import operators as ops


def _dense_L(n):
    """L = [Delta_x; Delta_y] as a dense matrix, one row per difference, in the
    order (Dx rows i-major, then Dy rows i-major), plus the padded-layout index of each row."""
    N = n * n
    rows, where = [], []
    for i in range(n):
        for j in range(n - 1):
            v = np.zeros(N); v[i * n + j + 1] = 1; v[i * n + j] = -1
            rows.append(v); where.append(("x", i, j))
    for i in range(n - 1):
        for j in range(n):
            v = np.zeros(N); v[(i + 1) * n + j] = 1; v[i * n + j] = -1
            rows.append(v); where.append(("y", i, j))
    return np.array(rows), where


def _to_rows(dx, dy, where):
    return np.array([(dx if a == "x" else dy)[i, j] for (a, i, j) in where])


def test_gazzola_step_edge_closed_form():
    """Two vertical edges of heights 1 and 0.5 on a flat background, D_0 = I:
    w = 1 on the tall edge -> D_1 = 0 there; w = 0.5 on the short one -> 1 - 0.5^p;
    every other row keeps 1. Second step: the short edge is now the maximum -> 0."""
    n = 8
    x = np.zeros((n, n)); x[:, 3:] = 1.0; x[:, 6:] = 1.5
    for p in (1.0, 2.0, 3.0):
        D0 = ops.identity_weights(n)
        (dx, dy), (wx, wy) = ops.gazzola_step(D0[0], D0[1], x, p)
        assert np.all(dx[:, 2] == 0.0)
        assert np.all(dx[:, 5] == 1.0 - 0.5 ** p)
        assert np.all(dx[:, [0, 1, 3, 4, 6]] == 1.0) and np.all(dx[:, 7] == 0.0)
        assert np.all(dy[:-1, :] == 1.0) and np.all(dy[-1, :] == 0.0)
        np.testing.assert_array_equal(wx, dx * dx)
        np.testing.assert_array_equal(wy, dy * dy)
        (dx2, dy2), _ = ops.gazzola_step(dx, dy, x, p)
        # |D_1 q|: 0 on the tall edge, (1 - 0.5^p) * 0.5 on the short one = the max
        assert np.all(dx2[:, 2] == 0.0) and np.all(dx2[:, 5] == 0.0)
        assert np.all(dx2[:, [0, 1, 3, 4, 6]] == 1.0)


def test_gazzola_step_ramp_and_constant():
    n = 7
    j = np.arange(n, dtype=float)
    x = np.tile(0.25 * j, (n, 1))            # Dx x = 0.25 everywhere, Dy x = 0
    D0 = ops.identity_weights(n)
    (dx, dy), _ = ops.gazzola_step(D0[0], D0[1], x, 2.0)
    assert np.all(dx == 0.0)                 # every x-row is a maximum
    assert np.all(dy[:-1, :] == 1.0) and np.all(dy[-1, :] == 0.0)
    # constant image: ||D q||_inf = 0 -> D unchanged (reading G31)
    (cx, cy), _ = ops.gazzola_step(D0[0], D0[1], np.full((n, n), 3.0), 2.0)
    np.testing.assert_array_equal(cx, D0[0])
    np.testing.assert_array_equal(cy, D0[1])


@pytest.mark.parametrize("p", [0.5, 2.0, 2.5])
def test_gazzola_step_matches_dense_L_definition(p):
    """D_{k+1} = diag(1 - (|D_k L x| / ||D_k L x||_inf)^p) D_k with L assembled from its
    rows; two chained steps from a random positive D_k."""
    n = 6
    Lm, where = _dense_L(n)
    g = np.random.Generator(np.random.PCG64(31))
    dx, dy = S.random_weights(32, n, 0.2, 1.0)
    x = S.random_vectors(33, (n, n))
    d = _to_rows(dx, dy, where)
    for _ in range(2):
        q = Lm @ x.ravel()
        w = np.abs(d * q) / np.max(np.abs(d * q))
        d_ref = (1.0 - w ** p) * d
        (dx, dy), (wx, wy) = ops.gazzola_step(dx, dy, x, p)
        np.testing.assert_allclose(_to_rows(dx, dy, where), d_ref, rtol=1e-14, atol=1e-15)
        np.testing.assert_allclose(_to_rows(wx, wy, where), d_ref ** 2, rtol=1e-14, atol=1e-15)
        assert np.all(dx[:, -1] == 0.0) and np.all(dy[-1, :] == 0.0)
        d = d_ref
        x = x + 0.3 * S.random_vectors(int(g.integers(1 << 30)), (n, n))


def test_gazzola_invariants_bounded_monotone_scale_free():
    """0 <= D_{k+1} <= D_k <= 1, at least one row hits 0 (the max), and the rule
    is invariant to scaling x (w is a ratio)."""
    n = 9
    x = S.random_vectors(40, (n, n))
    D = ops.identity_weights(n)
    for k in range(4):
        (dx, dy), _ = ops.gazzola_step(D[0], D[1], x, 2.0)
        assert np.all(dx >= 0) and np.all(dy >= 0)
        assert np.all(dx <= D[0]) and np.all(dy <= D[1])
        assert min(dx[:, :-1].min(), dy[:-1, :].min()) == 0.0
        (sx, sy), _ = ops.gazzola_step(D[0], D[1], 64.0 * x, 2.0)     # power of 2: exact
        np.testing.assert_array_equal(sx, dx)
        np.testing.assert_array_equal(sy, dy)
        D = (dx, dy)


def test_irn_iso_closed_form_and_dense_L():
    n = 5; tau = 1e-2
    x = np.zeros((n, n))
    x[2, 3] = 3.0                             # pixel (2,2): Dx = 3; pixel (1,3): Dy = 3
    wx, wy = ops.irn_weights_iso(x, tau)
    assert wx[2, 2] == 1.0 / np.sqrt(9.0 + tau * tau) == wy[2, 2]
    assert wx[1, 3] == 1.0 / np.sqrt(9.0 + tau * tau) == wy[1, 3]
    # pixel (2,3): Dx = -3, Dy = -3 -> |grad|^2 = 18
    assert wx[2, 3] == 1.0 / np.sqrt(18.0 + tau * tau) == wy[2, 3]
    assert np.all(wx[:, -1] == 0.0) and np.all(wy[-1, :] == 0.0)
    # against the per-pixel definition with L's rows assembled explicitly
    Lm, where = _dense_L(n)
    x = S.random_vectors(41, (n, n))
    q = Lm @ x.ravel()
    g2 = np.zeros(n * n)
    for (a, i, j), v in zip(where, q):
        g2[i * n + j] += v * v
    wpix = 1.0 / np.sqrt(g2 + tau * tau)
    ref = np.array([wpix[i * n + j] for (a, i, j) in where])
    wx, wy = ops.irn_weights_iso(x, tau)
    np.testing.assert_allclose(_to_rows(wx, wy, where), ref, rtol=1e-15)


def test_irn_iso_reduces_to_anisotropic_for_one_direction():
    n = 6; tau = 1e-3
    x = np.tile(np.cumsum(S.random_vectors(42, (n,))), (n, 1))    # varies along j only
    ax, ay = ops.irn_weights(x, tau)
    ix, iy = ops.irn_weights_iso(x, tau)
    np.testing.assert_array_equal(ix, ax)
    # Dy = 0 everywhere: the Dy rows see the pixel's Dx (isotropic) instead of 1/tau
    np.testing.assert_array_equal(iy[:-1, :-1], ax[:-1, :-1])
    assert np.all(iy[:-1, -1] == 1.0 / tau)


def test_lstar_settled_rule():
    assert not ops.lstar_settled([])
    assert not ops.lstar_settled([4, 4])
    assert ops.lstar_settled([4, 4, 4])
    assert not ops.lstar_settled([4, 4, 5])
    assert ops.lstar_settled([1, 7, 5, 5, 5])
    assert not ops.lstar_settled([5, 5, 6, 5, 5])


def test_oracle_run_gazzola_and_stop_rule():
    """Tiny nested solve with Gazzola's rule and the P:1042 stop: weights stay in [0, 1]
    and non-increasing; the run stops exactly when three l* agree (or at K_out)."""
    import dataclasses
    from oracle import pipeline as op
    cfg = dataclasses.replace(S.small_config(n=12, M=5, K_out=6), weight_rule="gazzola",
                              stop="lstar3")
    inp = S.make_inputs(cfg)
    out = op.run(cfg, inp)
    hist = out["lstar"]
    assert len(out["steps"]) == len(hist)
    for k in range(len(hist)):
        if ops.lstar_settled(hist[:k + 1]):
            assert k + 1 == len(hist)
    if len(hist) < cfg.K_out:
        assert ops.lstar_settled(hist)
    wx, wy = out["final_weights"]
    assert np.all((wx >= 0) & (wx <= 1)) and np.all((wy >= 0) & (wy <= 1))
    for st in out["steps"]:
        assert np.all(st.status == 0)
