"""CPU-side checks of the boundary: librsk builds for sm_100a, loads, exports every
symbol include/rsk.h declares, and the host-only helpers agree with closed forms."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "rsk.h")


def _declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:rsk_status|size_t|const char\*)\s+(rsk_\w+)\s*\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2306_15049_b200 import build
    build.build()
    from paper_2306_15049_b200 import _lib
    return _lib.load()


def test_every_declared_symbol_is_exported_and_bound(lib):
    from paper_2306_15049_b200 import _lib
    decl = _declared()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), name
        assert name in _lib.EXPORTED, f"{name} has no ctypes signature"


def test_sm100a_cubin_present():
    import subprocess
    so = os.path.join(ROOT, "paper_2306_15049_b200", "librsk.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_version(lib):
    assert b"sm_100a" in lib.rsk_version()


def test_host_sym_eig_and_svd():
    from paper_2306_15049_b200 import rsk
    rng = np.random.default_rng(3)
    A = rng.standard_normal((9, 9)); H = A + A.T
    th, V = rsk.sym_eig(H)
    np.testing.assert_allclose(th, np.linalg.eigvalsh(H), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(H @ V, V * th, atol=1e-11)
    R = np.triu(rng.standard_normal((7, 7)))
    U, s, Vt = rsk.svd_small(R)
    np.testing.assert_allclose(s, np.linalg.svd(R, compute_uv=False), rtol=1e-12)
    np.testing.assert_allclose(U @ np.diag(s) @ Vt.T, R, atol=1e-12)


def test_host_orth_guess_matches_normal_equations():
    """rsk_orth_guess vs eq:orthupdate solved densely (independent numpy formulation)."""
    from paper_2306_15049_b200 import rsk
    rng = np.random.default_rng(4)
    N, nc = 60, 6
    Ut, _ = np.linalg.qr(rng.standard_normal((N, nc)))
    Ad = rng.standard_normal((N, N)); Ad = Ad @ Ad.T / N + np.eye(N)
    Ed = rng.standard_normal((N, N)); Ed = Ed @ Ed.T / N
    b = rng.standard_normal(N)
    gs = 0.3
    ZA, ZE = Ad @ Ut, Ed @ Ut
    K, R = np.linalg.qr(ZA + gs * ZE)
    sg = np.sign(np.diag(R)); K = K * sg; R = R * sg[:, None]
    gammas = np.array([0.0, 0.01, 0.3, 5.0])
    C, st = rsk.orth_guess(R, K.T @ ZE, ZE.T @ ZE, ZE.T @ b, K.T @ b, gs, gammas)
    assert np.all(st == 0)
    for l, g in enumerate(gammas):
        coef, *_ = np.linalg.lstsq((Ad + g * Ed) @ Ut, b, rcond=None)
        np.testing.assert_allclose(C[:, l], coef, rtol=1e-8, atol=1e-10)


def test_host_oblique_guess_matches_petrov_galerkin():
    """rsk_oblique_guess vs eq:obliqueupdate in the independent form
    (K^T (A + gamma E) U~) c = K^T b (K^T r_0 = 0), solved densely."""
    from paper_2306_15049_b200 import rsk
    rng = np.random.default_rng(5)
    N, nc = 60, 6
    Ut, _ = np.linalg.qr(rng.standard_normal((N, nc)))
    Ad = rng.standard_normal((N, N)); Ad = Ad @ Ad.T / N + np.eye(N)
    Ed = rng.standard_normal((N, N)); Ed = Ed @ Ed.T / N
    b = rng.standard_normal(N)
    ga = 0.3
    ZA, ZE = Ad @ Ut, Ed @ Ut
    K, R = np.linalg.qr(ZA + ga * ZE)
    sg = np.sign(np.diag(R)); K = K * sg; R = R * sg[:, None]
    gammas = np.array([0.0, 0.01, 0.3, 5.0])
    C, st = rsk.oblique_guess(R, K.T @ ZE, K.T @ b, ga, gammas)
    assert np.all(st == 0)
    for l, g in enumerate(gammas):
        coef = np.linalg.solve(K.T @ (Ad + g * Ed) @ Ut, K.T @ b)
        np.testing.assert_allclose(C[:, l], coef, rtol=1e-9, atol=1e-11)
    # a singular system: K^T E U = -I / delta at delta = 1 -> I + P = 0
    Rs = np.eye(3)
    C, st = rsk.oblique_guess(Rs, -np.eye(3), np.ones(3), 0.0, np.array([1.0, 0.0]))
    assert st[0] == 6 and np.all(C[:, 0] == 0) and st[1] == 0
    np.testing.assert_array_equal(C[:, 1], np.ones(3))


def test_host_lcurve_corner_matches_oracle():
    from oracle import pipeline
    from paper_2306_15049_b200 import rsk
    rng = np.random.default_rng(5)
    rho = np.exp(np.cumsum(rng.uniform(0, 1, 20)))
    eta = np.exp(-np.cumsum(rng.uniform(0, 1, 20)))
    assert rsk.lcurve_corner(rho, eta)[0] == pipeline.lcurve_corner(rho, eta)[0]


def test_host_stabilize_small_cut():
    from paper_2306_15049_b200 import rsk
    rng = np.random.default_rng(6)
    Qa, _ = np.linalg.qr(rng.standard_normal((10, 10)))
    Qb, _ = np.linalg.qr(rng.standard_normal((10, 10)))
    R = Qa @ np.diag(np.logspace(0, -16, 10)) @ Qb.T
    Zs, nk = rsk.stabilize_small(R, np.ones(10), 1e10, 0)
    assert nk == int(np.sum(1.0 / np.logspace(0, -16, 10) < 1e10))
    Zs3, nk3 = rsk.stabilize_small(R, np.ones(10), 1e10, 3)
    assert nk3 == 3


def test_create_ct_argument_errors_need_no_device(lib):
    """rsk_create_ct rejects bad geometry before touching the device (EINVAL = 1)."""
    import ctypes as C
    from paper_2306_15049_b200 import _lib as L
    h = C.c_void_p()
    ang = np.arange(1, 11, dtype=np.float64)
    hp = ang.ctypes.data_as(C.POINTER(C.c_double))
    assert lib.rsk_create_ct(C.byref(h), 0, 1, 10, hp, 8, 0) == L.RSK_EINVAL         # n < 2
    assert lib.rsk_create_ct(C.byref(h), 0, 16, 0, hp, 8, 0) == L.RSK_EINVAL         # no angles
    assert lib.rsk_create_ct(C.byref(h), 0, 16, 10, hp, 0, 0) == L.RSK_EINVAL        # no bins
    bad = ang.copy(); bad[3] = np.nan
    assert lib.rsk_create_ct(C.byref(h), 0, 16, 10, bad.ctypes.data_as(C.POINTER(C.c_double)), 8, 0) == L.RSK_EINVAL
    assert lib.rsk_ct_info(None, None, None, None) == L.RSK_EINVAL
    assert lib.rsk_minres_workspace_bytes(None, 4, 9) == 0


def test_create_slab_argument_errors_need_no_device(lib):
    """rsk_create_slab rejects bad slab geometry before touching the device."""
    import ctypes as C
    from paper_2306_15049_b200 import _lib as L
    import rsk_synth as S
    h = C.c_void_p()
    psf = np.ascontiguousarray(S.gaussian_psf(4, 2.0))
    hp = psf.ctypes.data_as(C.POINTER(C.c_double))
    assert lib.rsk_create_slab(C.byref(h), 0, 256, 256, 0, 64, hp, 9, 9, 7, 0) == L.RSK_EINVAL     # halo < 2r
    assert lib.rsk_create_slab(C.byref(h), 0, 256, 256, 250, 64, hp, 9, 9, 8, 0) == L.RSK_EINVAL   # past the image
    assert lib.rsk_create_slab(C.byref(h), 0, 256, 256, 0, 4, hp, 9, 9, 8, 0) == L.RSK_EINVAL      # rows < halo
    assert lib.rsk_slab_info(None, None) == L.RSK_EINVAL


def test_product_path_fails_loudly_without_the_library(tmp_path):
    """No CPU fallback: loading a missing librsk raises (the product path never routes
    through the oracle), and the package has no import of oracle/."""
    from paper_2306_15049_b200 import _lib as L
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        L.load(str(tmp_path / "librsk.so"))
    pkg = os.path.join(ROOT, "paper_2306_15049_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f


def test_host_svd_relative_accuracy_on_graded_triangle():
    """rsk_svd_small (QR-preconditioned one-sided Jacobi) resolves the singular values of a
    graded triangular factor (1 .. 1e-12) to high relative accuracy -- what Alg. 1's 1e10
    cut needs -- checked against a 50-digit SVD (mpmath)."""
    mpmath = pytest.importorskip("mpmath")
    from paper_2306_15049_b200 import rsk
    rng = np.random.default_rng(5)
    k = 40
    R = np.triu(rng.standard_normal((k, k))) * np.logspace(0, -12, k)
    U, s, Vt = rsk.svd_small(R)
    mpmath.mp.dps = 50
    sm = np.sort(np.array([float(x) for x in mpmath.svd_r(mpmath.matrix(R.tolist()), compute_uv=False)]))[::-1]
    assert np.max(np.abs(s - sm) / sm) <= 1e-8
    np.testing.assert_allclose(U @ np.diag(s) @ Vt.T, R, atol=1e-14)


@pytest.mark.parametrize("n", [2, 5, 17, 40, 121])
def test_host_sym_eig_against_lapack(n):
    """rsk_sym_eig (Householder tridiagonalisation + implicit Wilkinson-shift QR, host C++)
    against LAPACK's eigh: eigenvalues, eigenvector residuals and orthogonality, with a
    cluster of equal eigenvalues and a wide dynamic range."""
    from paper_2306_15049_b200 import rsk
    rng = np.random.default_rng(n)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.concatenate([np.logspace(-8, 4, n - n // 4), np.full(n // 4, 3.0)])
    H = (Q * lam) @ Q.T
    th, V = rsk.sym_eig(H)
    ref = np.linalg.eigvalsh(H)
    scale = np.max(np.abs(lam))
    assert np.all(np.diff(th) >= 0)
    assert np.max(np.abs(th - ref)) <= 1e-13 * scale
    assert np.max(np.abs(H @ V - V * th)) <= 1e-12 * scale
    assert np.max(np.abs(V.T @ V - np.eye(n))) <= 1e-13


def test_host_svd_rank_deficient_right_vectors_orthogonal():
    """k >= 24 path (QR with column pivoting + Jacobi): Vr orthogonal also when R is
    rank-deficient (the null-space columns are completed)."""
    from paper_2306_15049_b200 import rsk
    rng = np.random.default_rng(9)
    k = 30
    B = rng.standard_normal((k, 20)) @ rng.standard_normal((20, k))    # rank 20
    U, s, Vt = rsk.svd_small(B)
    V = Vt   # rsk_svd_small returns Vr (columns = right singular vectors)
    assert np.max(np.abs(V.T @ V - np.eye(k))) <= 1e-12
    assert np.max(np.abs(U[:, :20] * s[:20] @ V[:, :20].T - B)) <= 1e-12 * np.max(np.abs(B))
