"""Thin Python binding of librsk (argument marshalling only).

Every method is one C-ABI call of include/rsk.h with the same name (minus the
`rsk_` prefix). Device memory is torch tensors (fp64, CUDA); a block of k images
("N x k column-major, ld = N" in the C ABI) is a contiguous torch tensor of
shape (k, N). No arithmetic on the data happens here.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L


class RskError(RuntimeError):
    """A librsk call returned an error status (`status`: the rsk_status value, or None)."""

    def __init__(self, msg, status=None):
        super().__init__(msg)
        self.status = status


def _dptr(t):
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == torch.float64 and (t.is_contiguous() or (t.dim() == 2 and t.stride(-1) == 1))):
        raise RskError("librsk needs CUDA float64 tensors with unit-stride rows")
    return t.data_ptr()


def _hp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ld(t) -> int:
    """Leading dimension (elements between consecutive vectors): row views of a wider
    batch (e.g. the owned rows of row-slab vectors) keep their parent's stride."""
    if t.dim() > 1:
        if t.stride(-1) != 1:
            raise ValueError("librsk vectors must be unit-stride")
        return t.stride(0) if t.shape[0] > 1 else max(t.stride(0), t.shape[-1])
    return t.numel()


def _nv(t) -> int:
    return t.shape[0] if t.dim() > 1 else 1


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Handle:
    """One librsk handle: a device, an ny x nx image grid and a PSF."""

    def __init__(self, ny: int, nx: int, psf: np.ndarray, device: int = 0):
        self.lib = L.load()
        self.ny, self.nx, self.N = int(ny), int(nx), int(ny) * int(nx)
        self.device = device
        psf = np.ascontiguousarray(psf, dtype=np.float64)
        h = C.c_void_p()
        st = self.lib.rsk_create(C.byref(h), device, self.ny, self.nx, _hp(psf), psf.shape[0],
                                 psf.shape[1], 0)
        if st != L.RSK_OK:
            raise RskError(f"rsk_create failed with status {st}")
        self.h = h
        self._psf = psf
        self.ndata = self.N

    @classmethod
    def slab(cls, ny_global: int, nx: int, row0: int, nrows: int, psf: np.ndarray, halo: int,
             device: int = 0) -> "Handle":
        """The handle of one row slab (rsk_create_slab): global rows [ext0, ext1) stored,
        [row0, row0 + nrows) owned; self.slab_info = (ny_global, ext0, ext1, row0, row1, halo)."""
        self = cls.__new__(cls)
        self.lib = L.load()
        psf = np.ascontiguousarray(psf, dtype=np.float64)
        h = C.c_void_p()
        st = self.lib.rsk_create_slab(C.byref(h), device, int(ny_global), int(nx), int(row0), int(nrows), _hp(psf),
                                      psf.shape[0], psf.shape[1], int(halo), 0)
        if st != L.RSK_OK:
            raise RskError(f"rsk_create_slab failed with status {st}")
        self.h = h
        self._psf = psf
        info = (C.c_int64 * 6)()
        self.lib.rsk_slab_info(h, info)
        self.slab_info = tuple(int(v) for v in info)
        self.ny, self.nx = self.slab_info[2] - self.slab_info[1], int(nx)
        self.N = self.ny * self.nx
        self.ndata = self.N
        self.device = device
        return self

    @classmethod
    def ct(cls, n: int, angles_deg, ndet: int, device: int = 0) -> "Handle":
        """A handle whose C is the parallel-beam CT matrix (rsk_create_ct; Example 2)."""
        self = cls.__new__(cls)
        self.lib = L.load()
        self.ny = self.nx = int(n)
        self.N = self.ny * self.nx
        self.device = device
        ang = np.ascontiguousarray(angles_deg, dtype=np.float64)
        h = C.c_void_p()
        st = self.lib.rsk_create_ct(C.byref(h), device, self.nx, len(ang), _hp(ang), int(ndet), 0)
        if st != L.RSK_OK:
            raise RskError(f"rsk_create_ct failed with status {st}")
        self.h = h
        self._psf = None
        nd, nnz, fro = C.c_int64(), C.c_int64(), C.c_double()
        self.lib.rsk_ct_info(h, C.byref(nd), C.byref(nnz), C.byref(fro))
        self.ndata, self.nnz, self.fro_unscaled = int(nd.value), int(nnz.value), float(fro.value)
        return self

    def close(self):
        if getattr(self, "h", None):
            self.lib.rsk_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, name, allow=(L.RSK_OK,)):
        if st not in allow:
            msg = self.lib.rsk_last_error(self.h)
            raise RskError(f"{name} failed ({st}): {msg.decode() if msg else ''}", st)
        return st

    # ------------------------------------------------------------------ weights
    def set_weights(self, wx, wy, stream=None):
        self._check(self.lib.rsk_set_weights(self.h, _dptr(wx), _dptr(wy), _stream(stream)),
                    "rsk_set_weights")

    # ------------------------------------------------------------ hot-path calls
    def apply_shifted(self, X, Y, gamma=None, EY=None, xdoty=None, mode=L.RSK_APPLY_SHIFTED,
                      stream=None, nvec=None):
        nv = nvec if nvec is not None else _nv(X)
        st = self.lib.rsk_apply_shifted(self.h, nv, _dptr(X), _ld(X), _dptr(gamma), _dptr(Y), _ld(Y),
                                        _dptr(EY), _ld(EY) if EY is not None else self.N,
                                        _dptr(xdoty), mode, _stream(stream))
        self._check(st, "rsk_apply_shifted")

    def apply_shifted_rows(self, X, Y, row0, row1, gamma=None, EY=None, xdoty=None, mode=L.RSK_APPLY_SHIFTED,
                           stream=None, nvec=None):
        """rsk_apply_shifted on the output rows [row0, row1) only. Returns False (nothing
        enqueued) where the library has no row-range path (RSK_EUNSUPPORTED)."""
        nv = nvec if nvec is not None else _nv(X)
        st = self.lib.rsk_apply_shifted_rows(self.h, nv, _dptr(X), _ld(X), _dptr(gamma), _dptr(Y), _ld(Y),
                                             _dptr(EY), _ld(EY) if EY is not None else self.N,
                                             _dptr(xdoty), mode, int(row0), int(row1), _stream(stream))
        if st == L.RSK_EUNSUPPORTED:
            return False
        self._check(st, "rsk_apply_shifted_rows")
        return True

    def recycle_project(self, op, U, V, Cm, k=None, nv=None, stream=None):
        """op = RSK_PROJ_UTV (Cm = U^T V), RSK_ADD_UC (V += U Cm), RSK_SUB_UC (V -= U Cm).
        U: (k, n) tensor, V: (nv, n), Cm: (nv, k) tensor (= column-major k x nv)."""
        k = k if k is not None else _nv(U)
        nv = nv if nv is not None else _nv(V)
        n = U.shape[-1]
        st = self.lib.rsk_recycle_project(self.h, op, n, k, _dptr(U), _ld(U), nv, _dptr(V), _ld(V),
                                          _dptr(Cm), k if Cm.dim() == 1 else Cm.shape[-1],
                                          _stream(stream))
        self._check(st, "rsk_recycle_project")

    def irn_weights(self, x, tau, wx=None, wy=None, eta2=None, stream=None):
        st = self.lib.rsk_irn_weights(self.h, _dptr(x), float(tau), _dptr(wx), _dptr(wy), _dptr(eta2),
                                      _stream(stream))
        self._check(st, "rsk_irn_weights")

    def irn_weights_iso(self, x, tau, wx=None, wy=None, eta2=None, stream=None):
        st = self.lib.rsk_irn_weights_iso(self.h, _dptr(x), float(tau), _dptr(wx), _dptr(wy), _dptr(eta2),
                                          _stream(stream))
        self._check(st, "rsk_irn_weights_iso")

    def gazzola_weights(self, x, p, dx, dy, wx, wy, stream=None):
        st = self.lib.rsk_gazzola_weights(self.h, _dptr(x), float(p), _dptr(dx), _dptr(dy), _dptr(wx),
                                          _dptr(wy), _stream(stream))
        self._check(st, "rsk_gazzola_weights")

    def gazzola_max(self, x, dx, dy, m, stream=None):
        st = self.lib.rsk_gazzola_max(self.h, _dptr(x), _dptr(dx), _dptr(dy), _dptr(m), _stream(stream))
        self._check(st, "rsk_gazzola_max")

    def gazzola_update(self, x, p, m, dx, dy, wx, wy, stream=None):
        st = self.lib.rsk_gazzola_update(self.h, _dptr(x), float(p), _dptr(m), _dptr(dx), _dptr(dy),
                                         _dptr(wx), _dptr(wy), _stream(stream))
        self._check(st, "rsk_gazzola_update")

    def cg_workspace_bytes(self, nshift, flags=0) -> int:
        return int(self.lib.rsk_cg_workspace_bytes(self.h, nshift, flags))

    def cg_recycled_batch(self, desc: L.CgDesc, out: L.CgOut, ws, stream=None) -> int:
        st = self.lib.rsk_cg_recycled_batch(self.h, C.byref(desc), C.byref(out), _dptr(ws) if ws.dtype == torch.float64 else ws.data_ptr(),
                                            ws.numel() * ws.element_size(), _stream(stream))
        return self._check(st, "rsk_cg_recycled_batch", allow=(L.RSK_OK, L.RSK_EPARTIAL))

    def minres_workspace_bytes(self, nshift, max_local_dim) -> int:
        return int(self.lib.rsk_minres_workspace_bytes(self.h, nshift, max_local_dim))

    def minres_recycled_batch(self, desc: L.CgDesc, out: L.CgOut, ws, stream=None) -> int:
        st = self.lib.rsk_minres_recycled_batch(self.h, C.byref(desc), C.byref(out), ws.data_ptr(),
                                                ws.numel() * ws.element_size(), _stream(stream))
        return self._check(st, "rsk_minres_recycled_batch", allow=(L.RSK_OK, L.RSK_EPARTIAL))

    # ------------------------------------------------------------ support calls
    def make_rhs(self, x_true, xi, nu, d, b, stream=None):
        self._check(self.lib.rsk_make_rhs(self.h, _dptr(x_true), _dptr(xi), float(nu), _dptr(d), _dptr(b),
                                          _stream(stream)), "rsk_make_rhs")

    def batch_dot(self, X, Y, out, stream=None):
        n = X.shape[-1]
        self._check(self.lib.rsk_batch_dot(self.h, n, _nv(X), _dptr(X), _ld(X), _dptr(Y), _ld(Y), _dptr(out),
                                           _stream(stream)), "rsk_batch_dot")

    def batch_axpby(self, a: np.ndarray, X, b: np.ndarray | None, Y, stream=None):
        a = np.ascontiguousarray(a, dtype=np.float64)
        bb = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        n = Y.shape[-1]
        self._check(self.lib.rsk_batch_axpby(self.h, n, _nv(Y), _hp(a), _dptr(X), _ld(X) if X is not None else n,
                                             _hp(bb) if bb is not None else None, _dptr(Y), _ld(Y),
                                             _stream(stream)), "rsk_batch_axpby")

    def qr_tall(self, V, Q, stream=None) -> np.ndarray:
        k, n = V.shape
        R = np.zeros((k, k), order="F")
        self._check(self.lib.rsk_qr_tall(self.h, n, k, _dptr(V), n, _dptr(Q), n, _hp(R), _stream(stream)),
                    "rsk_qr_tall")
        return R

    def lcurve_norms(self, X, d, rho, eta2, scratch, stream=None):
        self._check(self.lib.rsk_lcurve_norms(self.h, _nv(X), _dptr(X), _ld(X), _dptr(d), _dptr(rho), _dptr(eta2),
                                              _dptr(scratch), _stream(stream)), "rsk_lcurve_norms")

    def seminorm_rows(self, X, row0, row1, eta2, stream=None):
        self._check(self.lib.rsk_seminorm_rows(self.h, _nv(X), _dptr(X), _ld(X), int(row0), int(row1), _dptr(eta2),
                                               _stream(stream)), "rsk_seminorm_rows")

    def get_counters(self, reset=False):
        a, e, c = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.rsk_get_counters(self.h, C.byref(a), C.byref(e), C.byref(c), int(reset)),
                    "rsk_get_counters")
        return a.value, e.value, c.value


# -------------------------------------------------------------- host helpers
def _f(a):
    return np.asfortranarray(a, dtype=np.float64)


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def orth_guess(R, KtZE, ZEtZE, ZEtb, Ktb, gamma_star, gammas):
    """eq:orthupdate per shift (host C++). Returns (C (nc x m, Fortran order), status[m])."""
    lib = L.load()
    nc = R.shape[0]
    m = len(gammas)
    R, KtZE, ZEtZE = _f(R), _f(KtZE), _f(ZEtZE)
    ZEtb = np.ascontiguousarray(ZEtb, dtype=np.float64).ravel()
    Ktb = np.ascontiguousarray(Ktb, dtype=np.float64).ravel()
    g = np.ascontiguousarray(gammas, dtype=np.float64)
    Cm = np.zeros((nc, m), order="F")
    stt = np.zeros(m, dtype=np.int32)
    st = lib.rsk_orth_guess(nc, _hp(R), _hp(KtZE), _hp(ZEtZE), _hp(ZEtb), _hp(Ktb), float(gamma_star), m,
                            _hp(g), _hp(Cm), _ip(stt))
    if st != L.RSK_OK:
        raise RskError(f"rsk_orth_guess failed ({st})")
    return Cm, stt


def oblique_guess(R, KtZE, Ktb, gamma_anchor, gammas):
    """eq:obliqueupdate per shift (host C++). Returns (C (nc x m, Fortran order), status[m])."""
    lib = L.load()
    nc = R.shape[0]
    m = len(gammas)
    R, KtZE = _f(R), _f(KtZE)
    Ktb = np.ascontiguousarray(Ktb, dtype=np.float64).ravel()
    g = np.ascontiguousarray(gammas, dtype=np.float64)
    Cm = np.zeros((nc, m), order="F")
    stt = np.zeros(m, dtype=np.int32)
    st = lib.rsk_oblique_guess(nc, _hp(R), _hp(KtZE), _hp(Ktb), float(gamma_anchor), m, _hp(g), _hp(Cm),
                               _ip(stt))
    if st != L.RSK_OK:
        raise RskError(f"rsk_oblique_guess failed ({st})")
    return Cm, stt


def pencil_ritz(Ahat, Ehat, gamma, J):
    lib = L.load()
    nc = Ahat.shape[0]
    Wt = np.zeros((nc, J), order="F"); th = np.zeros(J)
    if lib.rsk_pencil_ritz(nc, _hp(_f(Ahat)), _hp(_f(Ehat)), float(gamma), J, _hp(Wt), _hp(th)) != L.RSK_OK:
        raise RskError("rsk_pencil_ritz failed")
    return Wt, th


def stabilize_small(R, colnorm2, condcap, cap):
    lib = L.load()
    k = R.shape[0]
    Zs = np.zeros((k, k), order="F"); nk = C.c_int()
    cn = np.ascontiguousarray(colnorm2, dtype=np.float64)
    if lib.rsk_stabilize_small(k, _hp(_f(R)), _hp(cn), float(condcap), int(cap), _hp(Zs),
                               C.byref(nk)) != L.RSK_OK:
        raise RskError("rsk_stabilize_small failed")
    return np.asfortranarray(Zs[:, :nk.value]), nk.value


def carried_select(g2, gh2, thr):
    lib = L.load()
    m = len(g2)
    g2 = np.ascontiguousarray(g2, dtype=np.float64); gh2 = np.ascontiguousarray(gh2, dtype=np.float64)
    sc = np.zeros(m); keep = np.zeros(m, dtype=np.int32)
    if lib.rsk_carried_select(m, _hp(g2), _hp(gh2), float(thr), _hp(sc), _ip(keep)) != L.RSK_OK:
        raise RskError("rsk_carried_select failed")
    return sc, keep


def sym_eig(H):
    lib = L.load()
    n = H.shape[0]
    H = np.asfortranarray(H, dtype=np.float64)
    th = np.zeros(n); V = np.zeros((n, n), order="F")
    if lib.rsk_sym_eig(n, _hp(H), _hp(th), _hp(V)) != L.RSK_OK:
        raise RskError("rsk_sym_eig failed")
    return th, V


def svd_small(R):
    lib = L.load()
    k = R.shape[0]
    R = np.asfortranarray(R, dtype=np.float64)
    U = np.zeros((k, k), order="F"); s = np.zeros(k); V = np.zeros((k, k), order="F")
    if lib.rsk_svd_small(k, _hp(R), _hp(U), _hp(s), _hp(V)) != L.RSK_OK:
        raise RskError("rsk_svd_small failed")
    return U, s, V


def chol_solve_small(G, Z):
    lib = L.load()
    n = G.shape[0]
    G = np.asfortranarray(G, dtype=np.float64)
    Z = np.asfortranarray(Z.reshape(n, -1), dtype=np.float64)
    X = np.zeros_like(Z, order="F")
    st = lib.rsk_chol_solve_small(n, _hp(G), Z.shape[1], _hp(Z), _hp(X))
    if st != L.RSK_OK:
        return None
    return X


def lcurve_corner(rho, eta):
    lib = L.load()
    rho = np.ascontiguousarray(rho, dtype=np.float64); eta = np.ascontiguousarray(eta, dtype=np.float64)
    M = len(rho)
    ls = C.c_int(); kap = np.zeros(M)
    if lib.rsk_lcurve_corner(M, _hp(rho), _hp(eta), C.byref(ls), _hp(kap)) != L.RSK_OK:
        raise RskError("rsk_lcurve_corner failed")
    return ls.value, kap
