"""Row-slab domain decomposition of the hot path (configs[4] = C5,
4096^2 pixels, split over 2/4/8 GPUs).

Rows [0, ny) are cut into contiguous slabs, one per rank. A slab stores its owned rows
plus up to H = 2r halo rows on each side (the band of A = C^T C; clipped at the image
edges) as an ordinary librsk image of ext_rows x nx. With the halo rows filled from the
neighbours, the fused apply of the extended slab is exact on every owned row: the
zero-boundary truncation of B = G^T G only acts within r rows of the extended array's
edge (apply_core.cuh), i.e. inside the halo, and the E_k stencil needs one halo row.

Per CG iteration a rank exchanges the halo of p (one send/recv pair per neighbour), and
all-reduces two small vectors: p.w (nshift doubles) and [r.r, (AW)^T r, (EW)^T r]
(nshift (2J+1) doubles). Every vector operation is a librsk call on the rank's own rows
(a contiguous column range of each extended row-major vector); the scalar steps are the
librsk host helpers rsk_cg_alpha / rsk_cg_scalars / rsk_gram_solve /
rsk_local_gram_factors. The recurrences are the oracle's O4 (oracle/defcg.py). Sums are
all-reduced, so results match one domain within rounding, not bitwise.

Communication is pluggable: DistComm (torch.distributed: NCCL on GPUs, gloo on CPU
tensors) or ThreadComm (ranks emulated as host threads on one GPU for tests; no kernel
ever waits on another rank's kernel, the host moves the halo rows between launches).
"""
from __future__ import annotations

import dataclasses
import threading

import numpy as np
import torch

from . import _lib as L
from .rsk import Handle, RskError

LOOP_ACTIVE, LOOP_RCONV, LOOP_DONE, LOOP_BREAKDOWN, LOOP_MAXIT = range(5)


@dataclasses.dataclass
class Slab:
    rank: int
    row0: int        # first owned row (global)
    row1: int        # one past the last owned row
    ext0: int        # first stored row (global)
    ext1: int
    top: int         # halo rows above the owned rows (0 on the first slab)
    bot: int         # halo rows below (0 on the last slab)

    @property
    def own_rows(self) -> int:
        return self.row1 - self.row0

    @property
    def ext_rows(self) -> int:
        return self.ext1 - self.ext0


class SlabPlan:
    """Contiguous row slabs with H = 2r halo rows (clipped at the image edges)."""

    def __init__(self, ny: int, nx: int, r: int, nranks: int):
        self.ny, self.nx, self.r, self.nranks = ny, nx, r, nranks
        self.H = 2 * r
        base, rem = divmod(ny, nranks)
        self.slabs = []
        r0 = 0
        for k in range(nranks):
            cnt = base + (1 if k < rem else 0)
            if cnt < self.H:
                raise ValueError(f"slab {k} has {cnt} rows < halo {self.H}")
            r1 = r0 + cnt
            e0, e1 = max(0, r0 - self.H), min(ny, r1 + self.H)
            self.slabs.append(Slab(k, r0, r1, e0, e1, r0 - e0, e1 - r1))
            r0 = r1

    def extend(self, full: torch.Tensor, rank: int) -> torch.Tensor:
        """Rows [ext0, ext1) of full image(s) (..., ny*nx) -> (..., ext_rows*nx), a copy."""
        s, nx = self.slabs[rank], self.nx
        return full[..., s.ext0 * nx:s.ext1 * nx].clone()

    def owned(self, full: torch.Tensor, rank: int) -> torch.Tensor:
        s, nx = self.slabs[rank], self.nx
        return full[..., s.row0 * nx:s.row1 * nx]


# ------------------------------------------------------------------ communication
class DistComm:
    """Halo exchange + all-reduce over torch.distributed (one rank per process)."""

    def __init__(self, plan: SlabPlan, rank: int):
        self.plan, self.rank = plan, rank

    def allreduce(self, t: torch.Tensor):
        import torch.distributed as dist
        dist.all_reduce(t)

    def halo(self, T: torch.Tensor):
        """T: (nv, ext_rows*nx). Fill the halo rows from the neighbours' owned rows."""
        import torch.distributed as dist
        p, k, nx = self.plan, self.rank, self.plan.nx
        s = p.slabs[k]
        off = s.top
        ops, recv = [], []
        if k > 0:
            up = p.slabs[k - 1]
            send = T[:, off * nx:(off + up.bot) * nx].contiguous()
            buf = torch.empty(T.shape[0], s.top * nx, dtype=T.dtype, device=T.device)
            ops += [dist.P2POp(dist.isend, send, k - 1), dist.P2POp(dist.irecv, buf, k - 1)]
            recv.append((buf, 0))
        if k < p.nranks - 1:
            dn = p.slabs[k + 1]
            send = T[:, (off + s.own_rows - dn.top) * nx:(off + s.own_rows) * nx].contiguous()
            buf = torch.empty(T.shape[0], s.bot * nx, dtype=T.dtype, device=T.device)
            ops += [dist.P2POp(dist.isend, send, k + 1), dist.P2POp(dist.irecv, buf, k + 1)]
            recv.append((buf, (off + s.own_rows) * nx))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for buf, at in recv:
            T[:, at:at + buf.shape[1]].copy_(buf)


class ThreadGroup:
    """Shared state of ranks emulated as host threads in one process."""

    def __init__(self, plan: SlabPlan):
        self.plan = plan
        self.bar = threading.Barrier(plan.nranks)
        self.buf = [None] * plan.nranks

    def comm(self, rank: int) -> "ThreadComm":
        return ThreadComm(self, rank)


class ThreadComm:
    def __init__(self, group: ThreadGroup, rank: int):
        self.g, self.rank, self.plan = group, rank, group.plan

    def _sync(self, t):
        if t.is_cuda:
            torch.cuda.synchronize(t.device)

    def allreduce(self, t: torch.Tensor):
        g = self.g
        self._sync(t)
        g.buf[self.rank] = t.clone()
        g.bar.wait()
        tot = g.buf[0].clone()
        for k in range(1, self.plan.nranks):     # fixed rank order
            tot += g.buf[k]
        self._sync(tot)
        g.bar.wait()
        t.copy_(tot)
        self._sync(t)

    def halo(self, T: torch.Tensor):
        g, p, k, nx = self.g, self.plan, self.rank, self.plan.nx
        s = p.slabs[k]
        self._sync(T)
        g.buf[k] = T
        g.bar.wait()
        if k > 0:
            up = p.slabs[k - 1]
            src = g.buf[k - 1]
            a = (up.top + up.own_rows - s.top) * nx
            T[:, :s.top * nx].copy_(src[:, a:a + s.top * nx])
        if k < p.nranks - 1:
            dn = p.slabs[k + 1]
            src = g.buf[k + 1]
            T[:, (s.top + s.own_rows) * nx:].copy_(src[:, dn.top * nx:(dn.top + s.bot) * nx])
        self._sync(T)
        g.bar.wait()


def run_threads(plan: SlabPlan, fn):
    """Run fn(rank, comm) for every rank of the plan on host threads; returns the results."""
    group = ThreadGroup(plan)
    out = [None] * plan.nranks
    err = []

    def body(k):
        try:
            out[k] = fn(k, group.comm(k))
        except BaseException as e:   # noqa: BLE001 (re-raised below)
            err.append(e)
            group.bar.abort()

    th = [threading.Thread(target=body, args=(k,)) for k in range(plan.nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out


# ------------------------------------------------------------------ per-rank operators
def _ptr(a):
    return a.ctypes.data_as(L.C.POINTER(L.C.c_double))


def _iptr(a):
    return a.ctypes.data_as(L.C.POINTER(L.C.c_int))


class SlabOps:
    """The rank's slab as a librsk image of ext_rows x nx; owned rows are a contiguous
    column range [own0, own0 + own_n) of every extended vector."""

    def __init__(self, plan: SlabPlan, rank: int, comm, psf: np.ndarray, device: int = 0):
        self.plan, self.rank, self.comm = plan, rank, comm
        self.s = plan.slabs[rank]
        self.nx = plan.nx
        self.ext_n = self.s.ext_rows * plan.nx
        self.own0 = self.s.top * plan.nx
        self.own_n = self.s.own_rows * plan.nx
        self.dev = torch.device("cuda", device)
        self.h = Handle(self.s.ext_rows, plan.nx, psf, device)
        self.lib = L.load()
        self.f = dict(dtype=torch.float64, device=self.dev)

    def own(self, T: torch.Tensor) -> torch.Tensor:
        """Owned rows of an extended vector (batch); owned-only vectors pass through."""
        if T.shape[-1] == self.own_n and self.own_n != self.ext_n:
            return T
        if T.shape[-1] != self.ext_n:
            raise ValueError(f"vector length {T.shape[-1]} is neither {self.ext_n} nor {self.own_n}")
        return T[..., self.own0:self.own0 + self.own_n]

    def set_weights(self, wx_full: torch.Tensor, wy_full: torch.Tensor):
        """Weights of the stored rows, cut from the global planes (wy of the last global
        row stays the zero pad; on interior slabs the halo rows carry true weights)."""
        self.h.set_weights(self.plan.extend(wx_full, self.rank).contiguous(),
                           self.plan.extend(wy_full, self.rank).contiguous())

    def apply(self, X: torch.Tensor, Y: torch.Tensor, gamma: torch.Tensor | None = None,
              mode=L.RSK_APPLY_SHIFTED, EY: torch.Tensor | None = None):
        """Y = A_gamma X on the owned rows (X: extended vectors, halo refreshed here)."""
        self.comm.halo(X)
        self.h.apply_shifted(X, Y, gamma=gamma, EY=EY, mode=mode)

    def dot(self, X, Y) -> torch.Tensor:
        """Per-vector X.Y over the whole image (owned-row partials, all-reduced)."""
        out = torch.empty(X.shape[0], **self.f)
        self.h.batch_dot(self.own(X), self.own(Y), out)
        self.comm.allreduce(out)
        return out

    def utv(self, U, V) -> torch.Tensor:
        """U^T V over the whole image: U (k, ext or own), V (nv, ...) -> (nv, k)."""
        k, nv = U.shape[0], V.shape[0]
        Cm = torch.empty(nv, k, **self.f)
        Uo, Vo = self.own(U), self.own(V)
        self.h.recycle_project(L.RSK_PROJ_UTV, Uo, Vo, Cm)
        self.comm.allreduce(Cm)
        return Cm

    def axpby(self, a: np.ndarray, X, b: np.ndarray | None, Y):
        """Y_s = a_s X_s + b_s Y_s on the owned rows (host coefficient arrays)."""
        Xo = None if X is None else self.own(X)
        Yo = self.own(Y)
        self.h.batch_axpby(np.ascontiguousarray(a, dtype=np.float64), Xo,
                           None if b is None else np.ascontiguousarray(b, dtype=np.float64), Yo)

    def irn_weights(self, x: torch.Tensor, tau: float, adopt: bool = True):
        """IRN weights of x (extended, halo refreshed here) for every stored row: owned rows
        and halo rows get the global values (each needs x one row below, present in the
        halo); only the last stored row of an interior slab is wrong (no row below) and no
        owned output reads it. adopt: make them the handle's W_k."""
        self.comm.halo(x[None] if x.dim() == 1 else x)
        wx = torch.empty(self.ext_n, **self.f)
        wy = torch.empty(self.ext_n, **self.f)
        self.h.irn_weights(x, tau, wx, wy)
        if adopt:
            self.h.set_weights(wx, wy)
        return wx, wy

    def seminorm2(self, X: torch.Tensor) -> torch.Tensor:
        """sum wx (Dx x)^2 + wy (Dy x)^2 over the whole image (L-curve eta^2) of each
        extended vector: owned-row partials (halo refreshed for Dy), all-reduced."""
        self.comm.halo(X)
        out = torch.empty(X.shape[0], **self.f)
        self.h.seminorm_rows(X, self.s.top, self.s.top + self.s.own_rows, out)
        self.comm.allreduce(out)
        return out

    def resnorm2(self, X: torch.Tensor, d: torch.Tensor) -> torch.Tensor:
        """||C x - d||^2 over the whole image (L-curve rho^2) of each extended vector."""
        Y = torch.empty_like(X)
        self.apply(X, Y, mode=L.RSK_APPLY_C_ONLY)
        D = self.own(d).expand(X.shape[0], -1).contiguous()
        self.axpby(np.full(X.shape[0], -1.0), D, np.ones(X.shape[0]), Y)
        return self.dot(Y, Y)

    def add_uc(self, op, U, V, Cm):
        """V (+/-)= U Cm on the owned rows (U owned rows, V extended or owned)."""
        self.h.recycle_project(op, self.own(U), self.own(V), Cm)


# ------------------------------------------------------------------ batched deflated CG
def _h(t: torch.Tensor) -> np.ndarray:
    return np.ascontiguousarray(t.detach().cpu().numpy(), dtype=np.float64)


def slab_cg(ops: SlabOps, gamma: np.ndarray, b: torch.Tensor, X: torch.Tensor,
            W=None, AW=None, EW=None, tol: float = 1e-8, maxit: int = 20000):
    """Deflated CG (O4) for nshift shifted systems on the rank's slab.
    b: (ext_n,) right-hand side (owned rows used); X: (nshift, ext_n) in x_p, out x.
    W, AW, EW: (J, own_n) owned rows of the deflation block (or None: plain CG).
    Returns dict(iters, applies, relres_true, status) (host arrays, identical on all ranks)."""
    lib = ops.lib
    f = ops.f
    S = len(gamma)
    gam = np.ascontiguousarray(gamma, dtype=np.float64)
    gam_d = torch.from_numpy(gam).to(ops.dev)
    J = 0 if W is None else W.shape[0]
    KM = L.RSK_MAX_LOCAL
    ones, zeros = np.ones(S), np.zeros(S)
    Bv = torch.empty(S, ops.own_n, **f)
    Bv.copy_(ops.own(b).expand(S, -1))
    nb = float(np.sqrt(_h(ops.dot(b[None], b[None]))[0]))
    if nb == 0.0:
        X.zero_()
        return dict(iters=np.zeros(S, np.int32), applies=np.zeros(S, np.int64), relres_true=np.zeros(S),
                    status=np.full(S, LOOP_DONE, np.int32))
    thr = tol * nb
    # ---- local Gram factors G_s = W^T (A + gamma_s E) W
    Lf = np.zeros(S * KM * KM)
    m = np.zeros(S, np.int32)
    hasg = np.zeros(S, np.int32)
    dropped = np.zeros(S, np.int32)
    if J:
        WA = np.zeros(256); WE = np.zeros(256)
        WA[:J * J] = _h(ops.utv(W, AW)).ravel()      # (J x J): row a = AW_a^T W -> column-major W^T AW
        WE[:J * J] = _h(ops.utv(W, EW)).ravel()
        Jh = np.array([J], np.int32)
        gos = np.zeros(S, np.int32)
        st = lib.rsk_local_gram_factors(S, 1, _iptr(Jh), _iptr(gos), _ptr(gam), _ptr(WA), _ptr(WE), None, None,
                                        None, None, _ptr(Lf), _iptr(m), _iptr(hasg), _iptr(dropped))
        if st != L.RSK_OK:
            raise RskError(f"rsk_local_gram_factors failed ({st})")

    def gram_solve(zA, zE):
        mu = np.zeros(S * KM)
        st2 = lib.rsk_gram_solve(S, J, _ptr(Lf), _iptr(m), _iptr(hasg), _ptr(gam), _ptr(zA),
                                 None if zE is None else _ptr(zE), None, _ptr(mu))
        if st2 != L.RSK_OK:
            raise RskError(f"rsk_gram_solve failed ({st2})")
        return mu.reshape(S, KM)

    def zcols(R):
        """(AW)^T r and (EW)^T r, J x S column-major (ld J)."""
        return (np.ascontiguousarray(_h(ops.utv(AW, R)).ravel()),
                np.ascontiguousarray(_h(ops.utv(EW, R)).ravel()))

    R = torch.empty(S, ops.own_n, **f)
    P = torch.zeros(S, ops.ext_n, **f)
    Wv = torch.empty(S, ops.ext_n, **f)
    applies = np.zeros(S, np.int64)
    # ---- r_p = b - A_gamma x_p (one fresh apply, G15)
    ops.apply(X, Wv, gam_d)
    applies += 1
    R.copy_(Bv)
    ops.axpby(-ones, Wv, ones, R)
    # ---- Galerkin start on Range(W): c = G^-1 W^T r_p; x += W c; r -= (AW + gamma EW) c
    if J:
        zW = np.ascontiguousarray(_h(ops.utv(W, R)).ravel())
        c = gram_solve(zW, None)
        Cm = torch.from_numpy(np.ascontiguousarray(c[:, :J])).to(ops.dev)
        ops.add_uc(L.RSK_ADD_UC, W, X, Cm)
        ops.add_uc(L.RSK_SUB_UC, AW, R, Cm)
        T = torch.zeros(S, ops.own_n, **f)
        ops.add_uc(L.RSK_ADD_UC, EW, T, Cm)
        ops.axpby(-gam, T, ones, R)
    rho = _h(ops.dot(R, R))
    state = np.where(np.sqrt(rho) <= thr, LOOP_RCONV, LOOP_ACTIVE).astype(np.int32)
    iters = np.zeros(S, np.int32)
    nconf = np.zeros(S, np.int32)
    rho_true = np.zeros(S)
    beta = np.zeros(S)
    alpha = np.zeros(S)

    def new_p(mask, mu):
        """p = r + beta p - W mu_W for the masked shifts."""
        a = np.where(mask, 1.0, 0.0)
        bb = np.where(mask, beta, 1.0)
        ops.axpby(a, R, bb, P)
        if J:
            Cm2 = torch.from_numpy(np.ascontiguousarray(np.where(mask[:, None], mu[:, :J], 0.0))).to(ops.dev)
            ops.add_uc(L.RSK_SUB_UC, W, P, Cm2)

    # p_0 = r_0 - W mu_0
    mu0 = gram_solve(*zcols(R)) if J else np.zeros((S, KM))
    new_p(state == LOOP_ACTIVE, mu0)
    guard = 0
    while np.any((state == LOOP_ACTIVE) | (state == LOOP_RCONV)):
        guard += 1
        if guard > 4 * maxit + 100:
            raise RskError("slab_cg: loop guard")
        mode = state.copy()
        act = mode == LOOP_ACTIVE
        conf = mode == LOOP_RCONV
        if act.any():
            ops.apply(P, Wv, gam_d)
            pw = _h(ops.dot(P, Wv))
            st = lib.rsk_cg_alpha(S, _ptr(rho), _ptr(pw), _ptr(alpha), _iptr(state))
            if st != L.RSK_OK:
                raise RskError(f"rsk_cg_alpha failed ({st})")
            ok = act & (state == LOOP_ACTIVE)
            a = np.where(ok, alpha, 0.0)
            ops.axpby(a, P, ones, X)                      # x += alpha p
            ops.axpby(-a, Wv, ones, R)                    # r -= alpha w
            applies += act
        if conf.any():                                    # true residual r = b - A_gamma x
            Wx = torch.empty(S, ops.ext_n, **f)
            ops.apply(X, Wx, gam_d)
            ops.axpby(np.where(conf, -1.0, 0.0), Wx, np.where(conf, 0.0, 1.0), R)
            ops.axpby(np.where(conf, 1.0, 0.0), Bv, ones, R)
            applies += conf
        rho_new = _h(ops.dot(R, R))
        zA, zE = zcols(R) if J else (np.zeros(1), np.zeros(1))
        mu = np.zeros(S * KM)
        st = lib.rsk_cg_scalars(S, J, _iptr(mode), _ptr(gam), _ptr(rho_new), _ptr(zA), _ptr(zE), None,
                                _iptr(m), _iptr(hasg), _ptr(Lf), float(thr), int(maxit), _ptr(rho), _ptr(beta),
                                _ptr(mu), _iptr(iters), _ptr(rho_true), _iptr(nconf), _iptr(state))
        if st != L.RSK_OK:
            raise RskError(f"rsk_cg_scalars failed ({st})")
        new_p(state == LOOP_ACTIVE, mu.reshape(S, KM))
    # final true residual for shifts that stopped without a confirmation
    unconf = state != LOOP_DONE
    if unconf.any():
        Wx = torch.empty(S, ops.ext_n, **f)
        ops.apply(X, Wx, gam_d)
        Rt = Bv.clone()
        ops.axpby(-ones, Wx, ones, Rt)
        rt = _h(ops.dot(Rt, Rt))
        rho_true = np.where(unconf, rt, rho_true)
        applies += unconf
    return dict(iters=iters, applies=applies, relres_true=np.sqrt(np.maximum(rho_true, 0.0)) / nb,
                status=state, m_used=m, dropped=dropped)
