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
import os
import threading

import numpy as np
import torch

from . import _lib as L
from .indices import shift_indices
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

    def _host(self) -> bool:
        # gloo (several ranks on one device, CPU tests) moves CUDA tensors through host memory
        import torch.distributed as dist
        return dist.get_backend() == "gloo"

    def allreduce(self, t: torch.Tensor, op: str = "sum"):
        import torch.distributed as dist
        rop = dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM
        if self._host() and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, op=rop)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=rop)

    def halo(self, T: torch.Tensor):
        """T: (nv, ext_rows*nx). Fill the halo rows from the neighbours' owned rows."""
        self.halo_finish(self.halo_start(T))

    def halo_start(self, T: torch.Tensor):
        """Post the halo exchange of T (send buffers are copies of the owned boundary rows;
        under NCCL the transfers run on NCCL's stream, concurrently with work the caller
        enqueues next on the current stream). Returns the pending state for halo_finish."""
        import torch.distributed as dist
        p, k, nx = self.plan, self.rank, self.plan.nx
        s = p.slabs[k]
        off = s.top
        ops, recv = [], []
        bdev = torch.device("cpu") if (self._host() and T.is_cuda) else T.device
        if k > 0:
            up = p.slabs[k - 1]
            send = T[:, off * nx:(off + up.bot) * nx].contiguous().to(bdev)
            buf = torch.empty(T.shape[0], s.top * nx, dtype=T.dtype, device=bdev)
            ops += [dist.P2POp(dist.isend, send, k - 1), dist.P2POp(dist.irecv, buf, k - 1)]
            recv.append((buf, 0))
        if k < p.nranks - 1:
            dn = p.slabs[k + 1]
            send = T[:, (off + s.own_rows - dn.top) * nx:(off + s.own_rows) * nx].contiguous().to(bdev)
            buf = torch.empty(T.shape[0], s.bot * nx, dtype=T.dtype, device=bdev)
            ops += [dist.P2POp(dist.isend, send, k + 1), dist.P2POp(dist.irecv, buf, k + 1)]
            recv.append((buf, (off + s.own_rows) * nx))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return T, reqs, recv, ops

    def halo_finish(self, pend):
        """Wait for the posted exchange (the current stream waits under NCCL) and copy the
        received rows into T's halo."""
        T, reqs, recv, _ops = pend
        for req in reqs:
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

    def allreduce(self, t: torch.Tensor, op: str = "sum"):
        g = self.g
        self._sync(t)
        g.buf[self.rank] = t.clone()
        g.bar.wait()
        tot = g.buf[0].clone()
        for k in range(1, self.plan.nranks):     # fixed rank order
            if op == "max":
                torch.maximum(tot, g.buf[k], out=tot)
            else:
                tot += g.buf[k]
        self._sync(tot)
        g.bar.wait()
        t.copy_(tot)
        self._sync(t)

    def halo_start(self, T: torch.Tensor):
        self.halo(T)      # host threads: the exchange completes here
        return None

    def halo_finish(self, pend):
        pass

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
        self.h = Handle.slab(plan.ny, plan.nx, self.s.row0, self.s.own_rows, psf, plan.H, device)
        self.overlap = os.environ.get("RSK_SLAB_OVERLAP", "1") != "0"   # halo / interior overlap
        assert self.h.slab_info[1:3] == (self.s.ext0, self.s.ext1), (self.h.slab_info, self.s)
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
        """Y = A_gamma X on the owned rows (X: extended vectors, halo refreshed here).
        The halo exchange is overlapped with the interior rows: an owned row
        at least H = 2r rows from a neighbour's slab reads only owned rows, so those rows
        are computed (rsk_apply_shifted_rows) while the halo rows are in flight, and the H
        rows next to each neighbour after they arrived. Handles without a row-range path
        (images below the strip core's size) exchange first and apply whole."""
        s, k, H = self.s, self.rank, self.plan.H
        # every range starts on a multiple of 8 rows of the slab image, as the whole-image
        # apply's 8-row output blocks do: the rows come out bit for bit as without overlap
        lo, hi = s.top, s.top + s.own_rows
        i0 = -(-(lo + (H if k > 0 else 0)) // 8) * 8
        i1 = (hi - (H if k < self.plan.nranks - 1 else 0)) // 8 * 8
        if self.overlap and i1 > i0 and mode in (L.RSK_APPLY_SHIFTED, L.RSK_APPLY_SPLIT):
            pend = self.comm.halo_start(X)
            if self.h.apply_shifted_rows(X, Y, i0, i1, gamma=gamma, EY=EY, mode=mode):
                self.comm.halo_finish(pend)
                if i0 > lo:
                    self.h.apply_shifted_rows(X, Y, lo // 8 * 8, i0, gamma=gamma, EY=EY, mode=mode)
                if i1 < hi:
                    self.h.apply_shifted_rows(X, Y, i1, hi, gamma=gamma, EY=EY, mode=mode)
                return
            self.comm.halo_finish(pend)
        else:
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
        if V.dim() == 1:
            V = V[None]
        if U.dim() == 1:
            U = U[None]
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

    def irn_weights_iso(self, x: torch.Tensor, tau: float, adopt: bool = True):
        """isotropic IRN weights, halo semantics as irn_weights"""
        self.comm.halo(x[None] if x.dim() == 1 else x)
        wx = torch.empty(self.ext_n, **self.f)
        wy = torch.empty(self.ext_n, **self.f)
        self.h.irn_weights_iso(x, tau, wx, wy)
        if adopt:
            self.h.set_weights(wx, wy)
        return wx, wy

    def gazzola_weights(self, x: torch.Tensor, p: float, dx, dy, wx, wy):
        """Gazzola's update on the slab: the slab's ||D_k L x||_inf (every row
        it stores is a true row of L except the missing Dy row of its last stored row,
        which is not counted), max-reduced over ranks, then the elementwise update of
        D (dx, dy in/out) and W = D^2 on every stored row (halo rows stay consistent with
        their owners; the last stored row's Dy entry is not, and no owned output reads it)."""
        self.comm.halo(x[None] if x.dim() == 1 else x)
        m = torch.empty(1, **self.f)
        self.h.gazzola_max(x, dx, dy, m)
        self.comm.allreduce(m, op="max")
        self.h.gazzola_update(x, p, m, dx, dy, wx, wy)

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
            W=None, AW=None, EW=None, tol: float = 1e-8, maxit: int = 20000, *, has_xp=None,
            groups=None, ghat=None, store=None, store_cap: int = 100, Gout=None):
    """Deflated CG (O4) for nshift shifted systems on the rank's slab, the slab counterpart of
    rsk_cg_recycled_batch (same recurrences, sums all-reduced).
    b: (ext_n,) right-hand side; X: (nshift, ext_n) in x_p (has_xp) / out x.
    Deflation: groups = dict(W, AW, EW: lists of (J_g, n) blocks, of_shift) -- or one block
    W, AW, EW -- plus optional carried columns ghat = (Gh, ZGh, has_g) ((nshift, n) each).
    store: (nshift * store_cap, n) residual store (seed solves); Gout: g = x - x_p.
    Blocks may be owned-row (n = own_n) or extended tensors. Returns the host arrays of
    rsk_cg_out (identical on all ranks)."""
    lib = ops.lib
    f = ops.f
    S = len(gamma)
    KM = L.RSK_MAX_LOCAL
    gam = np.ascontiguousarray(gamma, dtype=np.float64)
    gam_d = torch.from_numpy(gam).to(ops.dev)
    if groups is None and W is not None:
        groups = dict(W=[W], AW=[AW], EW=[EW], of_shift=np.zeros(S, np.int32))
    G = 0 if groups is None else len(groups["W"])
    gos = np.zeros(S, np.int32) if G == 0 else np.ascontiguousarray(groups["of_shift"], dtype=np.int32)
    Js = [0] * max(G, 1) if G == 0 else [int(w.shape[0]) for w in groups["W"]]
    Jm = max(Js) if G else 0
    Gh = ZGh = None
    has_g = np.zeros(S, np.int32)
    if G and ghat is not None:
        Gh, ZGh, hg0 = ghat
        has_g = np.ascontiguousarray(hg0, dtype=np.int32).copy()
    hx = np.ones(S, np.int32) if has_xp is None else np.ascontiguousarray(has_xp, dtype=np.int32)
    ones, zeros = np.ones(S), np.zeros(S)
    for s_ in range(S):
        if not hx[s_]:
            ops.own(X[s_:s_ + 1]).zero_()
    X0 = ops.own(X).clone() if Gout is not None else None
    Bv = torch.empty(S, ops.own_n, **f)
    Bv.copy_(ops.own(b).expand(S, -1))
    nb = float(np.sqrt(_h(ops.dot(b[None], b[None]))[0]))
    out = dict(iters=np.zeros(S, np.int32), applies=np.zeros(S, np.int64), relres=np.zeros(S),
               status=np.zeros(S, np.int32), m_used=np.zeros(S, np.int32), store_count=np.zeros(S, np.int32),
               prof=np.zeros(8))
    if nb == 0.0:
        ops.own(X).zero_()
        if Gout is not None:
            ops.own(Gout).zero_()
        out["status"][:] = L.RSK_CG_ZERO_RHS
        return out
    thr = tol * nb
    # ---- local Gram factors (rsk_local_gram_factors) from all-reduced pieces
    Lf = np.zeros(S * KM * KM)
    m = np.zeros(S, np.int32)
    hasg = has_g.copy()
    dropped = np.zeros(S, np.int32)
    if G:
        WA = np.zeros(G * 256); WE = np.zeros(G * 256)
        WZg = np.zeros(G * 16 * S); AWg = np.zeros(G * 16 * S); EWg = np.zeros(G * 16 * S)
        gzg = np.zeros(S)
        for g in range(G):
            J = Js[g]
            if J == 0:
                continue
            Wg, AWg_, EWg_ = groups["W"][g], groups["AW"][g], groups["EW"][g]
            WA[g * 256:g * 256 + J * J] = _h(ops.utv(Wg, AWg_)).ravel()
            WE[g * 256:g * 256 + J * J] = _h(ops.utv(Wg, EWg_)).ravel()
            if Gh is not None:
                WZg[g * 16 * S:g * 16 * S + J * S] = _h(ops.utv(Wg, ZGh)).ravel()
                AWg[g * 16 * S:g * 16 * S + J * S] = _h(ops.utv(AWg_, Gh)).ravel()
                EWg[g * 16 * S:g * 16 * S + J * S] = _h(ops.utv(EWg_, Gh)).ravel()
        if Gh is not None:
            gzg = _h(ops.dot(Gh, ZGh))
        Jh = np.ascontiguousarray(Js, dtype=np.int32)
        st = lib.rsk_local_gram_factors(S, G, _iptr(Jh), _iptr(gos), _ptr(gam), _ptr(WA), _ptr(WE), _ptr(WZg),
                                        _ptr(AWg), _ptr(EWg), _ptr(gzg), _ptr(Lf), _iptr(m), _iptr(hasg),
                                        _iptr(dropped))
        if st != L.RSK_OK:
            raise RskError(f"rsk_local_gram_factors failed ({st})")

    def zcols(Ua, Ue, R_):
        """per shift, its group's (Ua)^T r and (Ue)^T r (Jm x S column-major; Ue may be None)"""
        za = np.zeros(Jm * S); ze = np.zeros(Jm * S) if Ue is not None else None
        for g in range(G):
            J = Js[g]
            if J == 0:
                continue
            ca = _h(ops.utv(Ua[g], R_))                 # (S, J)
            ce = _h(ops.utv(Ue[g], R_)) if Ue is not None else None
            for s_ in np.nonzero(gos == g)[0]:
                za[s_ * Jm:s_ * Jm + J] = ca[s_]
                if ce is not None:
                    ze[s_ * Jm:s_ * Jm + J] = ce[s_]
        return za, ze

    def gram_solve(za, ze, zg):
        mu = np.zeros(S * KM)
        st2 = lib.rsk_gram_solve(S, Jm, _ptr(Lf), _iptr(m), _iptr(hasg), _ptr(gam), _ptr(za),
                                 None if ze is None else _ptr(ze), None if zg is None else _ptr(zg), _ptr(mu))
        if st2 != L.RSK_OK:
            raise RskError(f"rsk_gram_solve failed ({st2})")
        return mu.reshape(S, KM)

    def sub_u(mu, V, which, sign=-1.0):
        """V -= U mu (U = W / AW / EW of each shift's group) over the shifts' own columns"""
        op = L.RSK_SUB_UC if sign < 0 else L.RSK_ADD_UC
        for g in range(G):
            J = Js[g]
            if J == 0:
                continue
            nwv = m - hasg
            C = np.zeros((S, J))
            for s_ in np.nonzero(gos == g)[0]:
                k = min(J, int(nwv[s_]))
                C[s_, :k] = mu[s_, :k]
            if not C.any():
                continue
            ops.add_uc(op, groups[which][g], V, torch.from_numpy(np.ascontiguousarray(C)).to(ops.dev))

    def mu_g(mu):
        """coefficient of the carried column (0 where absent)"""
        nwv = m - hasg
        return np.array([mu[s_, nwv[s_]] if hasg[s_] else 0.0 for s_ in range(S)])

    R = torch.empty(S, ops.own_n, **f)
    P = torch.zeros(S, ops.ext_n, **f)
    Wv = torch.empty(S, ops.ext_n, **f)
    applies = np.zeros(S, np.int64)
    scnt = np.zeros(S, np.int32)
    # ---- r_p = b - A_gamma x_p (one fresh apply for the shifts with x_p, G15)
    ops.apply(X, Wv, gam_d)
    applies += hx
    R.copy_(Bv)
    ops.axpby(-hx.astype(np.float64), Wv, ones, R)
    # ---- Galerkin start on Range(U): c = G^-1 U^T r_p; x += U c; r -= Z c
    if G:
        za, _ = zcols(groups["W"], None, R)
        zg = _h(ops.dot(Gh, R)) if Gh is not None else None
        c = gram_solve(za, None, zg)
        sub_u(c, X, "W", +1.0)
        sub_u(c, R, "AW", -1.0)
        T = torch.zeros(S, ops.own_n, **f)
        sub_u(c, T, "EW", +1.0)
        ops.axpby(-gam, T, ones, R)
        if Gh is not None:
            cg_ = mu_g(c)
            ops.axpby(cg_, Gh, ones, X)
            ops.axpby(-cg_, ZGh, ones, R)
    rho = _h(ops.dot(R, R))
    state = np.where(np.sqrt(rho) <= thr, LOOP_RCONV, LOOP_ACTIVE).astype(np.int32)
    iters = np.zeros(S, np.int32)
    nconf = np.zeros(S, np.int32)
    rho_true = np.zeros(S)
    beta = np.zeros(S)
    alpha = np.zeros(S)

    def new_p(mask, mu, rho_now):
        """p = r + beta p - W mu_W - ghat mu_g for the masked shifts; residual store"""
        a = np.where(mask, 1.0, 0.0)
        bb = np.where(mask, beta, 1.0)
        ops.axpby(a, R, bb, P)
        if G:
            sub_u(np.where(mask[:, None], mu, 0.0), P, "W", -1.0)
            if Gh is not None:
                ops.axpby(-np.where(mask, mu_g(mu), 0.0), Gh, ones, P)
        if store is not None:
            for s_ in np.nonzero(mask)[0]:
                if scnt[s_] < store_cap:
                    row = int(s_) * store_cap + int(scnt[s_])
                    dst = store[row:row + 1]
                    sc = np.zeros(1)
                    ops.axpby(np.array([1.0 / np.sqrt(rho_now[s_])]), R[s_:s_ + 1], sc, dst)
                    scnt[s_] += 1

    # p_0 = r_0 - U mu_0 with mu_0 = G^-1 Z^T r_0
    if G:
        za, ze = zcols(groups["AW"], groups["EW"], R)
        mu0 = gram_solve(za, ze, _h(ops.dot(ZGh, R)) if Gh is not None else None)
    else:
        mu0 = np.zeros((S, KM))
    new_p(state == LOOP_ACTIVE, mu0, rho)
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
        if G:
            za, ze = zcols(groups["AW"], groups["EW"], R)
            zg = _h(ops.dot(ZGh, R)) if Gh is not None else None
        else:
            za, ze, zg = np.zeros(1), np.zeros(1), None
        mu = np.zeros(S * KM)
        st = lib.rsk_cg_scalars(S, Jm, _iptr(mode), _ptr(gam), _ptr(rho_new), _ptr(za), _ptr(ze),
                                None if zg is None else _ptr(zg), _iptr(m), _iptr(hasg), _ptr(Lf), float(thr),
                                int(maxit), _ptr(rho), _ptr(beta), _ptr(mu), _iptr(iters), _ptr(rho_true),
                                _iptr(nconf), _iptr(state))
        if st != L.RSK_OK:
            raise RskError(f"rsk_cg_scalars failed ({st})")
        new_p(state == LOOP_ACTIVE, mu.reshape(S, KM), rho)
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
    if Gout is not None:
        ops.own(Gout).copy_(ops.own(X))
        ops.axpby(-ones, X0, ones, Gout)
    stat = np.where(state == LOOP_DONE, np.where(dropped > 0, L.RSK_CG_DEFL_DROPPED, L.RSK_CG_CONVERGED),
                    np.where(state == LOOP_BREAKDOWN, L.RSK_CG_BREAKDOWN, L.RSK_CG_MAXIT))
    out.update(iters=iters, applies=applies, relres=np.sqrt(np.maximum(rho_true, 0.0)) / nb,
               status=stat.astype(np.int32), m_used=m, store_count=scnt, relres_true=None)
    out["relres_true"] = out["relres"]
    out["dropped"] = dropped
    return out


# ------------------------------------------------------------------ the outer step in slab mode
class SlabHandle:
    """The librsk Handle interface GpuSolver uses, with row-slab semantics: vectors are
    extended (ext_rows x nx) tensors, every reduction is over owned rows and all-reduced,
    applies refresh the halo first, the thin QR is the shifted Cholesky-QR3 with all-reduced
    Grams (rsk_cholqr_pass)."""

    def __init__(self, ops: SlabOps):
        self.o = ops
        self.lib = ops.lib

    def set_weights(self, wx, wy, stream=None):
        self.o.h.set_weights(wx, wy)

    def apply_shifted(self, X, Y, gamma=None, EY=None, xdoty=None, mode=L.RSK_APPLY_SHIFTED, stream=None, nvec=None):
        self.o.apply(X, Y, gamma, mode=mode, EY=EY)
        if xdoty is not None:
            xdoty.copy_(self.o.dot(X, Y))

    def recycle_project(self, op, U, V, Cm, k=None, nv=None, stream=None):
        if op == L.RSK_PROJ_UTV:
            Cm.copy_(self.o.utv(U, V).reshape(Cm.shape))
        else:
            self.o.add_uc(op, U, V, Cm)

    def batch_dot(self, X, Y, out, stream=None):
        out.copy_(self.o.dot(X, Y))

    def batch_axpby(self, a, X, b, Y, stream=None):
        self.o.axpby(a, X, b, Y)

    def qr_tall(self, V, Q, stream=None) -> np.ndarray:
        """V (k, n) -> Q with orthonormal rows over the whole image, R (k x k, Fortran):
        three shifted-Cholesky-QR passes (V -> Q -> V -> Q) with all-reduced Grams."""
        o = self.o
        k = V.shape[0]
        nglob = o.plan.ny * o.plan.nx
        Racc = np.zeros(k * k)
        T = np.zeros(k * k)
        src, dst = V, Q
        for pss in range(3):
            G = _h(o.utv(src, src)).ravel()                 # (k x k) row a = src^T src_a: symmetric
            st = self.lib.rsk_cholqr_pass(k, nglob, pss, _ptr(np.ascontiguousarray(G)), _ptr(T), _ptr(Racc))
            if st != L.RSK_OK:
                raise RskError(f"rsk_cholqr_pass failed ({st})")
            o.own(dst).zero_()
            # dst_j = sum_i src_i T[i, j]  ->  Cm[j, i] = T[i + j k]
            Cm = torch.from_numpy(np.ascontiguousarray(T.reshape(k, k))).to(o.dev)
            o.add_uc(L.RSK_ADD_UC, src, dst, Cm)
            src, dst = dst, src
        return np.asfortranarray(Racc.reshape((k, k), order="F"))   # R[i, j] = Racc[i + j k]

    def lcurve_norms(self, X, d, rho, eta2, scratch, stream=None):
        rho.copy_(torch.sqrt(self.o.resnorm2(X, d)))
        eta2.copy_(torch.sqrt(self.o.seminorm2(X)))

    def irn_weights(self, x, tau, wx=None, wy=None, eta2=None, stream=None):
        self.o.comm.halo(x[None])
        self.o.h.irn_weights(x, tau, wx, wy)

    def irn_weights_iso(self, x, tau, wx=None, wy=None, eta2=None, stream=None):
        self.o.comm.halo(x[None])
        self.o.h.irn_weights_iso(x, tau, wx, wy)

    def gazzola_weights(self, x, p, dx, dy, wx, wy, stream=None):
        self.o.gazzola_weights(x, p, dx, dy, wx, wy)

    def make_rhs(self, x_true, xi, nu, d, b, stream=None):
        """d = C x_true + nu ||C x_true|| xi / ||xi||, b = C^T d (norms over the image)"""
        o = self.o
        Xt = x_true.reshape(1, -1).clone()
        Cx = torch.empty_like(Xt)
        o.apply(Xt, Cx, mode=L.RSK_APPLY_C_ONLY)
        ncx = float(np.sqrt(_h(o.dot(Cx, Cx))[0]))
        xv = xi.reshape(1, -1).clone()
        nxi = float(np.sqrt(_h(o.dot(xv, xv))[0]))
        D = d.reshape(1, -1)
        o.own(D).copy_(o.own(Cx))
        o.axpby(np.array([nu * ncx / nxi]), xv, np.ones(1), D)
        Bm = b.reshape(1, -1)
        o.apply(D, Bm, mode=L.RSK_APPLY_CT_ONLY)

    def cg_workspace_bytes(self, nshift, flags=0) -> int:
        return 8


class SlabGpuSolver:
    """GpuSolver's nested solve (pipeline.py) on one row slab: the same outer step, run
    SPMD on every rank with SlabHandle for the vector work and slab_cg for the batched
    deflated CG. Vectors are extended slab vectors (ext_rows x nx)."""

    def __init__(self, cfg, psf: np.ndarray, gamma: np.ndarray, plan: SlabPlan, rank: int, comm, device: int = 0):
        from . import pipeline as pl
        from . import shard
        self._pl = pl
        torch.cuda.set_device(device)
        self.dev = torch.device("cuda", device)
        self.cfg = cfg
        self.plan, self.rank = plan, rank
        self.o = SlabOps(plan, rank, comm, psf, device)
        self.n, self.M = cfg.n, cfg.M
        self.N = self.o.ext_n
        self.gamma = np.ascontiguousarray(gamma, dtype=np.float64)
        self.h = SlabHandle(self.o)
        self.check_every = 8
        self.profile = False
        self.stream = None
        self.dist = shard.Dist(False)
        f = dict(dtype=torch.float64, device=self.dev)
        self.f = f
        N, M = self.N, self.M
        self.gam_dev = torch.from_numpy(self.gamma).to(self.dev)
        self.b = torch.empty(N, **f)
        self.d = torch.empty(N, **f)
        w0 = torch.ones(self.n, self.n, **f)
        w0[:, -1] = 0.0
        self.w0x = plan.extend(w0.reshape(-1), rank).contiguous()
        self.w0y = plan.extend(w0.t().contiguous().reshape(-1), rank).contiguous()
        self.wx = torch.empty(N, **f)
        self.wy = torch.empty(N, **f)
        self.ws = torch.empty(8, dtype=torch.uint8, device=self.dev)
        self.lc_scratch = torch.empty(M, N, **f)
        self.rho_dev = torch.empty(M, **f)
        self.eta_dev = torch.empty(M, **f)
        self.grp = np.array([0 if (l + 1) <= shift_indices(cfg).I_split else 1 for l in range(M)], dtype=np.int32)

    def set_data(self, x_true_full: torch.Tensor, xi_full: torch.Tensor):
        """the global seeded images, cut to this slab (each rank holds its rows + halo)"""
        xt = self.plan.extend(x_true_full.reshape(-1), self.rank)
        xi = self.plan.extend(xi_full.reshape(-1), self.rank)
        self.h.make_rhs(xt, xi, self.cfg.noise, self.d, self.b)

    def cg(self, gammas_idx, X, has_xp, Gout=None, groups=None, ghat=None, store=None, flags=0, order=None,
           inner="cg", ghat2=None, rhs=None, maxit=None):
        from .pipeline import STORE_CAP
        if inner != "cg" or ghat2 is not None or rhs is not None:
            raise NotImplementedError("row slabs run the recycled CG inner solve (north_star) only")
        return slab_cg(self.o, self.gamma[list(gammas_idx)], self.b, X, tol=self.cfg.tol,
                       maxit=self.cfg.maxit if maxit is None else maxit,
                       has_xp=has_xp, groups=groups, ghat=ghat, store=store, store_cap=STORE_CAP, Gout=Gout)

    def __getattr__(self, name):
        # the outer-step logic is GpuSolver's, bound to this object
        attr = getattr(self._pl.GpuSolver, name)
        if callable(attr):
            return attr.__get__(self, type(self))
        return attr


def main(argv=None):
    """Row-slab nested solve across GPUs (one rank per GPU, NCCL):
    python -m torch.distributed.run --nproc-per-node G -m paper_2306_15049_b200.slab --config C5 --outer 1"""
    import argparse
    import os
    import time

    import torch.distributed as dist

    import rsk_synth as S
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--outer", type=int, default=1)
    a = ap.parse_args(argv)
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    cfg = S.CONFIGS[a.config]
    inp = S.make_inputs(cfg)
    plan = SlabPlan(cfg.n, cfg.n, cfg.r, world)
    dev = torch.device("cuda", local)
    sol = SlabGpuSolver(cfg, inp["psf"], inp["gamma"], plan, rank, DistComm(plan, rank), device=local)
    t0 = time.perf_counter()
    sol.set_data(torch.from_numpy(inp["x_true"]).to(dev), torch.from_numpy(inp["xi"]).to(dev))
    outs = sol.run(K_out=a.outer)
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t0
    if rank == 0:
        for o in outs:
            print(f"outer {o.k}: iters {o.iters.tolist()} l* {o.lstar} status {o.status.tolist()}", flush=True)
        print(f"{cfg.name} on {world} row slabs: {dt:.1f} s", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
