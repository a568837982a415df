"""The outer IRN loop of Alg. 5 on the B200, driving librsk.

Orchestration only: every arithmetic step on data is a librsk call (device
kernels, or the host small-dense helpers of include/rsk.h). torch provides
memory (fp64 CUDA tensors), streams and copies. The readings of the paper
(D1-D4, G1-G29) are the ones listed in DESIGN.md and followed by the oracle.

One outer step k:
  1. k = 0: seed solves at gamma_i1, gamma_i2 (plain CG with a residual store)
     and Rayleigh-Ritz spaces V_i1, V_i2 (§5.1)
     k >= 1: raw block [V_i1, x^(k-1,1..M)] (eq:tildeUupdate P:654, reading G10)
  2. stabilize (Alg. 1): shifted Cholesky-QR3 + Jacobi SVD of R
  3. anchor (A + gamma_* E) U~ = K R (eq:establishU) and the Grams
  4. principal guesses x_0 = U~ C (eq:orthupdate)
  5. group Ritz blocks W_g, A W_g, E W_g from the pencil (Alg. 2/4)
  6. carried corrections g-hat (Alg. 3, reading D3) and their images
  7. batched deflated CG over all shifts (rsk_cg_recycled_batch)
  8. L-curve corner and the IRN weights of x* (north_star)
"""
from __future__ import annotations

import dataclasses
import math
import os
import time

import numpy as np
import torch

from . import _lib as L
from . import shard
from .indices import shift_indices
from .rsk import (Handle, carried_select, lcurve_corner, oblique_guess, orth_guess, pencil_ritz,
                  stabilize_small, sym_eig)

COND_CAP = 1e10
DUP_SIN = math.sqrt(1.0 - 0.999 ** 2)
STORE_CAP = 100


@dataclasses.dataclass
class StepOut:
    k: int
    iters: np.ndarray
    applies: np.ndarray
    status: np.ndarray
    relres: np.ndarray
    m_used: np.ndarray
    nc: int
    lstar: int
    rho: np.ndarray
    eta: np.ndarray
    overhead_applies: int
    has_xp: np.ndarray
    keep_ghat: np.ndarray | None
    ms: float = 0.0
    prof: np.ndarray | None = None


def _host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


class _Phases:
    """NVTX ranges for the phases of one outer step: an outer range, one nested range per
    phase (each call closes the previous phase)."""

    def __init__(self, name: str):
        torch.cuda.nvtx.range_push(name)
        self.open = False

    def __call__(self, phase: str):
        if self.open:
            torch.cuda.nvtx.range_pop()
        torch.cuda.nvtx.range_push(phase)
        self.open = True

    def end(self):
        if self.open:
            torch.cuda.nvtx.range_pop()
        torch.cuda.nvtx.range_pop()


class _nvtx:
    """NVTX range around a phase of the outer step (visible in Nsight Systems / ncu)."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        torch.cuda.nvtx.range_push(self.name)

    def __exit__(self, *a):
        torch.cuda.nvtx.range_pop()


def report_rows(outs, gamma) -> list[dict]:
    """Per (outer step k, shift l) accounting -- the quantity of the paper's matvec figures
    (P:1075-1081): gamma, inner iterations, A_gamma applies (each counts one
    A and one E matvec: shifted applies), true relative residual, status, local dimension,
    and the outer step's fixed applies (seeds, Ritz, anchoring, g-hat images) on l = -1."""
    rows = []
    for o in outs:
        for l in range(len(o.iters)):
            rows.append(dict(k=int(o.k), l=l + 1, gamma=float(gamma[l]), iters=int(o.iters[l]),
                             applies_A=int(o.applies[l]), applies_E=int(o.applies[l]),
                             relres=float(o.relres[l]), status=int(o.status[l]), m_used=int(o.m_used[l]),
                             principal_guess=int(o.has_xp[l]), lstar=int(o.lstar) + 1, nc=int(o.nc)))
        rows.append(dict(k=int(o.k), l=-1, gamma=float("nan"), iters=0, applies_A=int(o.overhead_applies),
                         applies_E=int(o.overhead_applies), relres=float("nan"), status=-1, m_used=0,
                         principal_guess=0, lstar=int(o.lstar) + 1, nc=int(o.nc)))
    return rows


class GpuSolver:
    """All device state of one configuration (one image grid, one PSF, M shifts)."""

    def __init__(self, cfg, psf: np.ndarray, gamma: np.ndarray, device: int = 0,
                 check_every: int = 8, profile: bool = False, stream=None, dist=None):
        torch.cuda.set_device(device)
        self.dev = torch.device("cuda", device)
        self.cfg = cfg
        self.n, self.N, self.M = cfg.n, cfg.N, cfg.M
        self.gamma = np.ascontiguousarray(gamma, dtype=np.float64)
        if getattr(cfg, "operator", "blur") == "ct":
            # Example 2 (f4): C = the parallel-beam CT matrix; the CG device loops embed the
            # stencil apply, so the inner solves (seeds included) are recycling MINRES
            if getattr(cfg, "inner", "cg") != "minres":
                raise ValueError("operator='ct' needs inner='minres'")
            self.h = Handle.ct(cfg.n, np.arange(1, cfg.n_angles + 1, dtype=np.float64), cfg.ndet, device)
        else:
            self.h = Handle(cfg.n, cfg.n, psf, device)
        self.check_every = check_every
        self.profile = profile
        self.stream = stream
        self.dist = dist if dist is not None else shard.Dist(False)
        f = dict(dtype=torch.float64, device=self.dev)
        N, M = self.N, self.M
        self.f = f
        self.gam_dev = torch.from_numpy(self.gamma).to(self.dev)
        self.b = torch.empty(N, **f)
        self.d = torch.empty(self.h.ndata, **f)       # data vector (ndata = N for the blur)
        w0 = torch.ones(self.n, self.n, **f)
        w0[:, -1] = 0.0
        self.w0x = w0.reshape(-1).contiguous()
        self.w0y = w0.t().contiguous().reshape(-1).contiguous()
        self.wx = torch.empty(N, **f)
        self.wy = torch.empty(N, **f)
        self.ws = torch.empty(self.h.cg_workspace_bytes(max(M, 2)), dtype=torch.uint8, device=self.dev)
        self.lc_scratch = torch.empty(M, self.h.ndata, **f)
        self.rho_dev = torch.empty(M, **f)
        self.eta_dev = torch.empty(M, **f)
        self.grp = np.array([0 if (l + 1) <= shift_indices(cfg).I_split else 1 for l in range(M)], dtype=np.int32)

    # ------------------------------------------------------------------ data
    def set_data(self, x_true: torch.Tensor, xi: torch.Tensor):
        """d = C x_true + e, b = C^T d on the device (rsk_make_rhs)."""
        self.h.make_rhs(x_true.reshape(-1), xi.reshape(-1), self.cfg.noise, self.d, self.b,
                        stream=self.stream)

    def reset_weights(self):
        self.h.set_weights(self.w0x, self.w0y, stream=self.stream)
        self.cur_w = (self.w0x, self.w0y)       # the handle's W_k (eq:delta needs W_{k-1})
        self.w_prev = None
        if getattr(self.cfg, "weight_rule", "irn") == "gazzola":
            # D_0 = I, held in the weights' padded layout
            self.Dx = self.w0x.clone()
            self.Dy = self.w0y.clone()

    # ------------------------------------------------------------- building blocks
    def cg(self, gammas_idx, X, has_xp, Gout=None, groups=None, ghat=None, store=None,
           flags=0, order=None, inner="cg", ghat2=None, rhs=None, maxit=None):
        """One batched inner solve over the shifts gammas_idx: recycled CG
        (rsk_cg_recycled_batch) or, with inner="minres", the paper's recycling MINRES
        (rsk_minres_recycled_batch) on the same descriptor."""
        cfg = self.cfg
        ns = len(gammas_idx)
        gam = np.ascontiguousarray(self.gamma[gammas_idx])
        d = L.CgDesc()
        d.nshift = ns
        d.gamma_h = gam.ctypes.data_as(L._hp)
        d.b = (self.b if rhs is None else rhs).data_ptr()
        d.X = X.data_ptr(); d.ldx = self.N
        hx = np.ascontiguousarray(has_xp, dtype=np.int32)
        d.has_xp_h = hx.ctypes.data_as(L.C.POINTER(L.C.c_int))
        d.Gout = Gout.data_ptr() if Gout is not None else None
        if order is not None:   # device-loop start order (longest predicted first)
            od = np.ascontiguousarray(order, dtype=np.int32)
            d.order_h = od.ctypes.data_as(L.C.POINTER(L.C.c_int))
        d.ldg = self.N
        keep = []
        if groups is not None:
            gos = np.ascontiguousarray(groups["of_shift"], dtype=np.int32)
            keep.append(gos)
            d.ngroups = len(groups["W"])
            d.group_of_shift_h = gos.ctypes.data_as(L.C.POINTER(L.C.c_int))
            for g in range(d.ngroups):
                d.W[g] = groups["W"][g].data_ptr()
                d.AW[g] = groups["AW"][g].data_ptr()
                d.EW[g] = groups["EW"][g].data_ptr()
                d.J[g] = groups["W"][g].shape[0]
            d.ldw = self.N
        else:
            d.ngroups = 0
            flags |= L.RSK_CG_NO_DEFLATION
        if ghat is not None:
            Gh, ZGh, hg = ghat
            hg = np.ascontiguousarray(hg, dtype=np.int32)
            keep.append(hg)
            d.Ghat = Gh.data_ptr(); d.ZGhat = ZGh.data_ptr(); d.ldgh = self.N
            d.has_ghat_h = hg.ctypes.data_as(L.C.POINTER(L.C.c_int))
        if ghat2 is not None:
            Gh2, ZGh2, hg2 = ghat2
            hg2 = np.ascontiguousarray(hg2, dtype=np.int32)
            keep.append(hg2)
            d.Ghat2 = Gh2.data_ptr(); d.ZGhat2 = ZGh2.data_ptr(); d.ldgh = self.N
            d.has_ghat2_h = hg2.ctypes.data_as(L.C.POINTER(L.C.c_int))
        if store is not None:
            d.store = store.data_ptr(); d.lds = self.N; d.store_cap = STORE_CAP
            flags |= L.RSK_CG_STORE_RES
        if self.profile:
            flags |= L.RSK_CG_PROFILE
        d.tol = cfg.tol; d.maxit = cfg.maxit if maxit is None else maxit; d.check_every = self.check_every; d.flags = flags
        if order is not None:
            keep.append(od)
        out = L.CgOut()
        iters = np.zeros(ns, dtype=np.int32); apl = np.zeros(ns, dtype=np.int64)
        rel = np.zeros(ns); stt = np.zeros(ns, dtype=np.int32); mu = np.zeros(ns, dtype=np.int32)
        sc = np.zeros(ns, dtype=np.int32); ms = np.zeros(8)
        P = L.C.POINTER
        out.iters = iters.ctypes.data_as(P(L.C.c_int)); out.applies = apl.ctypes.data_as(P(L.C.c_int64))
        out.relres_true = rel.ctypes.data_as(L._hp); out.status = stt.ctypes.data_as(P(L.C.c_int))
        out.m_used = mu.ctypes.data_as(P(L.C.c_int)); out.store_count = sc.ctypes.data_as(P(L.C.c_int))
        out.ms_loop = ms.ctypes.data_as(L._hp)
        if inner == "minres":
            kmax = (max(d.J[g] for g in range(d.ngroups)) + (1 if ghat is not None else 0)
                    + (1 if ghat2 is not None else 0)) if d.ngroups else 0
            need = self.h.minres_workspace_bytes(ns, kmax)
            if getattr(self, "ws_mr", None) is None or self.ws_mr.numel() < need:
                self.ws_mr = torch.empty(need, dtype=torch.uint8, device=self.dev)
            self.h.minres_recycled_batch(d, out, self.ws_mr, stream=self.stream)
        else:
            self.h.cg_recycled_batch(d, out, self.ws, stream=self.stream)
        return dict(iters=iters, applies=apl, relres=rel, status=stt, m_used=mu, store_count=sc, prof=ms)

    def stabilize(self, raw: torch.Tensor, cap: int | None) -> torch.Tensor:
        """Alg. 1 with column scaling (reading G6); zero columns are discarded."""
        k = raw.shape[0]
        nrm = torch.empty(k, **self.f)
        self.h.batch_dot(raw, raw, nrm, stream=self.stream)
        n2 = _host(nrm)
        nz = np.nonzero(n2 > 0)[0]
        V = raw[torch.from_numpy(nz).to(self.dev)].contiguous() if len(nz) < k else raw.clone()
        Q = torch.empty_like(V)
        R = self.h.qr_tall(V, Q, stream=self.stream)
        Zs, nk = stabilize_small(R, n2[nz], COND_CAP, cap or 0)
        Ut = torch.zeros(nk, self.N, **self.f)
        Cm = torch.from_numpy(np.ascontiguousarray(Zs.T)).to(self.dev)
        self.h.recycle_project(L.RSK_ADD_UC, Q, Ut, Cm, stream=self.stream)
        return Ut

    def utv(self, U, V):
        Cm = torch.empty(V.shape[0] if V.dim() > 1 else 1, U.shape[0], **self.f)
        self.h.recycle_project(L.RSK_PROJ_UTV, U, V, Cm, stream=self.stream)
        return Cm

    def combine(self, U, Cm_host_kxnv: np.ndarray) -> torch.Tensor:
        """U (k, N) times the k x nv host matrix -> (nv, N) via ADD_UC into zeros."""
        Cm = torch.from_numpy(np.ascontiguousarray(np.asarray(Cm_host_kxnv).T)).to(self.dev)
        out = torch.zeros(Cm.shape[0], self.N, **self.f)
        self.h.recycle_project(L.RSK_ADD_UC, U, out, Cm, stream=self.stream)
        return out

    def ritz(self, store_blk: torch.Tensor, gamma_idx: int, n_keep: int):
        """Rayleigh-Ritz on a seed's stored residuals (reading G9)."""
        Q = self.stabilize(store_blk, None)
        q = Q.shape[0]
        AQ = torch.empty_like(Q)
        gq = self.gam_dev[gamma_idx].repeat(q).contiguous()
        self.h.apply_shifted(Q, AQ, gamma=gq, stream=self.stream)
        H = _host(self.utv(Q, AQ)).T          # q x q  (column-major view)
        th, Z = sym_eig(H)
        kk = min(n_keep, q)
        return self.combine(Q, Z[:, :kk]), q

    # ------------------------------------------------------------- one outer step
    def _principal(self, k: int, st: dict, images: bool = True):
        """Rank-0 part of the outer step: raw block, stabilize (Alg. 1) and (images=True)
        the anchor images A U~, E U~ (n_c split applies; with several ranks they are
        column-split across the ranks instead, see outer_step).
        Returns (Ut, ZA, ZE, V_i1, overhead)."""
        cfg = self.cfg
        N, nc_cap = self.N, cfg.n_c
        overhead = 0
        i1, i2 = shift_indices(cfg).i1 - 1, shift_indices(cfg).i2 - 1
        V_i1 = st.get("V_i1")
        if k == 0:
            n1 = math.ceil(2 * (nc_cap - 2) / 3)
            n2 = nc_cap - 2 - n1
            Xs = torch.empty(2, N, **self.f)
            store = torch.empty(2 * STORE_CAP, N, **self.f)
            rs = self.cg([i1, i2], Xs, [0, 0], store=store, inner=getattr(cfg, "inner", "cg"))
            overhead += int(rs["applies"].sum())
            c1, c2 = int(rs["store_count"][0]), int(rs["store_count"][1])
            V_i1, q1 = self.ritz(store[:c1], i1, n1) if n1 > 0 and c1 > 0 else (Xs[:0], 0)
            V_i2, q2 = self.ritz(store[STORE_CAP:STORE_CAP + c2], i2, n2) if n2 > 0 and c2 > 0 else (Xs[:0], 0)
            overhead += q1 + q2
            raw = torch.cat([Xs, V_i1, V_i2], 0)
            del store
        elif getattr(cfg, "principal", "g10") == "vnew" and st.get("W_prev") is not None:
            V_new, a_new = self.principal_update(st)
            overhead += a_new
            raw = torch.cat([V_i1, V_new, st["X_prev"]], 0)
        else:
            raw = torch.cat([V_i1, st["X_prev"]], 0)
        Ut = self.stabilize(raw, nc_cap)
        nc = Ut.shape[0]
        del raw
        overhead += nc
        if not images:
            return Ut, None, None, V_i1, overhead
        ZA = torch.empty(nc, N, **self.f)
        ZE = torch.empty(nc, N, **self.f)
        self.h.apply_shifted(Ut, ZA, EY=ZE, mode=L.RSK_APPLY_SPLIT, stream=self.stream)
        return Ut, ZA, ZE, V_i1, overhead

    def principal_update(self, st: dict):
        """eq:delta (reading G36): at l_c solve
        (A + gamma_c E_k) dx = gamma_c (E_k - E_{k-1}) x^(k-1,l_c) by <= 100 CG steps from 0
        with the residual store; V^(new) = [dx, stored Krylov vectors]. The two E images
        are split applies under W_k and W_{k-1} (the handle's weights are swapped and
        restored). Returns (V_new, applies)."""
        cfg = self.cfg
        lc = shift_indices(cfg).l_c - 1
        x = st["X_prev"][lc:lc + 1].contiguous()
        Ax = torch.empty_like(x); Ek = torch.empty_like(x); Ep = torch.empty_like(x)
        self.h.apply_shifted(x, Ax, EY=Ek, mode=L.RSK_APPLY_SPLIT, stream=self.stream)
        wpx, wpy = st["W_prev"]
        self.h.set_weights(wpx, wpy, stream=self.stream)
        self.h.apply_shifted(x, Ax, EY=Ep, mode=L.RSK_APPLY_SPLIT, stream=self.stream)
        self.h.set_weights(self.cur_w[0], self.cur_w[1], stream=self.stream)
        gc = float(self.gamma[lc])
        self.h.batch_axpby(np.array([-gc]), Ep, np.array([gc]), Ek, stream=self.stream)   # q
        dx = torch.zeros(1, self.N, **self.f)
        store = torch.empty(STORE_CAP, self.N, **self.f)
        r = self.cg([lc], dx, [0], store=store, rhs=Ek, maxit=100, inner=getattr(cfg, "inner", "cg"))
        cnt = int(r["store_count"][0])
        return torch.cat([dx, store[:cnt]], 0), int(r["applies"][0]) + 2

    def outer_step(self, k: int, st: dict) -> tuple[StepOut, dict]:
        cfg = self.cfg
        N, M = self.N, self.M
        dist = self.dist
        t0 = time.perf_counter()
        ph = _Phases(f"rsk outer step k={k}")
        ph("principal space (seeds / Ritz / stabilize)")
        owners = shard.assignment(k, M, dist.world, st.get("prev_iters"), groups=self.grp, J=cfg.J)
        mine = owners[dist.rank]
        ml = len(mine)
        # ---- principal space on rank 0, broadcast once per outer step (§8(e1))
        V_i1 = st.get("V_i1")
        overhead = 0
        if dist.rank == 0:
            Ut, ZA, ZE, V_i1, overhead = self._principal(k, st, images=not dist.enabled)
            nc = Ut.shape[0]
        nc = dist.bcast_int(nc if dist.rank == 0 else 0, self.dev)
        if dist.rank != 0:
            Ut = torch.empty(nc, N, **self.f)
        if dist.enabled:
            # U~ from rank 0; the n_c anchoring applies A U~, E U~ column-split across the
            # ranks (contiguous blocks), then all-gathered
            torch.cuda.synchronize(self.dev)
            dist.bcast(Ut)
            cols = [list(range(r * nc // dist.world, (r + 1) * nc // dist.world)) for r in range(dist.world)]
            mc = cols[dist.rank]
            za = torch.empty(len(mc), N, **self.f)
            ze = torch.empty(len(mc), N, **self.f)
            if mc:
                self.h.apply_shifted(Ut[mc[0]:mc[-1] + 1], za, EY=ze, mode=L.RSK_APPLY_SPLIT, stream=self.stream)
            torch.cuda.synchronize(self.dev)
            ZA = dist.gather_rows(za, cols, nc)
            ZE = dist.gather_rows(ze, cols, nc)
        ph("anchoring + Grams")
        # ---- anchoring (eq:establishU) and Grams: identical on every rank
        gstar = float(self.gamma[shift_indices(cfg).istar - 1])
        Y = ZA.clone()
        self.h.batch_axpby(np.full(nc, gstar), ZE, None, Y, stream=self.stream)
        K = torch.empty_like(Y)
        R = self.h.qr_tall(Y, K, stream=self.stream)
        del Y
        KtZE = _host(self.utv(K, ZE)).T
        Ktb = _host(self.utv(K, self.b)).ravel()
        Ahat = _host(self.utv(Ut, ZA)).T
        Ehat = _host(self.utv(Ut, ZE)).T
        del K
        ph("principal guesses")
        # ---- principal guesses for this rank's shifts: eq:orthupdate, or the oblique
        # projections of §sec:oblique (f2(iii), Config.guess)
        mode = getattr(cfg, "guess", "orth")
        if mode == "orth":
            ZEtZE = _host(self.utv(ZE, ZE)).T
            ZEtb = _host(self.utv(ZE, self.b)).ravel()
            Cg, gst = orth_guess(R, KtZE, ZEtZE, ZEtb, Ktb, gstar, self.gamma)
        elif mode == "oblique":
            Cg, gst = oblique_guess(R, KtZE, Ktb, gstar, self.gamma)
        elif mode == "oblique2":
            Cg, gst = self._two_anchor_guesses(ZA, ZE, R, KtZE, Ktb, gstar)
        else:
            raise ValueError(f"unknown guess mode {mode!r}")
        has_xp = (gst == 0).astype(np.int32)
        X = self.combine(Ut, Cg[:, mine]) if ml else torch.zeros(0, N, **self.f)
        if getattr(self, "guess_hook", None) is not None:     # diagnostics (tools/probe_guess.py)
            self.guess_hook(k, mine, X, has_xp[mine])
        ph("group Ritz blocks")
        # ---- group Ritz blocks (Alg. 2 / Alg. 4)
        Wg, AWg, EWg = [], [], []
        for jidx in (shift_indices(cfg).J_L - 1, shift_indices(cfg).J_R - 1):
            Wt, _ = pencil_ritz(Ahat, Ehat, float(self.gamma[jidx]), min(cfg.J, nc))
            Wg.append(self.combine(Ut, Wt)); AWg.append(self.combine(ZA, Wt)); EWg.append(self.combine(ZE, Wt))
        del ZA, ZE
        groups = dict(W=Wg, AW=AWg, EW=EWg, of_shift=self.grp[mine])
        ph("carried corrections")
        # ---- carried corrections (Alg. 3, reading D3 / G12) for this rank's shifts
        ghat = None
        keep = None
        nL = int(np.sum(np.asarray(mine) < shift_indices(cfg).I_split))
        if k >= 1 and st.get("G_prev") is not None and ml:
            idx = torch.tensor(mine, dtype=torch.long, device=self.dev)
            Gp = st["G_prev"][idx].contiguous()
            Gh = Gp.clone()
            bounds = [(0, nL), (nL, ml)]
            for _ in range(2):
                for g, (a, bnd) in enumerate(bounds):
                    if bnd > a:
                        cf = self.utv(Wg[g], Gh[a:bnd])
                        self.h.recycle_project(L.RSK_SUB_UC, Wg[g], Gh[a:bnd], cf, stream=self.stream)
            g2 = torch.empty(ml, **self.f); gh2 = torch.empty(ml, **self.f)
            self.h.batch_dot(Gp, Gp, g2, stream=self.stream)
            self.h.batch_dot(Gh, Gh, gh2, stream=self.stream)
            scale, keep = carried_select(_host(g2), _host(gh2), DUP_SIN)
            self.h.batch_axpby(np.zeros(ml), None, scale, Gh, stream=self.stream)
            ZGh = torch.empty_like(Gh)
            self.h.apply_shifted(Gh, ZGh, gamma=self.gam_dev[idx].contiguous(), stream=self.stream)
            overhead += int(keep.sum())
            ghat = (Gh, ZGh, keep)
        ph("batched inner solve")
        # ---- batched deflated CG on this rank's shifts
        G = torch.empty(ml, N, **self.f)
        if ml and getattr(cfg, "local", "d3") == "seq":
            res = self._wavefront(mine, X, has_xp[mine], G, groups, ghat)
            overhead += res.pop("overhead")
            self.h.lcurve_norms(X, self.d, self.rho_dev, self.eta_dev, self.lc_scratch, stream=self.stream)
            rho_l, eta_l = _host(self.rho_dev)[:ml], _host(self.eta_dev)[:ml]
        elif ml:
            prev = st.get("prev_iters")
            order = None
            if prev is not None and len(prev) == M:   # longest-processing-time first
                order = np.argsort(-np.asarray(prev)[mine], kind="stable")
            res = self.cg(mine, X, has_xp[mine], Gout=G, groups=groups, ghat=ghat, order=order,
                          inner=getattr(cfg, "inner", "cg"))
            self.h.lcurve_norms(X, self.d, self.rho_dev, self.eta_dev, self.lc_scratch, stream=self.stream)
            rho_l, eta_l = _host(self.rho_dev)[:ml], _host(self.eta_dev)[:ml]
        else:
            res = dict(iters=np.zeros(0, np.int32), applies=np.zeros(0, np.int64), status=np.zeros(0, np.int32),
                       relres=np.zeros(0), m_used=np.zeros(0, np.int32), prof=np.zeros(8))
            rho_l = eta_l = np.zeros(0)
        ph("exchange + L-curve")
        # ---- exchange (allgather) and the L-curve
        if dist.enabled:
            torch.cuda.synchronize(self.dev)
            Xf = dist.gather_rows(X, owners, M)
            Gf = dist.gather_rows(G, owners, M)
            packed = np.stack([res["iters"], res["applies"], res["status"], res["relres"], res["m_used"],
                               rho_l, eta_l, has_xp[mine]], 1) if ml else np.zeros((0, 8))
            allp = dist.gather_np(packed, owners, M, self.dev)
            iters, applies, status = allp[:, 0].astype(np.int64), allp[:, 1].astype(np.int64), allp[:, 2].astype(np.int64)
            relres, m_used, rho, eta = allp[:, 3], allp[:, 4].astype(np.int64), allp[:, 5], allp[:, 6]
            overhead = dist.bcast_int(overhead, self.dev)
        else:
            Xf, Gf = X, G
            iters, applies, status = res["iters"], res["applies"], res["status"]
            relres, m_used, rho, eta = res["relres"], res["m_used"], rho_l, eta_l
        lstar, _ = lcurve_corner(rho, eta)
        torch.cuda.synchronize(self.dev)
        ph.end()
        out = StepOut(k, iters, applies, status, relres, m_used, nc, lstar, rho, eta, overhead,
                      has_xp, keep, time.perf_counter() - t0, res["prof"])
        nst = dict(X_prev=Xf, G_prev=Gf, V_i1=V_i1, xstar=Xf[lstar], prev_iters=np.asarray(iters))
        return out, nst

    def _wavefront(self, mine, X, has_xp, G, groups, ghat):
        """Alg. 3 / Alg. 4 local spaces U~_l = [W_g, g^(k-1,l), g^(k,l-1)] (
        SURVEY §8(f) f2(i), reading G35): shift l needs the correction g^(k,l-1) of its
        predecessor in the same group, so each group is a chain solved in order and the
        two chains run side by side (a batch of <= 2 shifts per wavefront step), with the
        paper's recycling MINRES as the inner solver."""
        cfg = self.cfg
        if getattr(cfg, "inner", "cg") != "minres":
            raise ValueError("local='seq' needs inner='minres' (two carried columns per shift)")
        if self.dist.enabled and self.dist.world > 1:
            raise NotImplementedError("local='seq' chains are solved on one rank")
        ml = len(mine)
        chains = [[i for i in range(ml) if (mine[i] + 1) <= shift_indices(cfg).I_split],
                  [i for i in range(ml) if (mine[i] + 1) > shift_indices(cfg).I_split]]
        out = dict(iters=np.zeros(ml, np.int32), applies=np.zeros(ml, np.int64), relres=np.zeros(ml),
                   status=np.zeros(ml, np.int32), m_used=np.zeros(ml, np.int32), prof=np.zeros(8),
                   overhead=0)
        gos = groups["of_shift"]
        for t in range(max(len(c) for c in chains)):
            batch = [c[t] for c in chains if t < len(c)]
            idx = torch.tensor(batch, dtype=torch.long, device=self.dev)
            nb = len(batch)
            Xb = X[idx].contiguous()
            Gb = torch.empty(nb, self.N, **self.f)
            gh_b = None
            if ghat is not None:
                gh_b = (ghat[0][idx].contiguous(), ghat[1][idx].contiguous(), np.asarray(ghat[2])[batch])
            # second carried column g^(k,l-1): CGS2 against [W_g, g-hat_l], footnote P:691 test
            Gh2 = torch.zeros(nb, self.N, **self.f)
            has2 = np.zeros(nb, np.int32)
            for j, i in enumerate(batch):
                if t == 0:
                    continue
                prev = [c for c in chains if i in c][0][t - 1]
                Wg = groups["W"][gos[i]]
                gp = G[prev:prev + 1]
                gh = gp.clone()
                for _ in range(2):
                    cf = self.utv(Wg, gh)
                    self.h.recycle_project(L.RSK_SUB_UC, Wg, gh, cf, stream=self.stream)
                    if gh_b is not None and gh_b[2][j]:
                        g1 = gh_b[0][j:j + 1]
                        c1 = self.utv(g1, gh)
                        self.h.recycle_project(L.RSK_SUB_UC, g1, gh, c1, stream=self.stream)
                n0 = torch.empty(1, **self.f); n1 = torch.empty(1, **self.f)
                self.h.batch_dot(gp, gp, n0, stream=self.stream)
                self.h.batch_dot(gh, gh, n1, stream=self.stream)
                scale, keep = carried_select(_host(n0), _host(n1), DUP_SIN)
                if keep[0]:
                    self.h.batch_axpby(np.zeros(1), None, scale, gh, stream=self.stream)
                    Gh2[j] = gh[0]
                    has2[j] = 1
            ZGh2 = torch.zeros_like(Gh2)
            if has2.any():
                sel = [j for j in range(nb) if has2[j]]
                sidx = torch.tensor(sel, dtype=torch.long, device=self.dev)
                gsel = self.gam_dev[torch.tensor([mine[batch[j]] for j in sel], device=self.dev)].contiguous()
                src = Gh2[sidx].contiguous()
                img = torch.empty_like(src)
                self.h.apply_shifted(src, img, gamma=gsel, stream=self.stream)
                ZGh2[sidx] = img
                out["overhead"] += len(sel)
            grp_b = dict(W=groups["W"], AW=groups["AW"], EW=groups["EW"], of_shift=np.asarray(gos)[batch])
            r = self.cg([mine[i] for i in batch], Xb, np.asarray(has_xp)[batch], Gout=Gb, groups=grp_b,
                        ghat=gh_b, inner="minres", ghat2=(Gh2, ZGh2, has2))
            X[idx] = Xb
            G[idx] = Gb
            for key in ("iters", "applies", "relres", "status", "m_used"):
                out[key][batch] = r[key]
        return out

    def _two_anchor_guesses(self, ZA, ZE, R, KtZE, Ktb, gstar):
        """eq:updates (reading G34): oblique guesses of the left group from
        the anchor gamma_{I_L}, of the right group from gamma_{I_R}; the images Z_A, Z_E
        are shared, each extra anchor costs one shifted CholQR3 and two projections."""
        cfg = self.cfg
        nI = shift_indices(cfg).I_split
        parts = []
        for (ia, sl) in ((shift_indices(cfg).I_L, slice(0, nI)), (shift_indices(cfg).I_R, slice(nI, self.M))):
            ga = float(self.gamma[ia - 1])
            if ga == gstar:
                Ra, KtZEa, Ktba = R, KtZE, Ktb
            else:
                Y = ZA.clone()
                self.h.batch_axpby(np.full(ZA.shape[0], ga), ZE, None, Y, stream=self.stream)
                Ka = torch.empty_like(Y)
                Ra = self.h.qr_tall(Y, Ka, stream=self.stream)
                del Y
                KtZEa = _host(self.utv(Ka, ZE)).T
                Ktba = _host(self.utv(Ka, self.b)).ravel()
                del Ka
            parts.append(oblique_guess(Ra, KtZEa, Ktba, ga, self.gamma[sl]))
        return (np.asfortranarray(np.concatenate([parts[0][0], parts[1][0]], axis=1)),
                np.concatenate([parts[0][1], parts[1][1]]))

    def next_weights(self, xstar: torch.Tensor):
        """W_{k+1} from x*, adopted by the handle. cfg.weight_rule: "irn" (north_star,
        reading G2), "irn_iso" (isotropic IRN) or "gazzola" (D_{k+1} =
        diag(1 - w.^p) D_k)."""
        rule = getattr(self.cfg, "weight_rule", "irn")
        # W_k is kept for eq:delta (f3) BEFORE the rule overwrites self.wx / self.wy in
        # place (from step 1 on they are the handle's current weights)
        self.w_prev = (self.cur_w[0].clone(), self.cur_w[1].clone())
        if rule == "irn":
            self.h.irn_weights(xstar, self.cfg.tau, self.wx, self.wy, stream=self.stream)
        elif rule == "irn_iso":
            self.h.irn_weights_iso(xstar, self.cfg.tau, self.wx, self.wy, stream=self.stream)
        elif rule == "gazzola":
            self.h.gazzola_weights(xstar, self.cfg.p, self.Dx, self.Dy, self.wx, self.wy,
                                   stream=self.stream)
        else:
            raise ValueError(f"unknown weight rule {rule!r}")
        self.h.set_weights(self.wx, self.wy, stream=self.stream)
        self.cur_w = (self.wx, self.wy)

    # ---- on-disk state of the nested solve between outer steps (checkpoint /
    # hand-off). What outer step k+1 needs from step k (Alg. 5): the weights
    # W_{k+1} (and W_k for eq:delta, D_k under Gazzola's rule), X^(k), G^(k), V_i1, x*.
    _STATE_TENSORS = ("X_prev", "G_prev", "V_i1", "xstar")

    def save_state(self, path: str, k_next: int, st: dict, lstars=()) -> None:
        """Writes the state from which outer step `k_next` starts (after next_weights)."""
        cpu = lambda t: None if t is None else t.detach().cpu()
        blob = {"format": 1, "config": self.cfg.name, "N": self.N, "M": self.M, "k_next": int(k_next),
                "gamma": np.asarray(self.gamma, dtype=np.float64), "lstars": [int(x) for x in lstars],
                "prev_iters": None if st.get("prev_iters") is None else np.asarray(st["prev_iters"]),
                "W_cur": tuple(cpu(t) for t in self.cur_w),
                "W_prev": None if st.get("W_prev") is None else tuple(cpu(t) for t in st["W_prev"]),
                "D": tuple(cpu(t) for t in (self.Dx, self.Dy)) if hasattr(self, "Dx") else None}
        for name in self._STATE_TENSORS:
            blob[name] = cpu(st.get(name))
        tmp = path + ".tmp"
        torch.save(blob, tmp)
        os.replace(tmp, path)

    def load_state(self, path: str) -> tuple[int, dict, list]:
        """Adopts a saved state (weights into the handle) and returns (k_next, st, l* so far).
        set_data must have been called with the same data; refuses another problem."""
        blob = torch.load(path, map_location="cpu", weights_only=False)
        if blob.get("format") != 1 or blob["N"] != self.N or blob["M"] != self.M or \
                not np.array_equal(blob["gamma"], np.asarray(self.gamma, dtype=np.float64)):
            raise ValueError(f"{path}: state of another problem (config {blob.get('config')!r}, "
                             f"N = {blob.get('N')}, M = {blob.get('M')})")
        dev = self.wx.device
        self.wx.copy_(blob["W_cur"][0])
        self.wy.copy_(blob["W_cur"][1])
        self.h.set_weights(self.wx, self.wy, stream=self.stream)
        self.cur_w = (self.wx, self.wy)
        if blob["D"] is not None:   # Gazzola's rule: D_k
            self.Dx, self.Dy = blob["D"][0].to(dev), blob["D"][1].to(dev)
        st = {name: (None if blob[name] is None else blob[name].to(dev)) for name in self._STATE_TENSORS}
        st = {k_: v for k_, v in st.items() if v is not None}
        if blob["prev_iters"] is not None:
            st["prev_iters"] = blob["prev_iters"]
        if blob["W_prev"] is not None:
            st["W_prev"] = tuple(t.to(dev) for t in blob["W_prev"])
            self.w_prev = st["W_prev"]
        return int(blob["k_next"]), st, list(blob["lstars"])

    def run(self, K_out: int | None = None, checkpoint: str | None = None, resume: str | None = None):
        """The whole nested solve: up to K_out outer steps from W_0 = I; with
        cfg.stop == "lstar3" it also stops once l* is the same for three consecutive
        steps. checkpoint: a file rewritten (atomically) after every outer step
        with the state the next step starts from; resume: such a file to continue from
        (the returned list then holds the remaining steps only)."""
        K = K_out or self.cfg.K_out
        settle = getattr(self.cfg, "stop", "fixed") == "lstar3"
        if resume:
            k0, st, lst = self.load_state(resume)
        else:
            self.reset_weights()
            k0, st, lst = 0, {}, []
        outs = []
        for k in range(k0, K):
            o, st = self.outer_step(k, st)
            outs.append(o)
            lst.append(int(o.lstar))
            if settle and len(lst) >= 3 and len(set(lst[-3:])) == 1:
                break
            if k + 1 < K:
                self.next_weights(st["xstar"])
                st["W_prev"] = self.w_prev
                if checkpoint and self.dist.rank == 0:   # every rank holds the full state
                    self.save_state(checkpoint, k + 1, st, lst)
        self.final = st
        return outs
