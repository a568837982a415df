"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no convolution, no gradient,
no solver step). It only draws the problem's raw ingredients from a seeded
generator so that `oracle/` and `paper_2306_15049_b200/` see the same bytes:

* x_true  -- piecewise-constant phantom (rectangles / discs, values U[0,1)),
             the edge-rich natural-image surrogate of PAPER.md §2.1
* psf     -- (2r+1)^2 Gaussian point-spread function normalised to sum 1,
             centred, the "symmetric, Gaussian blur" of §8.2
* xi      -- raw N(0, I) draw; each side scales it to the configured noise
             level itself (d = Cx + nu*||Cx|| xi/||xi||)
* gamma   -- the shift ladder, log-evenly spaced, ascending

Recipe: SURVEY.md §8(d) d1 (seed = 230615049 + config index, PCG64).
The per-config sizes follow BASELINE.json `configs` (C1..C5); readings of the
values BASELINE.json leaves open are the G-list of SURVEY.md §8(c), repeated
in DESIGN.md.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED_BASE = 230615049


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    index: int            # 1-based config index (C1..C5)
    n: int                # image is n x n, N = n*n
    M: int                # number of shifts
    gamma_lo: float
    gamma_hi: float
    r: int                # PSF half width, PSF is (2r+1)^2
    sigma: float
    noise: float          # relative noise level nu
    n_c: int              # principal recycle-space cap
    J: int                # Ritz vectors per shift group (|J|)
    K_out: int            # outer IRN steps
    tau: float            # IRN smoothing
    tol: float            # CG relative residual tolerance
    shapes: str           # phantom recipe key
    n_shapes: int
    maxit: int = 100000        # reading G14: C4 at k >= 1 (tau = 1e-4) needs > 20000 at gamma = 100
    weight_rule: str = "irn"   # outer weight update: "irn" (north_star), "irn_iso", "gazzola" (f1)
    p: float = 2.0             # Gazzola exponent (never given by the paper; SPEC S:421 default)
    stop: str = "fixed"        # outer stopping: "fixed" (K_out steps) or "lstar3"
    guess: str = "orth"        # principal guesses: "orth" (eq:orthupdate), "oblique" (one anchor,
                               # eq:obliqueupdate) or "oblique2" (two anchors, eq:updates) -- f2(iii)
    inner: str = "cg"          # inner solver: "cg" (north_star's recycled CG, reading G1) or
                               # "minres" (the paper's recycling MINRES, eq:minShift) -- f2(ii)
    local: str = "d3"          # local spaces: "d3" ([W, g^(k-1,l)], shift-independent, reading D3)
                               # or "seq" ([W, g^(k-1,l), g^(k,l-1)], Alg. 3/4; needs inner
                               # "minres", solved as a wavefront down each group) -- f2(i)
    principal: str = "g10"     # k >= 1 principal block: "g10" ([V_i1, X^(k-1)], reading G10) or
                               # "vnew" ([V_i1, V^(new), X^(k-1)], eq:delta / eq:tildeUupdate) -- f3
    operator: str = "blur"     # C: "blur" (Gaussian PSF, Example 1) or "ct" (parallel-beam Radon
                               # matrix, Example 2 P:1083-1098) -- SURVEY §8(f) f4
    n_angles: int = 0          # CT: projection angles 1, 2, ..., n_angles degrees
    idx: tuple = ()            # index overrides (i2, i*, I, J_L, J_R, l_c), 1-based; () = rules G11/G36
    psf_terms: tuple = ()      # rank-2 PSF of Example 1: ((band_x, sigma_x, band_y,
                               # sigma_y), ...) per Kronecker term; () = one Gaussian (r, sigma)

    @property
    def N(self) -> int:
        return self.n * self.n

    @property
    def ndet(self) -> int:
        """CT detector bins (reading G38): 2 ceil(n / sqrt 2) + 2 bins of unit width
        centred on the rotation axis (every ray of every angle through the image is
        sampled; an even count puts the bins at half-integer offsets, off the pixel
        grid lines of the axis-parallel angles)."""
        return 2 * math.ceil(self.n / math.sqrt(2.0)) + 2

    @property
    def ndata(self) -> int:
        """Length of the data vector d: N for the blur, n_angles * ndet for CT."""
        return self.n_angles * self.ndet if self.operator == "ct" else self.N


CONFIGS = {
    "C1": Config("C1", 1, 32, 8, 1e-4, 1.0, 4, 1.5, 0.01, 10, 2, 3, 1e-3, 1e-8, "rects", 6),
    "C2": Config("C2", 2, 256, 32, 1e-5, 10.0, 4, 2.0, 0.01, 40, 8, 5, 1e-3, 1e-8, "rects", 20),
    "C3": Config("C3", 3, 512, 64, 1e-6, 10.0, 7, 3.0, 0.02, 60, 10, 6, 1e-3, 1e-8, "rects+discs", 60),
    "C4": Config("C4", 4, 1024, 128, 1e-6, 100.0, 7, 4.0, 0.01, 80, 12, 8, 1e-4, 1e-8, "alternate", 200),
    "C5": Config("C5", 5, 4096, 16, 1e-5, 10.0, 10, 5.0, 0.01, 40, 8, 4, 1e-3, 1e-8, "alternate", 2000),
    # Example 2: n = 82, angles 1..135 degrees, C with unit
    # Frobenius norm, 1 % noise, 20 lambda log-spaced in [1e-4, 1e1] (gamma = lambda^2),
    # i1 = 1, i2 = 10, gamma_* = 12th, I = 16, l_c = 19, J_L = 15, J_R = 19;
    # 9 outer steps; n_c, |J|, tau, tol as C2 (readings G38)
    "C6": Config("C6", 6, 82, 20, 1e-8, 1e2, 0, 0.0, 0.01, 40, 8, 9, 1e-3, 1e-8, "alternate", 16,
                 operator="ct", n_angles=135, idx=(10, 12, 16, 15, 19, 19)),
    # Example 1 (§8.2, reading G40): 128 x 128, rank-2 blur
    # C = sum_{i=1,2} C_i^(1) (x) C_i^(2), Toeplitz bandwidths 8, 7, 12, 4 and sigma 3, 5/2,
    # 4, 2 (C_i^(1) along x, C_i^(2) along y; bandwidth b = half-width b - 1, Regtools'
    # blur), 0.5 % noise, 20 lambda log-spaced in [1e-4, 10^2.5] (gamma = lambda^2), I = 15,
    # i1 = 1, i2 = i* = 10, J_L = 15, J_R = 19, l_c = 18, 12 local Ritz vectors, principal
    # space 100 + 50 Ritz vectors + 2 solutions (n_c = 152), inner relres 1e-6,
    # the paper's own method: recycling MINRES, sequential local spaces, V^(new), Gazzola's
    # weights, stop on 3 equal l* (at most 11 outer steps)
    "C7": Config("C7", 7, 128, 20, 1e-8, 10.0 ** 5, 11, 0.0, 0.005, 152, 12, 11, 1e-3, 1e-6, "rects", 20,
                 weight_rule="gazzola", stop="lstar3", inner="minres", local="seq", principal="vnew",
                 idx=(10, 10, 15, 15, 19, 18), psf_terms=((8, 3.0, 7, 2.5), (12, 4.0, 4, 2.0))),
}


def kronecker_psf(terms) -> np.ndarray:
    """h = sum_i u_i v_i^T / total for Toeplitz factors with Regtools' blur shape (band b:
    entries exp(-k^2 / (2 sigma^2)) for |k| <= b - 1): v_i along x (columns, C_i^(1)),
    u_i along y (rows, C_i^(2)); centred in the (2r+1)^2 window, r = max band - 1, sum 1."""
    r = max(max(bx, by) for bx, _, by, _ in terms) - 1
    a = np.arange(-r, r + 1, dtype=np.float64)
    h = np.zeros((2 * r + 1, 2 * r + 1))
    for bx, sx, by, sy in terms:
        v = np.where(np.abs(a) <= bx - 1, np.exp(-a ** 2 / (2.0 * sx * sx)), 0.0)
        u = np.where(np.abs(a) <= by - 1, np.exp(-a ** 2 / (2.0 * sy * sy)), 0.0)
        h += np.outer(u, v)
    return h / h.sum()


def small_config(n: int = 16, M: int = 6, r: int = 2, sigma: float = 1.0, n_c: int = 8,
                 J: int = 2, K_out: int = 2, name: str = "tiny", n_shapes: int = 4,
                 gamma_lo: float = 1e-3, gamma_hi: float = 1.0, tau: float = 1e-3,
                 tol: float = 1e-10, noise: float = 0.01) -> Config:
    """A tiny configuration with the C1 recipe, for oracle pins and fast parity."""
    return Config(name, 1, n, M, gamma_lo, gamma_hi, r, sigma, noise, n_c, J, K_out,
                  tau, tol, "rects", n_shapes)


def rng_for(cfg: Config) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + cfg.index))


def _shape_params(cfg: Config):
    n = cfg.n
    if cfg.shapes in ("rects", "rects+discs"):
        s = (math.ceil(n / 16), math.ceil(n / 4))
        q = (math.ceil(n / 32), math.ceil(n / 8))
    else:  # "alternate" (C4, C5)
        if n <= 1024:
            s = (math.ceil(n / 64), math.ceil(n / 8))
            q = (math.ceil(n / 128), math.ceil(n / 16))
        else:
            s = (math.ceil(n / 256), math.ceil(n / 16))
            q = (math.ceil(n / 512), math.ceil(n / 32))
    return s, q


def phantom(cfg: Config, rng: np.random.Generator) -> np.ndarray:
    """Piecewise-constant phantom, later shapes overwrite earlier ones."""
    n = cfg.n
    x = np.zeros((n, n), dtype=np.float64)
    (s_lo, s_hi), (q_lo, q_hi) = _shape_params(cfg)
    s_hi = min(s_hi, n)
    if cfg.shapes == "rects":
        kinds = ["rect"] * cfg.n_shapes
    elif cfg.shapes == "rects+discs":
        kinds = ["rect"] * 50 + ["disc"] * 10
    else:
        kinds = ["rect" if k % 2 == 0 else "disc" for k in range(cfg.n_shapes)]
    ii, jj = np.mgrid[0:n, 0:n]
    for kind in kinds:
        val = rng.random()
        if kind == "rect":
            h = int(rng.integers(s_lo, s_hi + 1))
            w = int(rng.integers(s_lo, s_hi + 1))
            i0 = int(rng.integers(0, n - h + 1))
            j0 = int(rng.integers(0, n - w + 1))
            x[i0:i0 + h, j0:j0 + w] = val
        else:
            q = int(rng.integers(q_lo, q_hi + 1))
            ci = int(rng.integers(q, n - q))
            cj = int(rng.integers(q, n - q))
            i_a, i_b = max(0, ci - q), min(n, ci + q + 1)
            j_a, j_b = max(0, cj - q), min(n, cj + q + 1)
            sub = (ii[i_a:i_b, j_a:j_b] - ci) ** 2 + (jj[i_a:i_b, j_a:j_b] - cj) ** 2 <= q * q
            x[i_a:i_b, j_a:j_b][sub] = val
    return x


def gaussian_psf(r: int, sigma: float) -> np.ndarray:
    """h[a+r, b+r] proportional to exp(-(a^2+b^2)/(2 sigma^2)), sum(h) = 1."""
    a = np.arange(-r, r + 1, dtype=np.float64)
    h = np.exp(-(a[:, None] ** 2 + a[None, :] ** 2) / (2.0 * sigma * sigma))
    return h / h.sum()


def gamma_ladder(cfg: Config) -> np.ndarray:
    """gamma_l = 10^(log10 lo + (l-1)(log10 hi - log10 lo)/(M-1)), ascending."""
    lo, hi = math.log10(cfg.gamma_lo), math.log10(cfg.gamma_hi)
    if cfg.M == 1:
        return np.array([cfg.gamma_lo])
    return np.array([10.0 ** (lo + l * (hi - lo) / (cfg.M - 1)) for l in range(cfg.M)])


def make_inputs(cfg: Config) -> dict:
    """All seeded raw inputs of one configuration (fp64, C-contiguous)."""
    rng = rng_for(cfg)
    x_true = phantom(cfg, rng)
    if cfg.operator == "ct":
        xi = rng.standard_normal(cfg.ndata)       # noise in the sinogram (data) space
        return {"x_true": np.ascontiguousarray(x_true), "psf": None, "xi": xi,
                "gamma": gamma_ladder(cfg),
                "angles": np.arange(1, cfg.n_angles + 1, dtype=np.float64)}
    xi = rng.standard_normal((cfg.n, cfg.n))
    return {
        "x_true": np.ascontiguousarray(x_true),
        "psf": kronecker_psf(cfg.psf_terms) if cfg.psf_terms else gaussian_psf(cfg.r, cfg.sigma),
        "xi": np.ascontiguousarray(xi),
        "gamma": gamma_ladder(cfg),
    }


def random_vectors(seed: int, shape, dist: str = "normal") -> np.ndarray:
    """Seeded test vectors (parity cases, not part of any workload)."""
    g = np.random.Generator(np.random.PCG64(seed))
    if dist == "normal":
        return g.standard_normal(shape)
    if dist == "uniform":
        return g.random(shape)
    raise ValueError(dist)


def random_weights(seed: int, n: int, lo: float = 0.1, hi: float = 1000.0) -> tuple:
    """Bimodal positive weight planes with zero pads, the shape IRN weights take
    (about 1/tau on flats, about 1/|jump| on edges; SURVEY d1 'value structure')."""
    g = np.random.Generator(np.random.PCG64(seed))
    wx = np.exp(g.uniform(math.log(lo), math.log(hi), (n, n)))
    wy = np.exp(g.uniform(math.log(lo), math.log(hi), (n, n)))
    wx[:, n - 1] = 0.0
    wy[n - 1, :] = 0.0
    return wx, wy
