"""Shift indices of an outer step (1-based), readings G11 / G34 / G36 of DESIGN.md:
Example 1's choices (§8.2: M = 20, i2 = i* = 10, I = J_L = 15, J_R = 19,
l_c = 18) scaled to M shifts: i2 = i* = floor(M/2), I = round(3M/4), J_L = I, J_R = M - 1,
l_c = round(9M/10) clamped to [1, M], ties to even; I_L = i*, I_R = floor((I + M + 2)/2).
Config.idx overrides (i2, i*, I, J_L, J_R, l_c) (Example 2).
Integer arithmetic only (independent of the oracle's float rounding)."""
from __future__ import annotations

import dataclasses


def _round_frac(num: int, den: int) -> int:
    """round(num / den), ties to the even integer, for num, den >= 0."""
    q, r = divmod(num, den)
    if 2 * r > den or (2 * r == den and q % 2 == 1):
        q += 1
    return q


@dataclasses.dataclass(frozen=True)
class ShiftIndices:
    i1: int
    i2: int
    istar: int
    I_split: int
    J_L: int
    J_R: int
    l_c: int
    I_L: int
    I_R: int


def shift_indices(cfg) -> ShiftIndices:
    M = cfg.M
    o = tuple(getattr(cfg, "idx", ()) or ())
    if o:
        i2, ist, isp, jl, jr, lc = (int(v) for v in o)
    else:
        i2 = ist = M // 2
        isp = _round_frac(3 * M, 4)
        jl, jr = isp, M - 1
        lc = min(M, max(1, _round_frac(9 * M, 10)))
    return ShiftIndices(1, i2, ist, isp, jl, jr, lc, ist, (isp + M + 2) // 2)
