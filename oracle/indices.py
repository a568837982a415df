"""Shift indices of the outer step (TEST INFRASTRUCTURE: part of the oracle; only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import it).

The paper fixes them only for its two examples (1-based):
  Example 1 (§8.2, M = 20): i1 = 1, i2 = 10, i* = 10, I = 15 (the left group is
    the smallest 15 shifts), J_L = 15, J_R = 19, l_c = 18;
  Example 2 (§8.3, M = 20): i1 = 1, i2 = 10, gamma_* the 12th, I = 16, l_c = 19,
    J_L = 15, J_R = 19.
For other ladder lengths we scale Example 1 (reading G11 / G36): i1 = 1,
i2 = i* = M/2 (integer division), I = round(0.75 M), J_L = I, J_R = M - 1,
l_c = round(0.9 M); round() is Python's (ties to the even integer).  Config.idx, when set,
gives (i2, i*, I, J_L, J_R, l_c) explicitly (C6 = Example 2).
The anchors of the two-anchor oblique guesses (eq:updates P:1000-1005, reading G34):
I_L = i*, I_R = the middle of the right group, (I + 1 + M + 1) // 2.
"""
from __future__ import annotations

import dataclasses


@dataclasses.dataclass(frozen=True)
class Indices:
    i1: int
    i2: int
    istar: int
    I: int
    J_L: int
    J_R: int
    l_c: int
    I_L: int
    I_R: int


def indices(M: int, idx: tuple = ()) -> Indices:
    if idx:
        i2, istar, I, J_L, J_R, l_c = idx
    else:
        i2 = M // 2
        istar = M // 2
        I = int(round(0.75 * M))
        J_L = I
        J_R = M - 1
        l_c = max(1, min(M, int(round(0.9 * M))))
    return Indices(1, i2, istar, I, J_L, J_R, l_c, istar, (I + 1 + M + 1) // 2)


def of(cfg) -> Indices:
    return indices(cfg.M, tuple(getattr(cfg, "idx", ()) or ()))
