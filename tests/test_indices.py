"""Pins of the shift-index readings (G11 / G34 / G36) -- oracle/indices.py
against the values the paper prints and the survey's table, and the library-side
paper_2306_15049_b200/indices.py (independent integer code) against the oracle."""
import types

import pytest

import rsk_synth as S
from oracle.indices import indices, of
from paper_2306_15049_b200.indices import shift_indices


def _tup(ix):
    return (ix.i1, ix.i2, ix.istar, ix.I, ix.J_L, ix.J_R, ix.l_c)


def test_example1_values_printed_by_the_paper():
    """§8.2: M = 20, I = 15, i1 = 1, i2 = 10, i* = 10, J_L = 15, J_R = 19,
    l_c = 18 -- the G11 / G36 rules reproduce every one of them."""
    assert _tup(indices(20)) == (1, 10, 10, 15, 15, 19, 18)


def test_example2_override_printed_by_the_paper():
    """§8.3: i1 = 1, i2 = 10, gamma_* the 12th, I = 16, l_c = 19, J_L = 15,
    J_R = 19 (config C6 carries them in Config.idx)."""
    ix = of(S.CONFIGS["C6"])
    assert _tup(ix) == (1, 10, 12, 16, 15, 19, 19)


@pytest.mark.parametrize("M,exp", [
    # (I, i2, J_L, J_R) per ladder length
    (8, (6, 4, 6, 7)), (16, (12, 8, 12, 15)), (32, (24, 16, 24, 31)),
    (64, (48, 32, 48, 63)), (128, (96, 64, 96, 127)),
])
def test_survey_g11_table(M, exp):
    ix = indices(M)
    assert (ix.I, ix.i2, ix.J_L, ix.J_R) == exp
    assert ix.istar == ix.i2 and ix.i1 == 1


def test_configs_indices():
    """(i2, i*, I, J_L, J_R, l_c) of every BASELINE config."""
    want = {"C1": (4, 4, 6, 6, 7, 7), "C2": (16, 16, 24, 24, 31, 29), "C3": (32, 32, 48, 48, 63, 58),
            "C4": (64, 64, 96, 96, 127, 115), "C5": (8, 8, 12, 12, 15, 14)}
    for name, w in want.items():
        ix = of(S.CONFIGS[name])
        assert (ix.i2, ix.istar, ix.I, ix.J_L, ix.J_R, ix.l_c) == w, name


def test_groups_partition_and_anchor_in_left_group():
    for M in range(8, 260):   # J_R = M - 1 can fall in the left group for M < 8 (M = 3: I = J_R = 2)
        ix = indices(M)
        assert 1 <= ix.istar <= ix.I <= M and 1 <= ix.J_L <= ix.I and ix.J_R <= M
        if ix.I < M:   # a non-empty right group holds J_R and I_R
            assert ix.I < ix.J_R and ix.I < ix.I_R <= M
        assert ix.I_L == ix.istar


def test_ties_round_to_even():
    """round(0.75 M) at M = 6 is 4.5 -> 4; round(0.9 M) at M = 5 is 4.5 -> 4, at 15 13.5 -> 14."""
    assert indices(6).I == 4 and indices(10).I == 8 and indices(5).l_c == 4 and indices(15).l_c == 14


def test_library_indices_match_oracle():
    for M in range(1, 520):
        a = indices(M)
        b = shift_indices(types.SimpleNamespace(M=M, idx=()))
        assert (a.i1, a.i2, a.istar, a.I, a.J_L, a.J_R, a.l_c, a.I_L, a.I_R) == \
               (b.i1, b.i2, b.istar, b.I_split, b.J_L, b.J_R, b.l_c, b.I_L, b.I_R), M
    c6 = S.CONFIGS["C6"]
    assert _tup(of(c6)) == (lambda b: (b.i1, b.i2, b.istar, b.I_split, b.J_L, b.J_R, b.l_c))(shift_indices(c6))
