"""Oracle pins against the numbers the paper prints (-m "not gpu").

Model problem PAPER:1906-1934; readings R-1..R-3 of DESIGN.md (resolution counts the
boundary, 2D L1 normaliser 3R^2, one directional pass = one iteration).  Each expected
value is a table cell of PAPER.md (line numbers cited); tests/golden/paper_tables.txt
lists them with their citations.
"""
import pytest

from oracle.model import run_decomposed, run_lex


# Table "1D parallel Gauss-Seidel vs. 1D sequential Gauss-Seidel", R = 41
def test_1d_gs_sequential_rows():
    it, e = run_lex(1, 41, [1.0], [0], 1e-3)          # LRGS
    assert it == 979 and abs(e - 9.94266e-4) < 5e-10
    it, e = run_lex(1, 41, [1.0], [1], 1e-3)          # RLGS
    assert it == 960 and abs(e - 9.94266e-4) < 5e-10
    it, e = run_lex(1, 41, [1.0], [0, 1], 1e-3)       # SGS
    assert it == 976 and abs(e - 9.96647e-4) < 5e-10


@pytest.mark.parametrize("p,expected", [(2, 975), (4, 974), (6, 974), (8, 973), (10, 973), (14, 972)])
def test_1d_pgs_rows(p, expected):
    """PGS(p) rows PAPER:1977-1982: the decomposed sweep (balanced boxes, 2x2 coupled solves)."""
    it, _ = run_decomposed(1, 41, [p], [1.0], 1e-3)
    assert it == expected


def test_1d_sor_rows():
    """Table 1D SOR, R = 41 with the printed optimal omegas."""
    assert run_lex(1, 41, [1.86887], [0], 1e-3)[0] == 51            # LRSOR
    assert run_lex(1, 41, [1.86637], [1], 1e-3)[0] == 31            # RLSOR
    assert run_lex(1, 41, [1.0, 1.87776], [0, 1], 1e-3)[0] == 62    # SSOR (w_L, w_R)
    # the decomposed sweep with one box and the same (w_LR, w_RL) is the same SSOR
    assert run_decomposed(1, 41, [1], [1.0, 1.87776], 1e-3)[0] == 62


def test_1d_ssour_row():
    """Symmetric over/under-relaxation SSOUR, R = 41: per-direction factors
    (w_L, w_R) = (0.24825, 1.87087), 58 iterations (the sequential and the one-box decomposed
    sweep).  The PSOUR(p) rows of the same table are not reproduced."""
    assert run_lex(1, 41, [0.24825, 1.87087], [0, 1], 1e-3)[0] == 58
    assert run_decomposed(1, 41, [1], [0.24825, 1.87087], 1e-3)[0] == 58


def test_2d_rows_51():
    """2D tables at 51x51: GS RGS 1018, SGS 1006, FGS 1006 (frontal = one
    box on the paper's 4-direction cycle); SOR w=1.25 RSOR 616, SSOR 606,
    FSOR 605; SOR w=1.5 RSOR 348, FSOR 339."""
    it, e = run_lex(2, 51, [1.0], [0], 1e-3)
    assert it == 1018 and abs(e - 9.98560e-4) < 2e-9
    assert run_lex(2, 51, [1.0], [0, 3], 1e-3)[0] == 1006
    assert run_decomposed(2, 51, [1, 1], [1.0], 1e-3)[0] == 1006
    it, e = run_lex(2, 51, [1.25], [0], 1e-3)
    assert it == 616 and abs(e - 9.97982e-4) < 2e-9
    assert run_lex(2, 51, [1.25], [0, 3], 1e-3)[0] == 606
    assert run_decomposed(2, 51, [1, 1], [1.25], 1e-3)[0] == 605
    assert run_lex(2, 51, [1.5], [0], 1e-3)[0] == 348
    assert run_decomposed(2, 51, [1, 1], [1.5], 1e-3)[0] == 339


@pytest.mark.slow
def test_2d_rgs_101():
    """RGS at 101x101 = 4065."""
    assert run_lex(2, 101, [1.0], [0], 1e-3)[0] == 4065


def test_3d_rows_25():
    """3D tables at 25^3, stop 1e-2: GS RGS 110, SGS 104, FGS 104;
    SOR w=1.25 RSOR 69, SSOR 63; SOR w=1.5 RSOR 41,
    SSOR 36, FSOR 35.  (FSOR(1.25) = 62 at PAPER:2407 is not reproduced: 63 under every
    3D cycle order allowed by PAPER:781-807, R-5.)"""
    it, e = run_lex(3, 25, [1.0], [0], 1e-2)
    assert it == 110 and abs(e - 9.92078e-3) < 5e-9
    assert run_lex(3, 25, [1.0], [0, 7], 1e-2)[0] == 104
    assert run_decomposed(3, 25, [1, 1, 1], [1.0], 1e-2)[0] == 104
    assert run_lex(3, 25, [1.25], [0], 1e-2)[0] == 69
    assert run_lex(3, 25, [1.25], [0, 7], 1e-2)[0] == 63
    assert run_lex(3, 25, [1.5], [0], 1e-2)[0] == 41
    assert run_lex(3, 25, [1.5], [0, 7], 1e-2)[0] == 36
    assert run_decomposed(3, 25, [1, 1, 1], [1.5], 1e-2)[0] == 35
