"""Relaxation-factor search harness driven by the
oracle as the iteration counter (-m "not gpu").  The paper's printed optima are the pins: its
search must land on them (to its stated 1e-3 accuracy) with the printed iteration counts."""
import math

from oracle.model import run_lex
from paper_1008_3699_b200 import omega as OM


def lrsor(v):
    return run_lex(1, 41, [v[0]], [0], 1e-3)[0]


def test_refine_search_finds_the_papers_lrsor_optimum():
    # LRSOR at R = 41 needs 51 iterations at its optimum omega_L = 1.86887
    w, c = OM.refine_search(lrsor, 1.0, 2.0, accuracy=1e-3, coarse=0.1)
    assert c == 51
    assert abs(w - 1.86887) <= 1e-3


def test_grid_search_argmin_contains_the_papers_value():
    w, c, table = OM.grid_search(lrsor, 1.860, 1.880, 1e-3)
    assert c == 51 and table[1.869] == 51
    assert all(v is None or v >= 51 for v in table.values())


def test_coordinate_search_reaches_the_papers_ssour_count():
    # SSOUR (omega_L, omega_R) = (0.24825, 1.87087) -> 58 iterations
    cnt = lambda v: run_lex(1, 41, list(v), [0, 1], 1e-3)[0]  # noqa: E731
    vec, c = OM.coordinate_search(cnt, [0.25, 1.87], 0.0, 2.0, accuracy=1e-3, coarse=0.1, rounds=2)
    assert c == 58
    assert abs(vec[1] - 1.87087) < 5e-3


def test_search_treats_divergence_as_worst_and_breaks_ties_low():
    def cnt(v):
        w = v[0]
        if w > 1.5:
            return None                      # "did not converge"
        return 10 if abs(w - 1.2) < 0.051 else 20
    w, c, table = OM.grid_search(cnt, 1.0, 2.0, 0.05)
    assert c == 10 and math.isclose(w, 1.15)
    assert table[1.55] is None
    # one component of a vector, the others fixed
    w2, c2, _ = OM.grid_search(lambda v: int(abs(v[1] - 0.7) * 100) + int(v[0] * 0), 0.0, 1.0, 0.1, [1.0, 0.0], 1)
    assert math.isclose(w2, 0.7) and c2 == 0


def test_omega_opt_poisson():
    assert math.isclose(OM.omega_opt_poisson(256), 2.0 / (1.0 + math.sin(math.pi / 257)))
