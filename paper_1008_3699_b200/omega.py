"""Relaxation-factor search: per-direction omega and the brute-force search the
paper uses to find its "optimal" factors ("searching in [1.0, 2.0] with 1.e-3 accuracy",
PAPER:1996-1998; the over/under-relaxation pairs of SSOUR / PSOUR searched in [0, 2],
PAPER:2087-2095).

The search is host logic around a counting function ``count(omega) -> iterations or None``
(None = did not converge).  ``sweeps_to_tol`` is the counting function over the library's
decomposed SOR sweep (GPU); the tests also drive the search with the oracle as the counter.
The library's sweep already takes one omega per direction (2^d values indexed by the box's
start bits, DESIGN R-6), so the per-direction variants need no other device code.
"""
from __future__ import annotations

import math
from typing import Callable, Dict, List, Optional, Sequence, Tuple

Count = Callable[[Sequence[float]], Optional[int]]


def sweeps_to_tol(grid, omega: Sequence[float], tol: float = 1e-8, maxit: int = 20000, check_every: int = 10,
                  phase0: int = 0, x0=None) -> Optional[int]:
    """Decomposed SOR sweeps (library, GPU) from x0 (default 0) until the relative residual
    ||b - A x|| / ||b|| < tol, checked every `check_every` sweeps; None if maxit is reached.
    `omega` is one value or 2^d per-direction values (sw_sor_sweep)."""
    import numpy as np

    from . import binding
    shape = tuple(int(v) for v in reversed(grid.n_local))
    grid.set_vector(binding.X, np.zeros(shape) if x0 is None else x0)
    ph, n = phase0, 0
    while n < maxit:
        ph = grid.sor_sweep(list(omega), check_every, ph)
        n += check_every
        r = grid.residual_norm()
        if not math.isfinite(r):
            return None
        if r < tol:
            return n
    return None


def _key(c: Optional[int]) -> float:
    return math.inf if c is None else float(c)


def grid_search(count: Count, lo: float, hi: float, step: float, fixed: Sequence[float] = (), index: int = 0
                ) -> Tuple[float, Optional[int], Dict[float, Optional[int]]]:
    """Brute force over omega = lo, lo + step, ... <= hi for component `index` of the omega vector
    (the other components from `fixed`).  Returns (smallest minimiser, its count, all counts)."""
    table: Dict[float, Optional[int]] = {}
    n = int(math.floor((hi - lo) / step + 1e-9)) + 1
    best_w, best_c = None, None
    for t in range(n):
        w = round(lo + t * step, 12)
        vec = list(fixed)
        if not vec:
            vec = [w]
        else:
            vec[index] = w
        c = count(vec)
        table[w] = c
        if best_w is None or _key(c) < _key(best_c):
            best_w, best_c = w, c
    return best_w, best_c, table


def refine_search(count: Count, lo: float, hi: float, accuracy: float = 1e-3, coarse: float = 0.1,
                  fixed: Sequence[float] = (), index: int = 0) -> Tuple[float, Optional[int]]:
    """Coarse-to-fine search to `accuracy`: a grid of step `coarse` on [lo, hi], then grids ten times
    finer on [best - step, best + step] until the step reaches `accuracy`."""
    step = coarse
    a, b = lo, hi
    best_w, best_c, _ = grid_search(count, a, b, step, fixed, index)
    while step > accuracy * (1 + 1e-9):
        nstep = max(step / 10.0, accuracy)
        a, b = max(lo, best_w - step), min(hi, best_w + step)
        w, c, _ = grid_search(count, a, b, nstep, fixed, index)
        if _key(c) < _key(best_c) or (_key(c) == _key(best_c) and w < best_w):
            best_w, best_c = w, c
        step = nstep
    return best_w, best_c


def coordinate_search(count: Count, start: Sequence[float], lo: float, hi: float, accuracy: float = 1e-3,
                      coarse: float = 0.1, rounds: int = 3) -> Tuple[List[float], Optional[int]]:
    """Per-direction factors (e.g. the (omega_L, omega_R) pairs of SSOUR): refine one
    component at a time, keeping the others, until a round brings no improvement."""
    vec = list(start)
    best_c = count(vec)
    for _ in range(rounds):
        improved = False
        for i in range(len(vec)):
            w, c = refine_search(count, lo, hi, accuracy, coarse, vec, i)
            if _key(c) < _key(best_c):
                vec[i], best_c, improved = w, c, True
        if not improved:
            break
    return vec, best_c


def omega_opt_poisson(n: int) -> float:
    """Young's optimum for lexicographic SOR on the n^d-interior-node Poisson problem, h = 1/(n+1)."""
    return 2.0 / (1.0 + math.sin(math.pi / (n + 1)))
