"""Driver for ncu captures of the N3 / N4 kernels on config 3's grid (4096^2, 64 x 64 boxes):
    python tools/prof_next.py nine      -- a few nine-point sweeps (bench.py's Mehrstellen case)
    python tools/prof_next.py eik       -- eikonal passes once every box is reached (the fixed point)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding as B, gen  # noqa: E402


def main():
    import torch
    n = 4096
    if sys.argv[1] == "nine":
        g9 = B.Grid(2, (n, n), B.COEF_FACES).decompose((64, 64))
        g9.set_faces_global([np.full(tuple(reversed((n + (a == 0), n + (a == 1)))), 4.0) for a in range(2)])
        g9.set_diagonals(np.ones((n + 1, n + 1)), np.ones((n + 1, n + 1)))
        g9.set_vector(B.B, gen.uniform_field(0, gen.STREAM_RHS, (n, n)))
        g9.sor_sweep([1.0], 4, 0)
    else:
        ge = B.Grid(2, (n, n)).decompose((64, 64)).set_slowness(0.5 + gen.uniform_field(0, gen.STREAM_TEST, (n, n)) ** 2, 1.0 / n)
        u0 = np.full((n, n), np.inf)
        u0[n // 3, n // 2] = 0.0
        ge.set_vector(B.X, u0)
        ph = ge.eikonal_sweep(8, 0)
        while ge.eikonal_changes() > 0 and ph < 4000:
            ph = ge.eikonal_sweep(8, ph)
        ge.eikonal_sweep(2, ph)
        print("passes", ph)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
