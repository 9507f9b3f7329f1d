"""Per-pass timing of the nine-point sweep (N3) and the eikonal pass (N4) on config 3's grid
(4096^2, 64 x 64 boxes), as bench.py's secondary lines measure them."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding as B, gen  # noqa: E402


def main():
    import torch
    n = 4096
    g9 = B.Grid(2, (n, n), B.COEF_FACES).decompose((64, 64))
    g9.set_faces_global([np.full(tuple(reversed((n + (a == 0), n + (a == 1)))), 4.0) for a in range(2)])
    g9.set_diagonals(np.ones((n + 1, n + 1)), np.ones((n + 1, n + 1)))
    g9.set_vector(B.B, gen.uniform_field(0, gen.STREAM_RHS, (n, n)))
    g9.sor_sweep([1.0], 3, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g9.sor_sweep([1.0], 20, 3)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"sweep9 4096^2: {ms:.3f} ms/sweep, {n * n / ms / 1e6:.2f} GLUP/s, {56 * n * n / ms / 1e6 / 6536.4:.3f} of HBM")
    del g9
    ge = B.Grid(2, (n, n)).decompose((64, 64)).set_slowness(0.5 + gen.uniform_field(0, gen.STREAM_TEST, (n, n)) ** 2, 1.0 / n)
    u0 = np.full((n, n), np.inf)
    u0[n // 3, n // 2] = 0.0
    ge.set_vector(B.X, u0)
    ge.eikonal_sweep(2, 0)
    torch.cuda.synchronize()
    e0.record()
    ge.eikonal_sweep(8, 2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 8
    print(f"eikonal 4096^2: {ms:.3f} ms/pass, {n * n / ms / 1e6:.2f} GLUP/s, {24 * n * n / ms / 1e6 / 6536.4:.3f} of HBM")
    import time
    t0 = time.perf_counter()
    ph = 10
    while ge.eikonal_changes() > 0 and ph < 4000:
        ph = ge.eikonal_sweep(8, ph)
    print(f"eikonal fixed point: {ph} passes, {time.perf_counter() - t0:.3f} s")
    torch.cuda.synchronize()
    e0.record()
    ge.eikonal_sweep(8, ph)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 8
    print(f"eikonal all reached: {ms:.3f} ms/pass, {n * n / ms / 1e6:.2f} GLUP/s, {24 * n * n / ms / 1e6 / 6536.4:.3f} of HBM")


if __name__ == "__main__":
    main()
