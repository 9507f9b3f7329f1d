"""Config-3 kernel timings: 100 decomposed SOR sweeps (k_sweep2v) and ILU(0)-PCG per iteration."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding as B, gen  # noqa: E402
import bench  # noqa: E402


def main():
    import torch
    n = 4096
    g = B.Grid(2, (n, n), B.COEF_FACES).decompose((64, 64))
    k = gen.lognormal_k(0, (n + 2, n + 2), 1.0)
    g.set_coefficients_k(np.pad(k, [(1, 1), (0, 0)], constant_values=1.0), (1.0, 1.0))
    g.set_vector(B.B, gen.uniform_field(0, gen.STREAM_RHS, (n, n)) / float((n + 1) ** 2))
    for _ in range(3):
        ms = bench._time_sweeps(g, [1.0], 100)
        print(f"sweep2v: {ms * 1e3:.1f} us/sweep  {n * n / (ms * 1e-3) / 1e9:.1f} GLUP/s", flush=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    it, rel, ok = g.pcg_solve(B.PC_ILU0, 1.0, 0, 1e-8, 400)
    torch.cuda.synchronize()
    print(f"ILU-PCG 400 its: {1e3 * (time.perf_counter() - t) / it:.3f} ms/it")


if __name__ == "__main__":
    main()
