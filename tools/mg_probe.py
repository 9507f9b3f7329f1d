"""MG-PCG probe: iterations for a few (levels, nu, theta, coarse_scale) on a 2D / 3D problem."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding as B, gen  # noqa: E402


def run(dim, n, tile, law, settings):
    import torch
    nn = (n,) * dim
    g = B.Grid(dim, nn, B.COEF_FACES).decompose(tile)
    sig = 1.0 if dim == 2 else 0.5
    k = gen.lognormal_k(0, (n + 2,) * dim, sig)
    pad = [(0, 0)] * dim
    pad[0] = (1, 1)
    g.set_coefficients_k(np.pad(k, pad, constant_values=1.0), (1.0, 1.0) if dim == 2 or law == "iso" else (1.0, 0.1, 0.01))
    g.set_vector(B.B, gen.uniform_field(0, gen.STREAM_RHS, nn) / float((n + 1) ** 2))
    t = time.perf_counter()
    it, rel, ok = g.pcg_solve(B.PC_ILU0, 1.0, B.PAIR_SYMMETRIC, 1e-8, 20000)
    torch.cuda.synchronize()
    print(f"dim={dim} n={n} {law} ILU0: it={it} {time.perf_counter() - t:.3f}s")
    for (lv, nu, th, nc, sc) in settings:
        g.mg_setup(lv, nu, th, nc, sc)
        t = time.perf_counter()
        it, rel, ok = g.pcg_solve(B.PC_MG, 1.0, B.PAIR_SYMMETRIC, 1e-8, 20000)
        torch.cuda.synchronize()
        print(f"   MG levels={lv} nu={nu} theta={th} nc={nc} scale={sc}: it={it} ok={ok} {time.perf_counter() - t:.3f}s")


if __name__ == "__main__":
    S = [(4, 1, 0.5, 16, 1.0), (4, 1, 0.5, 16, 1.5), (4, 1, 0.6, 16, 1.8), (4, 2, 0.5, 16, 1.5), (5, 2, 0.6, 32, 1.5),
         (6, 2, 0.6, 64, 1.5)]
    run(2, 1024, (64, 64), "c3", S)
    run(3, 128, (32, 8, 4), "iso", S[:4])
    run(3, 128, (32, 8, 4), "c5", S[:4])
