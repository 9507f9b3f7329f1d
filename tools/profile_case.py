"""Small driver for ncu / timing experiments: a few decomposed sweeps on one config.

    python tools/profile_case.py --n 4096 --tile 64 [--faces] [--sweeps 4] [--dim 2]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1008_3699_b200 import binding, gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--tile", type=int, nargs="+", default=[64])
    ap.add_argument("--faces", action="store_true")
    ap.add_argument("--sweeps", type=int, default=4)
    ap.add_argument("--pcg", action="store_true")
    ap.add_argument("--maxit", type=int, default=20000)
    ap.add_argument("--pc", type=int, default=2, help="0 none, 1 SSOR, 2 ILU(0)")
    args = ap.parse_args()
    import torch
    d = args.dim
    n = [args.n] * d
    tile = (args.tile * d)[:d]
    kind = binding.COEF_FACES if args.faces else binding.COEF_POISSON
    g = binding.Grid(d, n, kind).decompose(tile)
    shape = tuple(reversed(n))
    if args.faces:
        ring = tuple(v + 2 for v in reversed(n))
        k = gen.lognormal_k(0, ring, 1.0)
        pad = [(0, 0)] * d
        pad[0] = (1, 1)
        g.set_coefficients_k(np.pad(k, pad, constant_values=1.0), (1.0, 0.1, 0.01)[:d] if d == 3 else (1.0,) * d)
    b = gen.uniform_field(0, gen.STREAM_RHS, shape) / float((args.n + 1) ** 2)
    g.set_vector(binding.B, b)
    if args.pcg:
        t = time.time()
        it, rel, ok = g.pcg_solve(args.pc, 1.0, 0, 1e-8, args.maxit)
        print("pcg", it, rel, ok, time.time() - t)
        return
    torch.cuda.synchronize()
    ph = 0
    for _ in range(2):
        ph = g.sor_sweep([1.0], 1, ph)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    ph = g.sor_sweep([1.0], args.sweeps, ph)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.sweeps
    N = int(np.prod(n))
    print(f"dim={d} n={args.n} tile={tile} faces={args.faces}: {ms:.4f} ms/sweep, {N / ms / 1e6:.2f} GLUP/s")
    g.check()


if __name__ == "__main__":
    main()
