"""Config 3 PCG probe (2D lognormal faces, 64 x 64 boxes): ILU(0)-PCG iterations and time per iteration."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding, gen  # noqa: E402


def main():
    import torch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
    g = binding.Grid(2, (n, n), binding.COEF_FACES).decompose((64, 64))
    k = gen.lognormal_k(0, (n + 2, n + 2), 1.0)
    g.set_coefficients_k(np.pad(k, [(1, 1), (0, 0)], constant_values=1.0), (1.0, 1.0))
    g.set_vector(binding.B, gen.uniform_field(0, gen.STREAM_RHS, (n, n)) / float((n + 1) ** 2))
    torch.cuda.synchronize()
    t = time.perf_counter()
    it, rel, ok = g.pcg_solve(binding.PC_ILU0, 1.0, binding.PAIR_SYMMETRIC, 1e-8, maxit)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"n={n} ilu0: it={it} ok={ok} {dt:.2f}s {dt / max(it, 1) * 1e3:.3f} ms/it")


if __name__ == "__main__":
    main()
