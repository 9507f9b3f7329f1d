"""MG-PCG settings probe for config 3 (2D lognormal faces, 64 x 64 boxes): python tools/mg_probe2d.py n L,nu,theta,nc,s ..."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding as B, gen  # noqa: E402


def main():
    import torch
    n = int(sys.argv[1])
    g = B.Grid(2, (n, n), B.COEF_FACES).decompose((64, 64))
    k = gen.lognormal_k(0, (n + 2, n + 2), 1.0)
    g.set_coefficients_k(np.pad(k, [(1, 1), (0, 0)], constant_values=1.0), (1.0, 1.0))
    g.set_vector(B.B, gen.uniform_field(0, gen.STREAM_RHS, (n, n)) / float((n + 1) ** 2))
    for a in sys.argv[2:]:
        S = tuple(float(x) if '.' in x else int(x) for x in a.split(','))
        g.mg_setup(*S)
        torch.cuda.synchronize()
        t = time.perf_counter()
        it, rel, ok = g.pcg_solve(B.PC_MG, 1.0, 0, 1e-8, 20000)
        torch.cuda.synchronize()
        print(f"n={n} MG {S}: it={it} ok={ok} {time.perf_counter() - t:.2f}s")


if __name__ == "__main__":
    main()
