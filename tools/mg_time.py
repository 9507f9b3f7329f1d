"""Per-configuration V/W-cycle cost (graph-captured sw_mg_apply) and MG-PCG iterations for config 3:
python tools/mg_time.py n L,nu,theta,nc,s[,axes[,gamma]] ..."""
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
    shp = tuple(int(v) for v in reversed(g.padded_shape)) if hasattr(g, "padded_shape") else None
    for a in sys.argv[2:]:
        S = tuple(float(x) if '.' in x else int(x) for x in a.split(','))
        g.mg_setup(*S[:6])
        g.mg_set_cycle(S[6] if len(S) > 6 else 1)
        torch.cuda.synchronize()
        t = time.perf_counter()
        it, rel, ok = g.pcg_solve(B.PC_MG, 1.0, 0, 1e-8, 20000)
        torch.cuda.synchronize()
        el = time.perf_counter() - t
        print(f"n={n} MG {S}: it={it} ok={ok} {el:.2f}s  {1e3 * el / max(it, 1):.3f} ms/it", flush=True)


if __name__ == "__main__":
    main()
