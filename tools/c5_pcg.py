"""Config 5 PCG probe: 3D anisotropic n^3, boxes 32 x 8 x 4, ILU(0)/SSOR-PCG (SYMMETRIC) to 1e-8."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding, gen  # noqa: E402


def main():
    import torch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    g = binding.Grid(3, (n, n, n), binding.COEF_FACES).decompose((32, 8, 4))
    k = gen.lognormal_k(0, (n + 2,) * 3, 0.5)
    g.set_coefficients_k(np.pad(k, [(1, 1), (0, 0), (0, 0)], constant_values=1.0), (1.0, 0.1, 0.01))
    del k
    g.set_vector(binding.B, gen.uniform_field(0, gen.STREAM_RHS, (n,) * 3) / float((n + 1) ** 2))
    for name, pc in (("ilu0", binding.PC_ILU0), ("ssor", binding.PC_SSOR)):
        torch.cuda.synchronize()
        l0 = g.launch_count()
        t = time.perf_counter()
        it, rel, ok = g.pcg_solve(pc, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 5000)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"n={n} {name}: it={it} rel={rel:.3e} ok={ok} {dt:.2f}s {dt / max(it, 1) * 1e3:.3f} ms/it "
              f"launches/it={(g.launch_count() - l0) / max(it, 1):.1f}")


if __name__ == "__main__":
    main()
