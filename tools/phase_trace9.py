"""Phase clocks of the nine-point sweep k_sweep9 (library built with SW_TRACE=1), bench.py's N3 grid."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding, gen  # noqa: E402


def make_g9(n):
    """bench.py's N3 grid: Mehrstellen Laplacian (axis faces 4, diagonals 1), U[-1,1) rhs."""
    g9 = binding.Grid(2, (n, n), binding.COEF_FACES).decompose((64, 64))
    F9 = [np.full(tuple(reversed((n + (a == 0), n + (a == 1)))), 4.0) for a in range(2)]
    g9.set_faces_global(F9)
    g9.set_diagonals(np.ones((n + 1, n + 1)), np.ones((n + 1, n + 1)))
    g9.set_vector(binding.B, gen.uniform_field(0, gen.STREAM_RHS, (n, n)) / float((n + 1) ** 2))
    return g9


def main():
    import torch
    n = 4096
    L = binding.load()
    L.sw_debug_phase_times.argtypes = [ctypes.c_void_p]
    g9 = make_g9(n)
    g9.sor_sweep([1.0], 2, 0)
    torch.cuda.synchronize()
    out = (ctypes.c_ulonglong * 16)()
    L.sw_debug_phase_times(out)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    g9.sor_sweep([1.0], 4, 2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 4
    L.sw_debug_phase_times(out)
    c = max(out[5], 1)
    print(f"nine-point 4096^2: {ms:.4f} ms/sweep, {n * n / ms / 1e6:.2f} GLUP/s")
    for i, nm in ((0, "stage-in"), (1, "alpha / r0"), (2, "set coefficients"), (3, "chains + wavefront"), (4, "  of which chains")):
        print(f"  {nm:18s} {out[i] / c:10.0f} cycles/CTA")


if __name__ == "__main__":
    main()
