"""Phase timeline of the streaming 3D kernel k_sweep3s (library built with SW_TRACE=1):
    python tools/phase_trace3s.py [n] [tile e.g. 32x8x4]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding, gen  # noqa: E402

NAMES = {0: "P: chunk 0 arrives", 1: "P: start-column compact", 2: "P: corner + edge chains", 3: "P: x-start sheet",
         4: "P: batch 0 + B_0 wait", 6: "P: chunk waits (batches)", 7: "P: barrier waits (batches)", 8: "P: total",
         9: "C: wait for B_0", 10: "C: barrier waits (loop)", 11: "C: loop", 12: "C: total", 13: "X: busy (batches)", 14: "P1: pair-barrier waits", 15: "P2: pair-barrier waits"}


def main():
    import torch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    tile = tuple(int(v) for v in sys.argv[2].split("x")) if len(sys.argv) > 2 else (32, 8, 4)
    L = binding.load()
    L.sw_debug_phase_times.argtypes = [ctypes.c_void_p]
    g = binding.Grid(3, (n,) * 3, binding.COEF_FACES).decompose(tile)
    k = gen.lognormal_k(0, (n + 2,) * 3, 0.5)
    g.set_coefficients_k(np.pad(k, [(1, 1), (0, 0), (0, 0)], constant_values=1.0), (1.0, 0.1, 0.01))
    g.set_vector(binding.B, gen.uniform_field(0, gen.STREAM_RHS, (n,) * 3) / float((n + 1) ** 2))
    g.sor_sweep([1.0], 2, 0)
    torch.cuda.synchronize()
    out = (ctypes.c_ulonglong * 16)()
    L.sw_debug_phase_times(out)
    g.sor_sweep([1.0], 4, 2)
    torch.cuda.synchronize()
    if L.sw_debug_phase_times(out) != 16:
        print("library not built with SW_TRACE=1")
        return
    ctas = max(out[5], 1)
    print(f"n={n} tile={tile} CTAs={ctas}")
    for i in sorted(NAMES):
        print(f"  {NAMES[i]:30s} {out[i] / ctas:10.0f} cycles/CTA")


if __name__ == "__main__":
    main()
