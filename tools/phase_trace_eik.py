"""Phase clocks of the eikonal pass (library built with SW_TRACE=1)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding, gen  # noqa: E402


def main():
    import torch
    n = 4096
    L = binding.load()
    L.sw_debug_phase_times.argtypes = [ctypes.c_void_p]
    ge = binding.Grid(2, (n, n)).decompose((64, 64))
    ge.set_slowness(0.5 + gen.uniform_field(0, gen.STREAM_TEST, (n, n)) ** 2, 1.0 / n)
    u0 = np.full((n, n), np.inf)
    u0[n // 3, n // 2] = 0.0
    ge.set_vector(binding.X, u0)
    ph = ge.eikonal_sweep(2, 0)
    if len(sys.argv) > 1 and sys.argv[1] == "reached":      # every box reached: the full per-node work
        while ge.eikonal_changes() > 0 and ph < 4000:
            ph = ge.eikonal_sweep(8, ph)
    torch.cuda.synchronize()
    out = (ctypes.c_ulonglong * 16)()
    L.sw_debug_phase_times(out)
    ge.eikonal_sweep(4, ph)
    torch.cuda.synchronize()
    L.sw_debug_phase_times(out)
    c = max(out[5], 1)
    for i, nm in ((0, "stage-in"), (1, "corner + chains"), (2, "levels")):
        print(f"  {nm:18s} {out[i] / c:10.0f} cycles/CTA")


if __name__ == "__main__":
    main()
