"""Wait / busy breakdown of the rolling 3D sweep k_sweep3r per box (library built with SW_TRACE=1)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding, gen  # noqa: E402

NAMES = {0: "producers: wait for the wavefront", 1: "producers: total", 2: "sets warp: wait chunk 0",
         3: "sets warp: wait later chunks", 4: "sets warp: corner + y/z edges", 5: "sets warp: x-sheet + pair data",
         6: "chain warp: wait sets", 7: "chain warp: wait chunks", 9: "wavefront: wait sets",
         10: "wavefront: wait pair data", 11: "wavefront: wait x-edge chain", 12: "wavefront: total",
         13: "sets warp: total", 14: "chain warp: total"}


def main():
    import torch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    L = binding.load()
    L.sw_debug_phase_times.argtypes = [ctypes.c_void_p]
    g = binding.Grid(3, (n,) * 3, binding.COEF_FACES).decompose((32, 8, 4))
    k = gen.lognormal_k(0, (n + 2,) * 3, 0.5)
    g.set_coefficients_k(np.pad(k, [(1, 1), (0, 0), (0, 0)], constant_values=1.0), (1.0, 0.1, 0.01))
    g.set_vector(binding.B, gen.uniform_field(0, gen.STREAM_RHS, (n,) * 3) / float((n + 1) ** 2))
    g.sor_sweep([1.0], 2, 0)
    torch.cuda.synchronize()
    out = (ctypes.c_ulonglong * 16)()
    L.sw_debug_phase_times(out)
    g.sor_sweep([1.0], 2, 2)
    torch.cuda.synchronize()
    if L.sw_debug_phase_times(out) != 16:
        print("library not built with SW_TRACE=1")
        return
    boxes = max(out[15], 1)
    print(f"n={n}: {boxes} boxes traced")
    for i, nm in NAMES.items():
        print(f"  {nm:36s} {out[i] / boxes:10.0f} cycles/box")


if __name__ == "__main__":
    main()
