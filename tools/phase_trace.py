"""Per-phase cycle breakdown of the 2D sweep kernel (library built with SW_TRACE=1)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding, gen  # noqa: E402

NAMES = ["stage-in wait", "partner+prologue", "corner+chains", "wavefront", "write-back", "", "chains (warp 1)",
         "wavefront (warp 0)", "3D: prologue (thr 0, own part)", "3D: wavefront (thr 0, no barrier)", "3D: wf steps 1-8", "3D: wf last 8 steps",
         "3D: corner (thr 0)", "3D: x-sheet", "3D: wf middle steps"]


def main():
    import torch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    faces = len(sys.argv) > 2 and sys.argv[2] == "faces"
    dim = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    tile = tuple(int(v) for v in sys.argv[4].split("x")) if len(sys.argv) > 4 else (64, 64)
    L = binding.load()
    L.sw_debug_phase_times.argtypes = [ctypes.c_void_p]
    g = binding.Grid(dim, (n,) * dim, binding.COEF_FACES if faces else binding.COEF_POISSON).decompose(tile)
    if faces:
        k = gen.lognormal_k(0, (n + 2,) * dim, 1.0)
        pad = [(0, 0)] * dim
        pad[0] = (1, 1)
        g.set_coefficients_k(np.pad(k, pad, constant_values=1.0), (1.0,) * dim)
    g.set_vector(binding.B, gen.uniform_field(0, gen.STREAM_RHS, (n,) * dim) / float((n + 1) ** 2))
    g.sor_sweep([1.9], 2, 0)
    torch.cuda.synchronize()
    out = (ctypes.c_ulonglong * 16)()
    L.sw_debug_phase_times(out)
    g.sor_sweep([1.9], 4, 2)
    torch.cuda.synchronize()
    if L.sw_debug_phase_times(out) != 16:
        print("library not built with SW_TRACE=1")
        return
    ctas = out[5]
    print(f"n={n} faces={faces} CTAs={ctas}")
    for i, nm in enumerate(NAMES[:15]):
        if nm:
            print(f"  {nm:18s} {out[i] / max(ctas, 1):10.0f} cycles/CTA")
    print(f"  {'total':18s} {sum(out[i] for i in range(5)) / max(ctas, 1):10.0f}")


if __name__ == "__main__":
    main()
