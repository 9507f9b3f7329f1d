"""Time the decomposed eikonal pass on bench.py's N4 grid (4096^2, 64x64 boxes)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_3699_b200 import binding, gen  # noqa: E402


def main():
    import torch
    n = 4096
    ge = binding.Grid(2, (n, n)).decompose((64, 64))
    ge.set_slowness(0.5 + gen.uniform_field(0, gen.STREAM_TEST, (n, n)) ** 2, 1.0 / n)
    u0 = np.full((n, n), np.inf)
    u0[n // 3, n // 2] = 0.0
    ge.set_vector(binding.X, u0)
    ph = ge.eikonal_sweep(2, 0)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    ph = ge.eikonal_sweep(8, ph)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 8
    print(f"eikonal 4096^2: {ms:.4f} ms/pass, {n * n / ms / 1e6:.2f} GLUP/s")


if __name__ == "__main__":
    main()
