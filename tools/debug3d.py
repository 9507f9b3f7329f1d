"""Locate differences between the fast 3D kernel and the oracle for one sweep (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_1008_3699_b200 import binding, gen  # noqa: E402
from tests.gpu_helpers import make_grid, rand_faces  # noqa: E402


def run(n, tile, var, omega, phase=0, beta=0.0):
    faces = rand_faces(n, 7) if var else None
    pb = O.tiled(n, tile, faces=faces, beta=beta)
    g = make_grid(binding, n, tile, faces, beta)
    x0 = gen.uniform_field(1, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(1, gen.STREAM_RHS, pb.shape)
    g.set_vector(binding.X, x0)
    g.set_vector(binding.B, b)
    g.sor_sweep(omega, 1, phase)
    got = g.get_vector(binding.X)
    ref = O.sweep(pb, omega, x0, b, phase=phase)
    bad = np.argwhere(got != ref)
    print(f"n={n} tile={tile} var={var} phase={phase}: {len(bad)} of {got.size} differ")
    if len(bad):
        # numpy order (z, y, x); report local box coords and counts by local position class
        bz, by, bx = bad[:, 0], bad[:, 1], bad[:, 2]
        lx, ly, lz = bx % tile[0], by % tile[1], bz % tile[2]
        print("  first:", [(int(x), int(y), int(z)) for z, y, x in bad[:8]])
        print("  local x hist:", np.bincount(lx, minlength=tile[0]))
        print("  local y hist:", np.bincount(ly, minlength=tile[1]))
        print("  local z hist:", np.bincount(lz, minlength=tile[2]))
        z, y, x = bad[0]
        print("  got", got[z, y, x], "ref", ref[z, y, x])


if __name__ == "__main__":
    run((32, 8, 4), (32, 8, 4), False, [1.0])
    run((32, 8, 4), (32, 8, 4), True, [1.0])
    run((64, 8, 4), (32, 8, 4), False, [1.0])
    run((32, 16, 4), (32, 8, 4), False, [1.0])
    run((32, 8, 8), (32, 8, 4), False, [1.0])
    run((32, 32, 32), (16, 8, 8), True, [1.0])
    for ph in range(8):
        run((64, 16, 8), (32, 8, 4), False, [1.0], phase=ph)


def levels(n, tile, var, omega, phase):
    faces = rand_faces(n, 7) if var else None
    pb = O.tiled(n, tile, faces=faces)
    g = make_grid(binding, n, tile, faces)
    x0 = gen.uniform_field(1, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(1, gen.STREAM_RHS, pb.shape)
    g.set_vector(binding.X, x0)
    g.set_vector(binding.B, b)
    g.sor_sweep(omega, 1, phase)
    got = g.get_vector(binding.X)
    ref = O.sweep(pb, omega, x0, b, phase=phase)
    bits, d = O.node_info(pb, phase)
    bad = got != ref
    nb = [n[a] // tile[a] for a in range(3)]
    for bz in range(nb[2]):
        for by in range(nb[1]):
            for bx in range(nb[0]):
                sl = (slice(bz * tile[2], (bz + 1) * tile[2]), slice(by * tile[1], (by + 1) * tile[1]),
                      slice(bx * tile[0], (bx + 1) * tile[0]))
                bb = bad[sl]
                if bb.any():
                    dd = d[sl][bb]
                    dmin = dd.min()
                    pos = np.argwhere(bb & (d[sl] == dmin))
                    print(f"  box ({bx},{by},{bz}) bits={bits[sl].flat[0]}: {bb.sum()} bad, min level {dmin}, at (z,y,x)",
                          pos[:4].tolist())


if __name__ == "__main__":
    print("---- levels")
    for ph in (0, 4):
        print("phase", ph)
        levels((64, 16, 8), (32, 8, 4), False, [1.0], ph)
