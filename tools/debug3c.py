import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from paper_1008_3699_b200 import binding, gen
from tests.gpu_helpers import make_grid, rand_faces, rel_maxdiff
for n, tile in [((20, 12, 8), (10, 4, 4)), ((16, 16, 16), (8, 8, 8)), ((64, 32, 16), (32, 8, 4)), ((20, 12, 8), (10, 12, 8))]:
    faces = rand_faces(n, 17)
    pb = O.tiled(n, tile, faces=faces)
    g = make_grid(binding, n, tile, faces)
    r = gen.uniform_field(5, gen.STREAM_TEST, pb.shape)
    g.ilu0_factor(0)
    inv = O.ilu0_factor(pb, phase=0)
    g.set_vector(binding.R, r)
    for pairing in (1, 0):
        g.ilu_apply(g.ptr(binding.R), g.ptr(binding.Z), pairing)
        z = g.get_vector(binding.Z)
        y = g.get_vector(binding.Y)
        zo = O.ilu_apply(pb, inv, r, pairing)
        print(n, tile, "pairing", pairing, "err", rel_maxdiff(z, zo))
        if pairing == 0:
            bad = np.argwhere(np.abs(z - zo) > 1e-12)
            print("  bad", len(bad), bad[:6].tolist())
