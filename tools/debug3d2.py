import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from paper_1008_3699_b200 import binding, gen
from tests.gpu_helpers import make_grid, rand_faces, rel_maxdiff
n, tile = (20, 12, 8), (10, 4, 4)
faces = rand_faces(n, 17)
pb = O.tiled(n, tile, faces=faces)
r = gen.uniform_field(5, gen.STREAM_TEST, pb.shape)
inv = O.ilu0_factor(pb, phase=0)
zo = O.ilu_apply(pb, inv, r, 0)
res = {}
for mode in ("0", "1"):
    os.environ["SW_DISABLE_FAST2D"] = mode
    g = make_grid(binding, n, tile, faces)
    g.ilu0_factor(0)
    g.set_vector(binding.R, r)
    g.ilu_apply(g.ptr(binding.R), g.ptr(binding.Z), 0)
    res[mode] = g.get_vector(binding.Z)
    print("fast" if mode == "0" else "generic", rel_maxdiff(res[mode], zo))
bad = np.argwhere(res["0"] != res["1"])
print(len(bad), bad[:10].tolist())
bits, d = O.node_info(pb, 0)
for z, y, x in bad[:10]:
    print((x, y, z), "box", (x // 10, y // 4, z // 4), "bits", bits[z, y, x], "d", d[z, y, x])
