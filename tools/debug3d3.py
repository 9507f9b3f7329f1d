import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from paper_1008_3699_b200 import binding, gen
from tests.gpu_helpers import make_grid, rand_faces, rel_maxdiff
os.environ["SW_DEBUG_T1ONLY"] = "1"
n, tile = (20, 12, 8), (10, 4, 4)
faces = rand_faces(n, 17)
pb = O.tiled(n, tile, faces=faces)
r = gen.uniform_field(5, gen.STREAM_TEST, pb.shape)
res = {}
for mode in ("0", "1"):
    os.environ["SW_DISABLE_FAST2D"] = mode
    g = make_grid(binding, n, tile, faces)
    g.ilu0_factor(0)
    g.set_vector(binding.R, r)
    g.set_vector(binding.Z, np.zeros(pb.shape))
    g.ilu_apply(g.ptr(binding.R), g.ptr(binding.Z), 0)
    res[mode] = (g.get_vector(binding.Z), g.get_vector(binding.Y))
print("Y equal:", np.array_equal(res["0"][1], res["1"][1]))
zf, zg = res["0"][0], res["1"][0]
# deg-0 nodes: where the generic T1 wrote (nonzero)
mask = zg != 0
bad = np.argwhere(mask & (zf != zg))
print("deg0 nodes", mask.sum(), "differ", len(bad), bad[:10].tolist())
