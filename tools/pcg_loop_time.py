import time, os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1008_3699_b200 import binding as B, gen
for n, tile, pc in [((256, 256), (64, 64), B.PC_ILU0), ((4096, 4096), (64, 64), B.PC_ILU0)]:
    g = B.Grid(2, n, B.COEF_FACES).decompose(tile)
    k = gen.lognormal_k(0, (n[1] + 2, n[0] + 2), 1.0)
    g.set_coefficients_k(np.pad(k, [(1, 1), (0, 0)], constant_values=1.0), (1.0, 1.0))
    g.set_vector(B.B, gen.uniform_field(0, gen.STREAM_RHS, (n[1], n[0])) / float((n[0] + 1) ** 2))
    for rep in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        it, rel, ok = g.pcg_solve(pc, 1.0, 0, 1e-8, 20000)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(n, os.environ.get('SW_PCG_HOSTLOOP'), it, rel, ok, f"{dt*1e3/it:.4f} ms/it")
