import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1008_3699_b200 import binding as B, gen
n = 256
g = B.Grid(2, (n, n)).decompose((64, 64))
g.set_vector(B.B, gen.uniform_field(0, gen.STREAM_RHS, (n, n)) / float((n + 1) ** 2))
for th in (0.5, 0.45, 0.4, 0.35):
    r = []
    for m in (2, 3, 4):
        g.set_precond_steps(m, th)
        it, rel, ok = g.pcg_solve(B.PC_SSOR, 1.0, B.PAIR_SYMMETRIC, 1e-8, 20000)
        r.append(it)
    g.set_precond_steps(1, 1.0)
    g.mg_setup(4, 1, th, 16, 1.2)
    itm, _, _ = g.pcg_solve(B.PC_MG, 1.0, B.PAIR_SYMMETRIC, 1e-8, 20000)
    print("theta", th, "mstep 2/3/4:", r, "mg4:", itm, flush=True)
