import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1008_3699_b200 import binding as B, gen
import torch
n = int(sys.argv[1])
nn = (n, n, n)
g = B.Grid(3, nn, B.COEF_FACES).decompose((32, 8, 4))
k = gen.lognormal_k(0, (n + 2,) * 3, 0.5)
g.set_coefficients_k(np.pad(k, [(1, 1), (0, 0), (0, 0)], constant_values=1.0), (1.0, 0.1, 0.01))
g.set_vector(B.B, gen.uniform_field(0, gen.STREAM_RHS, nn) / float((n + 1) ** 2))

SETS = [tuple(float(x) if '.' in x else int(x) for x in a.split(',')) for a in sys.argv[2:]] or [(4,1,0.5,8,1.2)]
for S in SETS:
    g.mg_setup(*S[:6])
    g.mg_set_cycle(S[6] if len(S) > 6 else 1)
    t = time.perf_counter(); it, rel, ok = g.pcg_solve(B.PC_MG, 1.0, 0, 1e-8, 5000); torch.cuda.synchronize()
    print(f"  MG {S}: it={it} ok={ok} {time.perf_counter()-t:.2f}s")
