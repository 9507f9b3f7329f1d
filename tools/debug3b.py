import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from paper_1008_3699_b200 import binding, gen
L = binding.load()
L.sw_debug3.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
n, T = (64, 16, 8), (32, 8, 4)
pb = O.tiled(n, T)
x0 = gen.uniform_field(1, gen.STREAM_X0, pb.shape); b = gen.uniform_field(1, gen.STREAM_RHS, pb.shape)
g = binding.Grid(3, n).decompose(T)
g.set_vector(binding.X, x0); g.set_vector(binding.B, b)
L.sw_debug3(0, None, 0)
g.sor_sweep([1.0], 1, 0)
buf = np.zeros(2 * 8192)
L.sw_debug3(-2, buf.ctypes.data_as(ctypes.c_void_p), 2 * 8192)
np.save("gpurun_out/dbg3_X.npy", buf)
np.save("gpurun_out/dbg3_out.npy", g.get_vector(binding.X))
print("ok")
