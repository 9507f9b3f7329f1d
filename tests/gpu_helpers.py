"""Helpers shared by the GPU parity tests (inputs come from gen.py; expectations from oracle/)."""
import numpy as np

import oracle as O
from paper_1008_3699_b200 import gen


def rand_faces(n, seed, lo=0.5, hi=2.0):
    return tuple(lo + (hi - lo) * gen.unit(seed, gen.STREAM_TEST + a, int(np.prod(O.face_shape(n, a)))).reshape(
        O.face_shape(n, a)) for a in range(len(n)))


def make_grid(binding, n, tile, faces=None, beta=0.0):
    kind = binding.COEF_POISSON if faces is None else binding.COEF_FACES
    g = binding.Grid(len(n), n, kind, beta).decompose(tile)
    if faces is not None:
        g.set_faces_global(faces)
    return g


def rel_maxdiff(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    scale = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / scale)
