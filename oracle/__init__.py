"""CPU oracle for the decomposed multi-frontal sweeps of arXiv 1008.3699.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py, never by the product path.
It shares no code with ``paper_1008_3699_b200`` (the CUDA path); both only share
the seeded input generators in ``paper_1008_3699_b200/gen.py``.

The arithmetic lives in ``oracle.c`` (plain single-threaded C, -O2
-ffp-contract=off); this file only marshals numpy arrays through ctypes.

Parity pins: see tests/test_oracle_*.py.  Functions without an external pin say
"parity unpinned" in their docstring (none at present).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_ESINGULAR, OR_ENOCONV, OR_EORDER, OR_ENOMEM, OR_EINVAL = 0, 2, 3, 4, 5, 6


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, strict IEEE: no contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Grid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int),
                ("n", ctypes.c_int64 * 3),
                ("face", ctypes.c_void_p * 3),
                ("beta", ctypes.c_double),
                ("nbox", ctypes.c_int * 3),
                ("bounds", ctypes.c_void_p * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        I = ctypes.c_int
        L = _lib
        L.or_sweep.argtypes = [P, P, I, I64, I, P, P, P, P]
        L.or_sor_lex.argtypes = [P, D, I, P, P]
        L.or_apply_A.argtypes = [P, P, P]
        L.or_relres.argtypes = [P, P, P]
        L.or_relres.restype = D
        L.or_ilu0_factor.argtypes = [P, I64, I, P]
        L.or_ilu_apply.argtypes = [P, I64, I, P, I, P, P, P]
        L.or_ssor_apply.argtypes = [P, D, I64, I, I, P, P, P]
        L.or_pcg.argtypes = [P, I, D, I, I, I64, I, D, I, P, P, P, P]
        L.or_faces_from_k.argtypes = [I, P, P, P, P]
        L.or_node_info.argtypes = [P, I64, I, P, P]
        L.or_base_bits.argtypes = [I, I64, I]
        L.or_eik_sweep.argtypes = [P, I64, I, P, D, P, P]
        L.or_eik_classical.argtypes = [P, I, P, D, P]
        L.or_sweep9.argtypes = [P, P, P, P, I, I64, I, P, P, P, P]
        L.or_sor9_frontal.argtypes = [P, P, P, D, I, P, P, P]
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def face_shape(n: Sequence[int], a: int):
    """numpy (C-order, slow axis first) shape of the axis-a face array for interior size n (x,y,z order)."""
    dim = len(n)
    m = list(n)
    m[a] += 1
    return tuple(reversed(m))


@dataclass
class Problem:
    """Structured-grid problem A u = b on n interior nodes (x, y, z order).

    faces: None (Poisson, every face 1.0) or one array per axis with shape face_shape(n, a).
    bounds: per axis box boundaries [0, ..., n_a]."""
    n: tuple
    bounds: tuple
    faces: Optional[tuple] = None
    beta: float = 0.0
    _keep: list = field(default_factory=list, repr=False)

    @property
    def dim(self):
        return len(self.n)

    @property
    def shape(self):
        """numpy shape (slow axis first)"""
        return tuple(reversed(self.n))

    @property
    def size(self):
        return int(np.prod(self.n))

    def struct(self) -> _Grid:
        g = _Grid()
        g.dim = self.dim
        keep = []
        for a in range(3):
            g.n[a] = int(self.n[a]) if a < self.dim else 1
            if a < self.dim:
                b = np.ascontiguousarray(np.asarray(self.bounds[a], dtype=np.int64))
                keep.append(b)
                g.nbox[a] = len(b) - 1
                g.bounds[a] = b.ctypes.data
                if self.faces is not None:
                    f = np.ascontiguousarray(self.faces[a], dtype=np.float64)
                    assert f.shape == face_shape(self.n, a), (f.shape, face_shape(self.n, a))
                    keep.append(f)
                    g.face[a] = f.ctypes.data
                else:
                    g.face[a] = None
            else:
                g.nbox[a] = 1
                g.bounds[a] = None
                g.face[a] = None
        g.beta = float(self.beta)
        self._keep = keep
        return g


def uniform_bounds(n: int, tile: int):
    assert n % tile == 0
    return np.arange(0, n + 1, tile, dtype=np.int64)


def balanced_bounds(n: int, p: int):
    """Balanced split, earlier boxes get the extra node (SPEC decompose)."""
    q, r = divmod(n, p)
    sizes = [q + 1] * r + [q] * (p - r)
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def tiled(n: Sequence[int], tile: Sequence[int], faces=None, beta=0.0) -> Problem:
    return Problem(tuple(int(v) for v in n), tuple(uniform_bounds(int(v), int(t)) for v, t in zip(n, tile)),
                   faces, beta)


def _arr(x, shape):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    assert a.size == int(np.prod(shape)), (a.shape, shape)
    return a.reshape(shape)


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


def _check(st, what):
    if st != OR_OK:
        raise OracleError(st, what)


def _omega_arr(omega):
    w = np.ascontiguousarray(np.atleast_1d(np.asarray(omega, dtype=np.float64)))
    return w


def sweep(pb: Problem, omega, x_old, b, phase: int = 0, override: int = -1, return_minpiv=False):
    """One decomposed SOR sweep (SURVEY §8(c) C-SOR)."""
    g = pb.struct()
    w = _omega_arr(omega)
    xo = _arr(x_old, pb.shape)
    bb = _arr(b, pb.shape)
    xn = np.empty(pb.shape)
    mp = ctypes.c_double(np.inf)
    _check(lib().or_sweep(ctypes.byref(g), _ptr(w), len(w), int(phase), int(override), _ptr(xo), _ptr(bb),
                          _ptr(xn), ctypes.byref(mp)), "sweep")
    return (xn, mp.value) if return_minpiv else xn


def sor_lex(pb: Problem, omega: float, x, b, corner: int = 0):
    """Classical in-place directional SOR sweep from `corner`."""
    g = pb.struct()
    xx = np.array(_arr(x, pb.shape), copy=True)
    bb = _arr(b, pb.shape)
    _check(lib().or_sor_lex(ctypes.byref(g), float(omega), int(corner), _ptr(xx), _ptr(bb)), "sor_lex")
    return xx


def apply_A(pb: Problem, x):
    g = pb.struct()
    xx = _arr(x, pb.shape)
    y = np.empty(pb.shape)
    lib().or_apply_A(ctypes.byref(g), _ptr(xx), _ptr(y))
    return y


def relres(pb: Problem, x, b) -> float:
    g = pb.struct()
    return float(lib().or_relres(ctypes.byref(g), _ptr(_arr(x, pb.shape)), _ptr(_arr(b, pb.shape))))


def ilu0_factor(pb: Problem, phase: int = 0, override: int = -1):
    """inverse of D~ (reading R-C of DESIGN.md)."""
    g = pb.struct()
    inv = np.empty(pb.shape)
    _check(lib().or_ilu0_factor(ctypes.byref(g), int(phase), int(override), _ptr(inv)), "ilu0_factor")
    return inv


def ilu_apply(pb: Problem, invD, r, pairing: int = 0, phase: int = 0, override: int = -1):
    g = pb.struct()
    z = np.empty(pb.shape)
    _check(lib().or_ilu_apply(ctypes.byref(g), int(phase), int(override), _ptr(_arr(invD, pb.shape)), int(pairing),
                              _ptr(_arr(r, pb.shape)), _ptr(z), None), "ilu_apply")
    return z


def ssor_apply(pb: Problem, omega: float, r, pairing: int = 0, phase: int = 0, override: int = -1):
    g = pb.struct()
    z = np.empty(pb.shape)
    _check(lib().or_ssor_apply(ctypes.byref(g), float(omega), int(phase), int(override), int(pairing),
                               _ptr(_arr(r, pb.shape)), _ptr(z), None), "ssor_apply")
    return z


def pcg(pb: Problem, b, precond: int = 2, omega: float = 1.0, pairing: int = 0, flexible: bool = False,
        rtol: float = 1e-8, maxit: int = 10000, phase: int = 0, override: int = -1):
    """PCG; returns (x, iterations, relres, converged)."""
    g = pb.struct()
    x = np.empty(pb.shape)
    it = ctypes.c_int(0)
    rr = ctypes.c_double(0.0)
    st = lib().or_pcg(ctypes.byref(g), int(precond), float(omega), int(pairing), int(bool(flexible)), int(phase),
                      int(override), float(rtol), int(maxit), _ptr(_arr(b, pb.shape)), _ptr(x), ctypes.byref(it),
                      ctypes.byref(rr))
    if st not in (OR_OK, OR_ENOCONV):
        raise OracleError(st, "pcg")
    return x, it.value, rr.value, st == OR_OK


def faces_from_k(n: Sequence[int], k_ring, scale=(1.0, 1.0, 1.0)):
    """Harmonic-mean face coefficients from node values incl. boundary ring."""
    dim = len(n)
    nn = (ctypes.c_int64 * 3)(*(list(n) + [1] * (3 - dim)))
    kr = np.ascontiguousarray(np.asarray(k_ring, dtype=np.float64))
    assert kr.size == int(np.prod([v + 2 for v in n]))
    sc = np.ascontiguousarray(np.asarray(list(scale) + [1.0] * (3 - len(scale)), dtype=np.float64)[:3])
    faces = [np.empty(face_shape(n, a)) for a in range(dim)]
    fp = (ctypes.c_void_p * 3)(*([f.ctypes.data for f in faces] + [None] * (3 - dim)))
    lib().or_faces_from_k(dim, nn, _ptr(kr), _ptr(sc), fp)
    return tuple(faces)


def node_info(pb: Problem, phase: int = 0, override: int = -1):
    """(direction bits, wavefront index) of every node."""
    g = pb.struct()
    bits = np.empty(pb.shape, dtype=np.int32)
    d = np.empty(pb.shape, dtype=np.int64)
    _check(lib().or_node_info(ctypes.byref(g), int(phase), int(override), _ptr(bits), _ptr(d)), "node_info")
    return bits, d


def base_bits(dim: int, phase: int, override: int = -1) -> int:
    return int(lib().or_base_bits(int(dim), int(phase), int(override)))


def scc_stats(pb: Problem, phase: int = 0, override: int = -1):
    """{size: (count, total nnz)} of the coupled systems of one forward sweep."""
    g = pb.struct()
    hist = (ctypes.c_int64 * 9)()
    nnz = (ctypes.c_int64 * 9)()
    L = lib()
    L.or_scc_stats.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    _check(L.or_scc_stats(ctypes.byref(g), int(phase), int(override), hist, nnz), "scc_stats")
    return {s: (hist[s], nnz[s]) for s in range(1, 9) if hist[s]}


# ---------------------------------------------------------------- eikonal
def eik_sweep(pb: Problem, f, h: float, u_old, phase: int = 0, override: int = -1):
    """One decomposed fast-sweeping pass for |grad u| = f (Godunov update, coupled sets solved
    exactly by ordered fixing; DESIGN R-E1..R-E3).  2D / 1D."""
    g = pb.struct()
    u = np.empty(pb.shape)
    _check(lib().or_eik_sweep(ctypes.byref(g), int(phase), int(override), _ptr(_arr(f, pb.shape)), float(h),
                              _ptr(_arr(u_old, pb.shape)), _ptr(u)), "eik_sweep")
    return u


def eik_classical(pb: Problem, corner: int, f, h: float, u):
    """Textbook in-place fast-sweeping pass from `corner` (Zhao 2005); ignores boxes."""
    g = pb.struct()
    uu = np.array(_arr(u, pb.shape), copy=True)
    _check(lib().or_eik_classical(ctypes.byref(g), int(corner), _ptr(_arr(f, pb.shape)), float(h), _ptr(uu)),
           "eik_classical")
    return uu


# ------------------------------------------------------------ nine-point molecule
def diag_shape(n):
    """numpy shape of a diagonal coefficient array ((n1 + 1) x (n0 + 1)) for a 2D grid n = (n0, n1)."""
    return (n[1] + 1, n[0] + 1)


def sweep9(pb: Problem, diag, omega, x_old, b, phase: int = 0, override: int = -1, return_minpiv=False):
    """One decomposed nine-point SOR sweep (reading R-N3).  diag = (dd, da): SW-NE
    and SE-NW coefficients, shape diag_shape(n); pb.faces are the axis faces (None = 1)."""
    g = pb.struct()
    dd = _arr(diag[0], diag_shape(pb.n))
    da = _arr(diag[1], diag_shape(pb.n))
    w = _omega_arr(omega)
    xn = np.empty(pb.shape)
    mp = ctypes.c_double(np.inf)
    _check(lib().or_sweep9(ctypes.byref(g), _ptr(dd), _ptr(da), _ptr(w), len(w), int(phase), int(override),
                           _ptr(_arr(x_old, pb.shape)), _ptr(_arr(b, pb.shape)), _ptr(xn), ctypes.byref(mp)), "sweep9")
    return (xn, mp.value) if return_minpiv else xn


def sor9_frontal(pb: Problem, diag, omega: float, x_old, b, corner: int = 0):
    """Textbook frontal nine-point SOR from `corner` (one box; new W, S, SW, old E, N, NE, SE, NW)."""
    g = pb.struct()
    xn = np.empty(pb.shape)
    _check(lib().or_sor9_frontal(ctypes.byref(g), _ptr(_arr(diag[0], diag_shape(pb.n))),
                                 _ptr(_arr(diag[1], diag_shape(pb.n))), float(omega), int(corner),
                                 _ptr(_arr(x_old, pb.shape)), _ptr(_arr(b, pb.shape)), _ptr(xn)), "sor9_frontal")
    return xn
