"""Thin Python binding of the C ABI in include/sweep.h (argument marshalling only).

Every step of the method runs in the CUDA library ``libsweep.so`` (built in-tree for
sm_100a by ``paper_1008_3699_b200.build``).  There is no CPU fallback: ``load()``
raises if the library or a GPU is missing.  PyTorch is used only for device memory
views, streams and (in ``parallel.py``) process groups.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SW_LIBRARY selects another build of the same library in this directory (the race-exposure build
# libsweep_jitter.so of tests/test_gpu_jitter.py); it is never a CPU path.
LIB_PATH = os.path.join(HERE, os.path.basename(os.environ.get("SW_LIBRARY", "libsweep.so")))

SW_OK, SW_EINVAL, SW_ESINGULAR, SW_ENOCONV, SW_ECUDA, SW_ENCCL, SW_ENOMEM, SW_ESTATE = 0, 1, 2, 3, 4, 5, 6, 7
COEF_POISSON, COEF_FACES = 0, 1
PC_NONE, PC_SSOR, PC_ILU0, PC_MG = 0, 1, 2, 3
PAIR_SYMMETRIC, PAIR_PAPER = 0, 1
X, B, R, Z, P, Q, INVD, Y, W1, W2 = range(10)

_lib = None

# host-transport callbacks of sw_comm_init_host (include/sweep.h)
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)


class SweepError(RuntimeError):
    def __init__(self, code: int, what: str, msg: str):
        super().__init__(f"{what} failed: status {code}: {msg}")
        self.code = code


def load():
    """Load libsweep.so (the CUDA path).  Fails loudly if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"CUDA extension {LIB_PATH} is missing: run paper_1008_3699_b200.build.build()")
    L = ctypes.CDLL(LIB_PATH)
    P_ = ctypes.c_void_p
    I64 = ctypes.c_int64
    I = ctypes.c_int
    D = ctypes.c_double
    L.sw_create_grid.argtypes = [I, P_, I, D, I, ctypes.POINTER(P_)]
    L.sw_decompose.argtypes = [P_, P_, I, I, P_]
    L.sw_comm_unique_id.argtypes = [P_]
    L.sw_comm_init_nccl.argtypes = [P_, I, I, I, ctypes.POINTER(P_)]
    L.sw_comm_init_host.argtypes = [I, I, EXCHANGE_FN, ALLGATHER_FN, P_, ctypes.POINTER(P_)]
    L.sw_comm_destroy.argtypes = [P_]
    L.sw_local_shape.argtypes = [P_, P_, P_, P_, P_]
    L.sw_set_vector.argtypes = [P_, I, P_, I, P_]
    L.sw_get_vector.argtypes = [P_, I, P_, I, P_]
    L.sw_ghost_view.argtypes = [P_, I, ctypes.POINTER(P_)]
    L.sw_set_faces.argtypes = [P_, P_, P_]
    L.sw_set_coefficients_k.argtypes = [P_, P_, P_, P_]
    L.sw_sor_sweep.argtypes = [P_, P_, I, I, ctypes.POINTER(I64), P_]
    L.sw_residual_norm.argtypes = [P_, ctypes.POINTER(D), P_]
    L.sw_ilu0_factor.argtypes = [P_, I64, P_]
    L.sw_ilu_apply.argtypes = [P_, P_, P_, I, P_]
    L.sw_ssor_apply.argtypes = [P_, D, P_, P_, I, P_]
    L.sw_pcg_solve.argtypes = [P_, I, D, I, D, I, ctypes.POINTER(I), ctypes.POINTER(D), P_]
    L.sw_set_precond_steps.argtypes = [P_, I, D]
    L.sw_mg_setup.argtypes = [P_, I, I, D, I, D, I]
    L.sw_mg_apply.argtypes = [P_, P_, P_, P_]
    L.sw_mg_set_cycle.argtypes = [P_, I]
    L.sw_set_pcg_flexible.argtypes = [P_, I]
    L.sw_precond_stages.argtypes = [P_, I]
    L.sw_precond_stages.restype = I
    L.sw_ilu_apply_stage.argtypes = [P_, I, P_, P_, I, P_]
    L.sw_ssor_apply_stage.argtypes = [P_, I, D, P_, P_, I, P_]
    L.sw_apply_A.argtypes = [P_, P_, P_, P_, P_]
    L.sw_dot.argtypes = [P_, P_, P_, P_, P_]
    L.sw_axpy2.argtypes = [P_, D, P_, P_, P_, P_, P_, P_]
    L.sw_xpby.argtypes = [P_, P_, D, P_, P_]
    L.sw_axpby.argtypes = [P_, D, P_, D, P_, P_, P_]
    L.sw_set_diagonals.argtypes = [P_, P_, P_, P_]
    L.sw_set_slowness.argtypes = [P_, P_, D, P_]
    L.sw_eikonal_sweep.argtypes = [P_, I, ctypes.POINTER(I64), P_]
    L.sw_eikonal_changes.argtypes = [P_, ctypes.POINTER(I64), P_]
    L.sw_check_status.argtypes = [P_, P_]
    L.sw_launch_count.argtypes = [P_]
    L.sw_launch_count.restype = I64
    L.sw_destroy.argtypes = [P_]
    L.sw_last_error.restype = ctypes.c_char_p
    L.sw_debug_set_jitter.argtypes = [ctypes.c_uint]
    L.sw_debug_set_jitter.restype = I
    seed = os.environ.get("SW_JITTER_SEED")
    if seed is not None and L.sw_debug_set_jitter(int(seed)) != 1:
        raise RuntimeError(f"SW_JITTER_SEED set but {LIB_PATH} is not the jitter build")
    _lib = L
    return L


def _check(st: int, what: str, allow=()):
    if st != SW_OK and st not in allow:
        raise SweepError(st, what, load().sw_last_error().decode())
    return st


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return int(stream)


class _CAI:
    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _host_ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _bytes_at(ptr, nbytes):
    """numpy uint8 view of host memory the library hands to a callback (valid during the call)."""
    if not ptr or not nbytes:
        return None
    return np.ctypeslib.as_array((ctypes.c_uint8 * int(nbytes)).from_address(int(ptr)))


def unique_id() -> bytes:
    """NCCL unique id for sw_comm_init_nccl (rank 0 creates it, the caller broadcasts it)."""
    buf = (ctypes.c_uint8 * 128)()
    _check(load().sw_comm_unique_id(buf), "sw_comm_unique_id")
    return bytes(buf)


class Comm:
    """A communicator of the ranks of one slab decomposition (sw_comm)."""

    def __init__(self, handle, keep=()):
        self.h = handle
        self._keep = keep

    @classmethod
    def nccl(cls, uid: bytes, rank: int, nranks: int, device: int) -> "Comm":
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = ctypes.c_void_p()
        _check(load().sw_comm_init_nccl(buf, int(rank), int(nranks), int(device), ctypes.byref(h)), "sw_comm_init_nccl")
        return cls(h)

    @classmethod
    def host(cls, rank: int, nranks: int, transport) -> "Comm":
        """transport.exchange(send_lo, recv_lo, send_hi, recv_hi) and transport.allgather(send, recv)
        on numpy uint8 views (None where there is no neighbour); exceptions become SW_ENCCL."""
        def xfn(_ctx, slo, rlo, blo, shi, rhi, bhi):
            try:
                transport.exchange(_bytes_at(slo, blo), _bytes_at(rlo, blo), _bytes_at(shi, bhi), _bytes_at(rhi, bhi))
                return 0
            except Exception:                          # reported as SW_ENCCL by the library
                import traceback
                traceback.print_exc()
                return 1

        def gfn(_ctx, send, recv, nbytes):
            try:
                transport.allgather(_bytes_at(send, nbytes), _bytes_at(recv, nbytes * nranks))
                return 0
            except Exception:
                import traceback
                traceback.print_exc()
                return 1
        cx, cg = EXCHANGE_FN(xfn), ALLGATHER_FN(gfn)
        h = ctypes.c_void_p()
        _check(load().sw_comm_init_host(int(rank), int(nranks), cx, cg, None, ctypes.byref(h)), "sw_comm_init_host")
        return cls(h, keep=(cx, cg, transport))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                load().sw_comm_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Grid:
    """A structured grid with its decomposition, owned device arrays and operations."""

    def __init__(self, dim: int, n: Sequence[int], kind: int = COEF_POISSON, beta: float = 0.0, device: int = 0):
        L = load()
        self.dim = dim
        self.n = tuple(int(v) for v in n)
        nn = (ctypes.c_int64 * 3)(*(list(self.n) + [1] * (3 - dim)))
        h = ctypes.c_void_p()
        _check(L.sw_create_grid(dim, nn, kind, float(beta), int(device), ctypes.byref(h)), "sw_create_grid")
        self.h = h
        self.kind = kind
        self.device = device

    def __del__(self):
        try:
            if getattr(self, "h", None):
                load().sw_destroy(self.h)      # before its communicator (self.comm) goes
                self.h = None
        except Exception:
            pass

    # -------------------------------------------------------------- geometry
    def decompose(self, tile: Sequence[int], rank: int = 0, nranks: int = 1, comm: Optional[Comm] = None):
        """comm: a Comm of the same ranks (the library then exchanges ghost layers and sums
        reductions itself); kept alive by the grid."""
        t = (ctypes.c_int * 3)(*(list(tile) + [1] * (3 - self.dim)))
        _check(load().sw_decompose(self.h, t, int(rank), int(nranks), comm.h if comm is not None else None),
               "sw_decompose")
        self.comm = comm
        nl = (ctypes.c_int64 * 3)()
        pad = (ctypes.c_int64 * 3)()
        off = ctypes.c_int64()
        org = ctypes.c_int64()
        _check(load().sw_local_shape(self.h, nl, ctypes.byref(off), pad, ctypes.byref(org)), "sw_local_shape")
        self.n_local = tuple(nl[a] for a in range(self.dim))
        self.slab_offset = off.value
        self.pad = tuple(pad[a] for a in range(3))
        self.origin = org.value
        self.tile = tuple(tile)
        self.rank, self.nranks = rank, nranks
        return self

    @property
    def local_shape(self):
        """numpy shape of the local slab interior (slow axis first)."""
        return tuple(reversed(self.n_local))

    @property
    def padded_shape(self):
        return tuple(reversed(self.pad[: self.dim]))

    # -------------------------------------------------------------- vectors
    def set_vector(self, which: int, src, stream=None):
        """src: local-slab interior values (numpy array, or torch tensor on host/device).

        numpy arrays are copied synchronously.  torch tensors are copied stream-ordered on
        `stream` and the call returns at once (so uploads can overlap other work): a host
        tensor must stay unchanged until that stream has passed the copy."""
        try:
            import torch
            if isinstance(src, torch.Tensor):
                assert src.dtype == torch.float64 and src.is_contiguous()
                assert src.numel() == int(np.prod(self.n_local))
                _check(load().sw_set_vector(self.h, which, ctypes.c_void_p(src.data_ptr()), int(src.is_cuda),
                                            _stream(stream)), "sw_set_vector")
                return
        except ImportError:
            pass
        a = np.ascontiguousarray(np.asarray(src, dtype=np.float64))
        assert a.size == int(np.prod(self.n_local)), (a.shape, self.n_local)
        _check(load().sw_set_vector(self.h, which, _host_ptr(a), 0, _stream(stream)), "sw_set_vector")
        self.sync(stream)

    def get_vector(self, which: int, out=None, stream=None):
        """Local-slab interior values into `out` (a new numpy array if None).

        numpy: synchronous.  torch tensor: stream-ordered on `stream`, returns at once; for a
        host (e.g. pinned) tensor synchronise that stream before reading it."""
        if out is None:
            out = np.empty(self.local_shape)
        try:
            import torch
            if isinstance(out, torch.Tensor):
                _check(load().sw_get_vector(self.h, which, ctypes.c_void_p(out.data_ptr()), int(out.is_cuda),
                                            _stream(stream)), "sw_get_vector")
                return out
        except ImportError:
            pass
        _check(load().sw_get_vector(self.h, which, _host_ptr(out), 0, _stream(stream)), "sw_get_vector")
        self.sync(stream)
        return out

    def view(self, which: int):
        """torch tensor (padded shape) aliasing the library's device array (borrowed)."""
        import torch
        p = ctypes.c_void_p()
        _check(load().sw_ghost_view(self.h, which, ctypes.byref(p)), "sw_ghost_view")
        return torch.as_tensor(_CAI(p.value, self.padded_shape), device=f"cuda:{self.device}")

    def ptr(self, which: int) -> int:
        p = ctypes.c_void_p()
        _check(load().sw_ghost_view(self.h, which, ctypes.byref(p)), "sw_ghost_view")
        return p.value

    # -------------------------------------------------------------- coefficients
    def set_faces_slab(self, faces_ext, stream=None):
        """faces_ext[a]: slab-extended face arrays (see sw_set_faces)."""
        arrs = [np.ascontiguousarray(f, dtype=np.float64) for f in faces_ext]
        ptrs = (ctypes.c_void_p * 3)(*([a.ctypes.data for a in arrs] + [None] * (3 - self.dim)))
        _check(load().sw_set_faces(self.h, ptrs, _stream(stream)), "sw_set_faces")

    def set_faces_global(self, faces, stream=None):
        """Single rank convenience: faces in the oracle layout (face[a] has n_a+1 along axis a)."""
        ext = []
        for a, f in enumerate(faces):
            f = np.asarray(f, dtype=np.float64)
            pad = [(0, 0)] * self.dim
            pad[0] = (2, 2)                                     # numpy axis 0 = slab (slowest) axis
            ext.append(np.pad(f, pad))
        self.set_faces_slab(ext, stream)

    def set_coefficients_k(self, k_ext, scale=(1.0, 1.0, 1.0), stream=None):
        k = np.ascontiguousarray(np.asarray(k_ext, dtype=np.float64))
        sc = np.ascontiguousarray(np.asarray(list(scale) + [1.0] * (3 - len(scale)), dtype=np.float64)[:3])
        _check(load().sw_set_coefficients_k(self.h, _host_ptr(k), _host_ptr(sc), _stream(stream)),
               "sw_set_coefficients_k")

    # -------------------------------------------------------------- operations
    def sor_sweep(self, omega, nsweeps: int = 1, phase: int = 0, stream=None) -> int:
        w = np.ascontiguousarray(np.atleast_1d(np.asarray(omega, dtype=np.float64)))
        ph = ctypes.c_int64(int(phase))
        _check(load().sw_sor_sweep(self.h, _host_ptr(w), len(w), int(nsweeps), ctypes.byref(ph), _stream(stream)),
               "sw_sor_sweep")
        self._w = w
        return ph.value

    def residual_norm(self, stream=None) -> float:
        r = ctypes.c_double()
        _check(load().sw_residual_norm(self.h, ctypes.byref(r), _stream(stream)), "sw_residual_norm")
        return r.value

    def ilu0_factor(self, phase: int = 0, stream=None):
        _check(load().sw_ilu0_factor(self.h, int(phase), _stream(stream)), "sw_ilu0_factor")

    def ilu_apply(self, r_ptr: int, z_ptr: int, pairing: int = PAIR_SYMMETRIC, stream=None):
        _check(load().sw_ilu_apply(self.h, ctypes.c_void_p(r_ptr), ctypes.c_void_p(z_ptr), int(pairing),
                                   _stream(stream)), "sw_ilu_apply")

    def ssor_apply(self, omega: float, r_ptr: int, z_ptr: int, pairing: int = PAIR_SYMMETRIC, stream=None):
        _check(load().sw_ssor_apply(self.h, float(omega), ctypes.c_void_p(r_ptr), ctypes.c_void_p(z_ptr),
                                    int(pairing), _stream(stream)), "sw_ssor_apply")

    def set_precond_steps(self, m: int, theta: float = 0.5):
        """m-step preconditioner (sw_set_precond_steps): z_{j+1} = z_j + P^-1 (r - theta A z_j)."""
        _check(load().sw_set_precond_steps(self.h, int(m), float(theta)), "sw_set_precond_steps")
        return self

    def mg_setup(self, levels: int, nu: int = 1, theta: float = 0.5, nu_coarse: int = 8, coarse_scale: float = 1.0,
                 axes: int = 0):
        """Geometric multigrid preconditioner with the decomposed sweep as smoother (sw_mg_setup);
        axes = bit mask of the coarsened axes (0 = all)."""
        _check(load().sw_mg_setup(self.h, int(levels), int(nu), float(theta), int(nu_coarse), float(coarse_scale),
                                  int(axes)), "sw_mg_setup")
        return self

    def set_pcg_flexible(self, mode: int):
        """-1 auto (flexible beta with the PAPER pairing), 0 standard, 1 flexible (sw_set_pcg_flexible)."""
        _check(load().sw_set_pcg_flexible(self.h, int(mode)), "sw_set_pcg_flexible")
        return self

    def mg_set_cycle(self, gamma: int):
        """1 = V-cycle, 2 = W-cycle (sw_mg_set_cycle)."""
        _check(load().sw_mg_set_cycle(self.h, int(gamma)), "sw_mg_set_cycle")
        return self

    def mg_apply(self, r_ptr: int, z_ptr: int, stream=None):
        _check(load().sw_mg_apply(self.h, ctypes.c_void_p(r_ptr), ctypes.c_void_p(z_ptr), _stream(stream)), "sw_mg_apply")

    def pcg_solve(self, precond: int = PC_ILU0, omega: float = 1.0, pairing: int = PAIR_SYMMETRIC,
                  rtol: float = 1e-8, maxit: int = 10000, stream=None):
        it = ctypes.c_int()
        rr = ctypes.c_double()
        st = _check(load().sw_pcg_solve(self.h, int(precond), float(omega), int(pairing), float(rtol), int(maxit),
                                        ctypes.byref(it), ctypes.byref(rr), _stream(stream)), "sw_pcg_solve",
                    allow=(SW_ENOCONV,))
        return it.value, rr.value, st == SW_OK

    # -------------------------------------------------------------- staged / vector primitives
    # (device pointers of PADDED local-slab arrays; used by the multi-rank PCG in parallel.py)
    def precond_stages(self, pairing: int = PAIR_SYMMETRIC) -> int:
        return int(load().sw_precond_stages(self.h, int(pairing)))

    def precond_apply_stage(self, precond: int, stage: int, r_ptr: int, z_ptr: int, omega: float = 1.0,
                            pairing: int = PAIR_SYMMETRIC, stream=None):
        if precond == PC_ILU0:
            _check(load().sw_ilu_apply_stage(self.h, int(stage), ctypes.c_void_p(r_ptr), ctypes.c_void_p(z_ptr),
                                             int(pairing), _stream(stream)), "sw_ilu_apply_stage")
        elif precond == PC_SSOR:
            _check(load().sw_ssor_apply_stage(self.h, int(stage), float(omega), ctypes.c_void_p(r_ptr),
                                              ctypes.c_void_p(z_ptr), int(pairing), _stream(stream)),
                   "sw_ssor_apply_stage")
        else:
            raise ValueError("no stages for this preconditioner")

    def apply_A(self, x_ptr: int, y_ptr: int, dd_ptr: int, stream=None):
        _check(load().sw_apply_A(self.h, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr), ctypes.c_void_p(dd_ptr),
                                 _stream(stream)), "sw_apply_A")

    def dot(self, a_ptr: int, b_ptr: int, dd_ptr: int, stream=None):
        _check(load().sw_dot(self.h, ctypes.c_void_p(a_ptr), ctypes.c_void_p(b_ptr), ctypes.c_void_p(dd_ptr),
                             _stream(stream)), "sw_dot")

    def axpy2(self, alpha: float, x_ptr: int, r_ptr: int, p_ptr: int, q_ptr: int, dd_ptr: int, stream=None):
        _check(load().sw_axpy2(self.h, float(alpha), ctypes.c_void_p(x_ptr), ctypes.c_void_p(r_ptr),
                               ctypes.c_void_p(p_ptr), ctypes.c_void_p(q_ptr), ctypes.c_void_p(dd_ptr),
                               _stream(stream)), "sw_axpy2")

    def xpby(self, z_ptr: int, beta: float, p_ptr: int, stream=None):
        _check(load().sw_xpby(self.h, ctypes.c_void_p(z_ptr), float(beta), ctypes.c_void_p(p_ptr), _stream(stream)),
               "sw_xpby")

    def axpby(self, a: float, x_ptr: int, b: float, y_ptr: int, out_ptr: int, stream=None):
        """out = a x + b y (interior; products and sum rounded separately)."""
        _check(load().sw_axpby(self.h, float(a), ctypes.c_void_p(x_ptr), float(b), ctypes.c_void_p(y_ptr),
                               ctypes.c_void_p(out_ptr), _stream(stream)), "sw_axpby")

    # -------------------------------------------------------------- nine-point molecule
    def set_diagonals(self, dd, da, stream=None):
        """Diagonal coefficients of the nine-point operator: GLOBAL arrays of shape (n1 + 1, n0 + 1)
        (dd couples c - (1, 1) and c; da couples (c_x - 1, c_y) and (c_x, c_y - 1)); sw_sor_sweep then
        runs the nine-point decomposed sweep."""
        a = np.ascontiguousarray(np.asarray(dd, dtype=np.float64))
        b = np.ascontiguousarray(np.asarray(da, dtype=np.float64))
        assert a.shape == b.shape == (self.n[1] + 1, self.n[0] + 1), a.shape
        _check(load().sw_set_diagonals(self.h, _host_ptr(a), _host_ptr(b), _stream(stream)), "sw_set_diagonals")
        return self

    # -------------------------------------------------------------- eikonal
    def set_slowness(self, f, h: float, stream=None):
        """Slowness f > 0 over the local slab (numpy, slow axis first) and the grid spacing h."""
        a = np.ascontiguousarray(np.asarray(f, dtype=np.float64))
        assert a.size == int(np.prod(self.n_local)), (a.shape, self.n_local)
        _check(load().sw_set_slowness(self.h, _host_ptr(a), float(h), _stream(stream)), "sw_set_slowness")
        return self

    def eikonal_sweep(self, nsweeps: int = 1, phase: int = 0, stream=None) -> int:
        ph = ctypes.c_int64(int(phase))
        _check(load().sw_eikonal_sweep(self.h, int(nsweeps), ctypes.byref(ph), _stream(stream)), "sw_eikonal_sweep")
        return ph.value

    def eikonal_changes(self, stream=None) -> int:
        c = ctypes.c_int64()
        _check(load().sw_eikonal_changes(self.h, ctypes.byref(c), _stream(stream)), "sw_eikonal_changes")
        return c.value

    def check(self, stream=None):
        _check(load().sw_check_status(self.h, _stream(stream)), "sw_check_status")

    def sync(self, stream=None):
        import torch
        torch.cuda.synchronize(self.device)

    def launch_count(self) -> int:
        return int(load().sw_launch_count(self.h))
