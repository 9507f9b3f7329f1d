"""Slab helpers of the multi-rank GPU tests: slab-extended face arrays, per-rank grids, scatter /
gather of the local slabs, and ranks run as threads of one process (parallel.ThreadHub) or as
processes (tests/test_gpu_multiproc.py)."""
import threading

import numpy as np

from paper_1008_3699_b200 import binding as B, parallel


def slab_faces(faces, n, off, n_loc):
    """Slab-extended face arrays for sw_set_faces (2 extra layers per side of the slab axis)."""
    dim = len(n)
    out = []
    for a, f in enumerate(faces):
        f = np.asarray(f)
        ext = n_loc + 4 + (1 if a == dim - 1 else 0)
        shape = list(f.shape)
        shape[0] = ext
        e = np.zeros(shape)
        for j in range(ext):
            gj = off - 2 + j
            if 0 <= gj < f.shape[0]:
                e[j] = f[gj]
        out.append(e)
    return out


def make_slabs(n, tile, nranks, faces=None, beta=0.0):
    kind = B.COEF_POISSON if faces is None else B.COEF_FACES
    grids = []
    for r in range(nranks):
        g = B.Grid(len(n), n, kind, beta).decompose(tile, r, nranks)
        if faces is not None:
            g.set_faces_slab(slab_faces(faces, n, g.slab_offset, g.n_local[-1]))
        grids.append(g)
    return grids


def scatter(grids, which, full):
    for g in grids:
        sl = full[g.slab_offset:g.slab_offset + g.n_local[-1]]
        g.set_vector(which, np.ascontiguousarray(sl))


def gather(grids, which):
    return np.concatenate([g.get_vector(which) for g in grids], axis=0)


def make_slab(n, tile, rank, nranks, faces=None, beta=0.0, comm=None):
    kind = B.COEF_POISSON if faces is None else B.COEF_FACES
    g = B.Grid(len(n), n, kind, beta).decompose(tile, rank, nranks, comm)
    if faces is not None:
        g.set_faces_slab(slab_faces(faces, n, g.slab_offset, g.n_local[-1]))
    return g


def local_part(g, full):
    return np.ascontiguousarray(full[g.slab_offset:g.slab_offset + g.n_local[-1]])


def run_threads(world, fn):
    """fn(rank, comm) in `world` threads, each with its own HOST communicator of one ThreadHub;
    returns [fn's result per rank]; re-raises the first exception."""
    hub = parallel.ThreadHub(world)
    out = [None] * world
    errs = []

    def body(r):
        try:
            import torch
            torch.cuda.set_device(0)
            comm = parallel.host_comm(r, world, hub.endpoint(r))
            out[r] = fn(r, comm)
        except BaseException as e:          # noqa: BLE001 (re-raised below)
            errs.append(e)
            hub.barrier.abort()
    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return out
