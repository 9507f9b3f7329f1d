"""The multi-process slab path on one GPU ("a single process cannot stand in for this"):
2 and 4 processes, one rank each, every one driving its own slab grid through the C ABI with a
HOST communicator over torch.distributed gloo (parallel.GlooTransport; NCCL needs one GPU per
rank).  Inside the library: multi-sweep sw_sor_sweep with the exchange behind the interior rows,
sw_residual_norm, the multi-rank ILU(0) / SSOR application and sw_pcg_solve.  Results are gathered
in the parent and compared with the ORACLE: sweeps and preconditioner applications bitwise, PCG
iterations within 1, the solution's oracle residual < 2e-8.  No kernel waits on another process:
every wait is on the host, inside gloo."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from paper_1008_3699_b200 import binding as B, gen
from tests.gpu_helpers import rand_faces

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_1008_3699_b200 import parallel
    from tests.slab_helpers import local_part, make_slab
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        n, tile, var, nsw, pc = case["n"], case["tile"], case["var"], case["nsw"], case["pc"]
        faces, x0, b, r0 = case["faces"], case["x0"], case["b"], case["r0"]
        comm = parallel.host_comm(rank, world, parallel.GlooTransport())
        out = {}
        g = make_slab(n, tile, rank, world, faces, 0.0, comm)
        g.set_vector(B.X, local_part(g, x0))
        g.set_vector(B.B, local_part(g, b))
        out["phase"] = g.sor_sweep(case["w"], nsw, 0)
        out["x"] = g.get_vector(B.X)
        out["rel"] = g.residual_norm()
        g.set_vector(B.R, local_part(g, r0))
        if pc == B.PC_ILU0:
            g.ilu0_factor(0)
            g.ilu_apply(g.ptr(B.R), g.ptr(B.Z), B.PAIR_SYMMETRIC)
        else:
            g.ssor_apply(1.2, g.ptr(B.R), g.ptr(B.Z), B.PAIR_SYMMETRIC)
        out["z"] = g.get_vector(B.Z)
        g.set_vector(B.B, local_part(g, case["bp"]))
        out["pcg"] = g.pcg_solve(pc, 1.0, B.PAIR_SYMMETRIC, 1e-8, 5000)
        out["xp"] = g.get_vector(B.X)
        g.check()
        q.put((rank, out))
    except BaseException as e:  # noqa: BLE001 (reported to the parent)
        import traceback
        q.put((rank, {"error": repr(e) + "\n" + traceback.format_exc()}))
    finally:
        dist.destroy_process_group()


CASES = [((256, 512), (64, 64), 2, False, 5, B.PC_ILU0), ((256, 512), (64, 64), 4, True, 5, B.PC_SSOR),
         ((64, 32, 32), (32, 8, 4), 2, True, 9, B.PC_ILU0), ((64, 16, 64), (32, 8, 4), 4, True, 9, B.PC_ILU0)]


@pytest.mark.parametrize("n,tile,world,var,nsw,pc", CASES)
def test_multiprocess_slabs_match_oracle(n, tile, world, var, nsw, pc):
    faces = rand_faces(n, 29) if var else None
    pb = O.tiled(n, tile, faces=faces)
    w = [1.2] if var else [1.8]
    case = dict(n=n, tile=tile, var=var, nsw=nsw, pc=pc, faces=faces, w=w,
                x0=gen.uniform_field(5, gen.STREAM_X0, pb.shape), b=gen.uniform_field(5, gen.STREAM_RHS, pb.shape),
                r0=gen.uniform_field(5, gen.STREAM_TEST, pb.shape),
                bp=gen.uniform_field(6, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    errs = [v["error"] for v in res.values() if "error" in v]
    assert not errs, errs[0]
    assert all(p.exitcode == 0 for p in procs)
    cat = lambda k: np.concatenate([res[r][k] for r in range(world)], axis=0)  # noqa: E731
    x = case["x0"]
    for k in range(nsw):
        x = O.sweep(pb, w, x, case["b"], phase=k)
    assert all(res[r]["phase"] == nsw for r in range(world))
    assert np.array_equal(cat("x"), x)
    rel_o = O.relres(pb, x, case["b"])
    assert all(abs(res[r]["rel"] - rel_o) <= 1e-12 * rel_o for r in range(world))
    if pc == B.PC_ILU0:
        zo = O.ilu_apply(pb, O.ilu0_factor(pb), case["r0"], 0)
    else:
        zo = O.ssor_apply(pb, 1.2, case["r0"], 0)
    assert np.array_equal(cat("z"), zo)
    its = {res[r]["pcg"][0] for r in range(world)}
    assert len(its) == 1 and all(res[r]["pcg"][2] for r in range(world))
    _, ito, _, oko = O.pcg(pb, case["bp"], precond=pc, omega=1.0, pairing=0, rtol=1e-8, maxit=5000)
    assert oko and abs(its.pop() - ito) <= 1
    assert O.relres(pb, cat("xp"), case["bp"]) < 2e-8
