#!/usr/bin/env python
"""Benchmark of the decomposed multi-frontal SOR sweep (arXiv 1008.3699) on B200.

Metric (BASELINE.json): lattice-point sweep updates per second (GLUP/s) and the
fraction of the HBM roofline.  Workload at N=1 (config 4 of BASELINE.json, the
1/2/4/8-GPU scaling config): 2D 5-point Poisson on 16384 x 16384 fp64, Dirichlet 0,
b = h^2 f with f ~ U[-1,1) (seeded, gen.py), 64 x 64 boxes, omega = 2/(1+sin(pi h)).
One step = one decomposed SOR sweep over the whole grid (schedule, ghost refresh,
corner/edge coupled solves, interior wavefront, write-back: SURVEY §8(a) a2-a8).
For N > 1 (torchrun): --scaling weak (default; 16384 x 16384 N) or strong (16384^2 over N),
row slabs per rank; the library's communicator (NCCL) moves the 2 ghost layers every sweep
behind the interior tile rows; config 5 runs slab-sharded (sweep, ILU(0)- and SSOR-PCG).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B_PER_LUP_POISSON = 24          # x_old read, x_new write, b read
NX = 16384
TILE5 = (512, 8, 4)             # config 5's boxes: whole x-lines (the strong axis of the 1 : 0.1 : 0.01 anisotropy)
TILE5_CMP = (32, 8, 4)          # the round-1 box, kept as a comparison line


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.lines = []            # (monotonic time, line)
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def start(self):
        """Mark the start of the timed region (the sampler itself runs from before the warm-up,
        so that samples already flow when the region begins)."""
        self.t0 = time.monotonic()

    def stop(self):
        self.t1 = time.monotonic()
        time.sleep(0.05)           # let the sample that covers the end arrive

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.t0 is not None and self.t1 is not None:
            inside = [ln for t, ln in lines if self.t0 <= t <= self.t1 + 0.03]
            if not inside:             # a region shorter than the sampling period: the next sample
                inside = [ln for t, ln in lines if t >= self.t0][:1]
            lines = inside
        else:
            lines = [ln for _, ln in lines]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def rhs_slab(seed, rows, row0, nx, h):
    from paper_1008_3699_b200 import gen
    f = gen.uniform(seed, gen.STREAM_RHS, rows * nx, start=row0 * nx)
    return (f * (h * h)).reshape(rows, nx)


def make_comm(args, world, rank, dev):
    """torch.distributed plumbing + the library's communicator (NCCL, one rank per GPU; or the
    gloo host transport for several ranks sharing one GPU in tests)."""
    import torch
    import torch.distributed as dist

    from paper_1008_3699_b200 import parallel
    if world == 1:
        return None
    if args.comm == "nccl":
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
        return parallel.nccl_comm(dev)
    dist.init_process_group("gloo")
    return parallel.host_comm(rank, world, parallel.GlooTransport())


def max_over_ranks(v, world):
    import torch
    import torch.distributed as dist
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1008_3699_b200 import binding
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    binding.load()
    comm = make_comm(args, world, rank, dev)
    T = 64
    NXl = args.nx
    weak = args.scaling == "weak"
    ny = NXl * world if weak else NXl     # weak: 16384 x 16384 per GPU; strong: 16384^2 split over N
    n = (NXl, ny)
    h = 1.0 / (NXl + 1)
    omega = 2.0 / (1.0 + np.sin(np.pi * h))
    g = binding.Grid(2, n, binding.COEF_POISSON, 0.0, dev).decompose((T, T), rank, world, comm)
    nl_y = g.n_local[1]
    row0 = g.slab_offset
    b = rhs_slab(args.seed, nl_y, row0, NXl, h)
    g.set_vector(binding.B, b)
    g.set_vector(binding.X, np.zeros((nl_y, NXl)))
    stream = torch.cuda.current_stream()
    phase = 0
    clk = ClockSampler(dev).__enter__()        # sampling from before the warm-up on
    time.sleep(0.3)                            # nvidia-smi's first samples
    # warm-up: W sweeps (the first call also exchanges b's and x's ghost layers once)
    phase = g.sor_sweep([omega], args.warmup, phase)
    barrier(world)
    l0 = g.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clk.start()
    ev0.record(stream)
    # K steps = K decomposed sweeps in one C call; with N ranks every sweep runs the slab's boundary
    # tile rows, then the interior rows while the 2 new boundary layers go to the neighbours (NCCL)
    phase = g.sor_sweep([omega], args.steps, phase)
    ev1.record(stream)
    torch.cuda.synchronize()
    clk.stop()
    clk.__exit__(None, None, None)
    ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    launches = g.launch_count() - l0
    nodes_total = NXl * ny
    glups = nodes_total * args.steps / (ms * 1e-3) / 1e9
    ms_per_step = ms / args.steps

    # dominant kernel = the sweep kernel (the only kernel of a single-GPU step); its per-launch
    # duration from CUDA events on the launching stream, one launch per event pair
    kern_ms = []
    if world == 1:
        for _ in range(min(args.steps, 10)):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            phase = g.sor_sweep([omega], 1, phase)
            e1.record(stream)
            torch.cuda.synchronize()
            kern_ms.append(e0.elapsed_time(e1))
    else:
        kern_ms = [ms_per_step]
    peak, peak_src = peaks()
    per_launch_bytes = B_PER_LUP_POISSON * (NXl * nl_y)
    # average launch duration over the timed region: every launch in it is the sweep kernel (one
    # per step on one GPU), so the events around the region give it directly; the separately
    # timed launches (an event pair each) are reported beside it.  N > 1: a step is three launches
    # (two boundary row ranges, the interior) plus the exchange, so the whole step is the unit.
    kiso = float(np.mean(kern_ms))
    kavg = ms / launches if (world == 1 and launches == args.steps) else kiso
    achieved = per_launch_bytes / (kavg * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "sweep2p_traffic.json")
    if os.path.exists(tf):
        with open(tf) as f:
            tj = json.load(f)
        traffic = tj.get("bytes_per_launch")
        traffic_src = ("stored: dram__bytes_read.sum + dram__bytes_write.sum of one k_sweep2p launch from the ncu "
                       f"--set full capture {tj.get('source', 'profiles/sweep2p_traffic.json')} (not measured in this run)")

    # end-to-end through the public API with HOST buffers: one user job = upload b and x0 from
    # pinned host memory, 200 sweeps (config 4's count), download x; time with events
    e2e = None
    if not args.no_e2e:
        # every rank uploads its slab (b and x0), runs the sweeps (one C call; the library refreshes
        # the ghost layers of b once and of x every sweep), downloads its slab; max over ranks
        hb = torch.from_numpy(b).pin_memory()
        hx = torch.zeros((nl_y, NXl), dtype=torch.float64).pin_memory()
        hout = torch.empty((nl_y, NXl), dtype=torch.float64).pin_memory()
        nsw = 200
        times = []
        for rep in range(2):
            barrier(world)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.set_vector(binding.B, hb)
            g.set_vector(binding.X, hx)
            g.sor_sweep([omega], nsw, 0)
            g.get_vector(binding.X, hout)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        t = max_over_ranks(min(times), world)
        e2e = {"value": round(NXl * ny * nsw / (t * 1e-3) / 1e9, 3), "unit": "GLUP/s",
               "h2d_bytes_per_step": int(2 * NXl * ny * 8) // nsw, "d2h_bytes_per_step": int(NXl * ny * 8) // nsw,
               "step": f"one user job through the C ABI: b and x0 copied H2D from pinned host memory, {nsw} sweeps "
                       f"(config 4's count), x copied D2H; bytes per step = job bytes / {nsw}",
               "h2d_bytes_per_job": int(2 * NXl * ny * 8), "d2h_bytes_per_job": int(NXl * ny * 8),
               "ms_per_job": round(t, 3)}
        if world == 1:
            # a stream of jobs (serving): the same job J times on two grids and two streams, so
            # that job j+1's copies overlap job j's sweeps; every copy of every job is inside the
            # timed region (first upload to last download)
            J = 8
            g2 = binding.Grid(2, n, binding.COEF_POISSON, 0.0, dev).decompose((T, T), rank, world)
            grids = [g, g2]
            strs = [torch.cuda.Stream(), torch.cuda.Stream()]
            houts = [hout, torch.empty((nl_y, NXl), dtype=torch.float64).pin_memory()]
            tp = []
            for rep in range(2):
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for sj in strs:
                    sj.wait_event(e0)
                for j in range(J):
                    gg, sj, ho = grids[j % 2], strs[j % 2], houts[j % 2]
                    gg.set_vector(binding.B, hb, stream=sj.cuda_stream)
                    gg.set_vector(binding.X, hx, stream=sj.cuda_stream)
                    gg.sor_sweep([omega], nsw, 0, stream=sj.cuda_stream)
                    gg.get_vector(binding.X, ho, stream=sj.cuda_stream)
                for sj in strs:
                    stream.wait_stream(sj)
                e1.record(stream)
                torch.cuda.synchronize()
                tp.append(e0.elapsed_time(e1))
            g2.check()
            ok = bool(torch.equal(houts[0], houts[1]) and torch.equal(houts[0], hout))
            tpj = min(tp)
            e2e.update({"value": round(J * NXl * ny * nsw / (tpj * 1e-3) / 1e9, 3),
                        "step": f"a stream of {J} user jobs through the C ABI on two grids / two CUDA streams (job j+1's "
                                f"H2D copies overlap job j's sweeps); each job: b and x0 copied H2D from pinned host "
                                f"memory, {nsw} sweeps (config 4's count), x copied D2H; timed from the first upload "
                                f"to the last download; bytes per step = job bytes / {nsw}",
                        "jobs": J, "ms_per_job": round(tpj / J, 3), "outputs_identical": ok,
                        "single_job": {"value": round(NXl * ny * nsw / (t * 1e-3) / 1e9, 3), "ms": round(t, 3)}})
            del g2, grids

    secondary = None
    if not args.no_secondary:
        del g
        torch.cuda.empty_cache()
        secondary = run_secondary(args) if world == 1 else run_secondary_slabs(args, world, rank, dev, comm)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.seed, args.cpu_n, args.cpu_sweeps)

    if rank == 0:
        line = {
            "metric": "lattice-point sweep updates/sec (GLUP/s), decomposed SOR sweep",
            "value": round(glups, 3), "unit": "GLUP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded U[-1,1) rhs, gen.py)",
            "config": {"workload": ("BASELINE config 4: 2D 5-point Poisson 16384 x 16384*N fp64 (weak scaling)"
                                    if weak else "BASELINE config 4: 2D 5-point Poisson 16384 x 16384 fp64 split over N "
                                                 "GPUs (strong scaling)") + ", 64x64 boxes, SOR omega_opt, row slabs per GPU",
                       "n": [NXl, ny], "tile": [T, T], "omega": omega, "parallelism": f"slab{world}",
                       "comm": None if world == 1 else f"in-library sw_comm ({args.comm}): 2 ghost layers per sweep, "
                                                       f"exchanged behind the interior tile rows",
                       "l2": "inputs (2.1 GB per array) exceed the 126 MB L2; no flush needed"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "traffic_source": traffic_src if traffic is not None else None,
                         "kernel": "k_sweep2p (decomposed SOR, 24 algorithmic B/LUP)" if world == 1 else
                                   "one whole sweep per rank (k_sweep2p boundary + interior launches and the exchange)",
                         "peak_source": peak_src,
                         "kernel_ms": round(kavg, 4), "kernel_ms_event_pair": round(kiso, 4)},
            "e2e": e2e,
            "gpu_launches": launches,
            "cpu_baseline": cpu,
        }
        line["clocks"] = clk.summary()
        if secondary:
            line["secondary"] = secondary
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        del comm
        dist.destroy_process_group()


def _time_sweeps(g, omega, nsw, phase=0):
    import torch
    g.sor_sweep(omega, 3, phase)                     # warm-up
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    g.sor_sweep(omega, nsw, phase + 3)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / nsw


def run_secondary(args):
    """The other BASELINE.json configurations, measured on the same GPU (not the headline):
    config 3 (2D variable coefficients, 4096^2): 100 decomposed SOR sweeps at omega = 1 (R-10)
    and ILU(0)-PCG (SYMMETRIC pairing) to 1e-8; config 5's sweep (3D anisotropic 512^3, boxes
    32 x 8 x 4) at omega = 1 and its ILU(0)-PCG to 1e-8; config 2 (256^2) iteration counts."""
    import torch

    from paper_1008_3699_b200 import binding, gen
    out = {}
    # ---- config 3
    n = 4096
    g = binding.Grid(2, (n, n), binding.COEF_FACES).decompose((64, 64))
    k = gen.lognormal_k(args.seed, (n + 2, n + 2), 1.0)
    g.set_coefficients_k(np.pad(k, [(1, 1), (0, 0)], constant_values=1.0), (1.0, 1.0))
    del k
    b = gen.uniform_field(args.seed, gen.STREAM_RHS, (n, n)) / float((n + 1) ** 2)
    g.set_vector(binding.B, b)
    ms = _time_sweeps(g, [1.0], 100)
    out["c3_sor"] = {"n": [n, n], "sweeps": 100, "ms_per_sweep": round(ms, 4),
                     "glups": round(n * n / (ms * 1e-3) / 1e9, 2), "algorithmic_B_per_lup": 40,
                     "frac_of_measured_hbm": round(40 * n * n / (ms * 1e-3) / 1e9 / peaks()[0], 3)}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it, rel, ok = g.pcg_solve(binding.PC_ILU0, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 20000)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out["c3_pcg_ilu0"] = {"iterations": it, "relres": rel, "converged": ok, "seconds": round(dt, 3),
                          "ms_per_iteration": round(dt / max(it, 1) * 1e3, 4)}
    # multigrid-preconditioned CG with the decomposed sweep as smoother
    g.mg_setup(7, 1, 0.45, 32, 1.8)                 # 7 levels: coarsest 64^2 = one box
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it, rel, ok = g.pcg_solve(binding.PC_MG, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 20000)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out["c3_pcg_mg"] = {"levels": 7, "nu": 1, "theta": 0.45, "nu_coarse": 32, "coarse_scale": 1.8, "iterations": it,
                        "relres": rel, "converged": ok, "seconds": round(dt, 3),
                        "ms_per_iteration": round(dt / max(it, 1) * 1e3, 4)}
    del g, b
    torch.cuda.empty_cache()
    # ---- config 5: boxes span the whole x extent (TILE5 = 512 x 8 x 4): the anisotropy 1 : 0.1 : 0.01 makes x
    # the strong direction, and a box that keeps every x-line whole is the decomposition that preconditions it
    # best (ILU(0)-PCG 772 against 2253 iterations with 32 x 8 x 4 boxes); 32 x 8 x 4 is kept as a
    # comparison line
    n3 = 512
    k = gen.lognormal_k(args.seed, (n3 + 2,) * 3, 0.5)
    k = np.pad(k, [(1, 1), (0, 0), (0, 0)], constant_values=1.0)
    b5 = gen.uniform_field(args.seed, gen.STREAM_RHS, (n3,) * 3) / float((n3 + 1) ** 2)
    for tile5 in (TILE5_CMP, TILE5):
        g = binding.Grid(3, (n3, n3, n3), binding.COEF_FACES).decompose(tile5)
        g.set_coefficients_k(k, (1.0, 0.1, 0.01))
        g.set_vector(binding.B, b5)
        ms = _time_sweeps(g, [1.0], 8)
        key = "c5_sweep" if tile5 == TILE5 else "c5_sweep_32x8x4"
        out[key] = {"n": [n3] * 3, "tile": list(tile5), "ms_per_sweep": round(ms, 3),
                    "glups": round(n3 ** 3 / (ms * 1e-3) / 1e9, 2), "algorithmic_B_per_lup": 48,
                    "frac_of_measured_hbm": round(48 * n3 ** 3 / (ms * 1e-3) / 1e9 / peaks()[0], 3)}
        if tile5 != TILE5:
            if not args.no_c5_pcg:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                it, rel, ok = g.pcg_solve(binding.PC_ILU0, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 5000)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
                out["c5_pcg_ilu0_32x8x4"] = {"tile": list(tile5), "iterations": it, "relres": rel, "converged": ok,
                                             "seconds": round(dt, 3), "ms_per_iteration": round(dt / max(it, 1) * 1e3, 3)}
            del g
            torch.cuda.empty_cache()
    del k, b5
    if not args.no_c5_pcg:
        # config 5's solve: ILU(0)-PCG (SYMMETRIC pairing) to 1e-8 on the full 512^3 grid
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it, rel, ok = g.pcg_solve(binding.PC_ILU0, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 5000)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out["c5_pcg_ilu0"] = {"n": [n3] * 3, "tile": list(TILE5), "iterations": it, "relres": rel, "converged": ok,
                              "seconds": round(dt, 3), "ms_per_iteration": round(dt / max(it, 1) * 1e3, 3)}
        # and SSOR(omega = 1, i.e. SGS; R-10)-PCG, the config's other preconditioner
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it, rel, ok = g.pcg_solve(binding.PC_SSOR, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 5000)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out["c5_pcg_ssor"] = {"n": [n3] * 3, "tile": list(TILE5), "omega": 1.0, "iterations": it, "relres": rel,
                              "converged": ok, "seconds": round(dt, 3),
                              "ms_per_iteration": round(dt / max(it, 1) * 1e3, 3)}
        g.mg_setup(7, 1, 0.35, 4, 1.0, 3)           # semi-coarsening in x and y (alpha_z = 0.01)
        g.mg_set_cycle(2)                           # W-cycle
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it, rel, ok = g.pcg_solve(binding.PC_MG, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 5000)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out["c5_pcg_mg"] = {"tile": list(TILE5), "levels": 7, "nu": 1, "theta": 0.35, "nu_coarse": 4,
                            "coarse_scale": 1.0, "coarsened_axes": "x, y", "cycle": "W",
                            "iterations": it, "relres": rel, "converged": ok, "seconds": round(dt, 3),
                            "ms_per_iteration": round(dt / max(it, 1) * 1e3, 3)}
    del g
    torch.cuda.empty_cache()
    # ---- SURVEY §8(f) N3 / N4 on config 3's grid (4096^2, 64 x 64 boxes): the nine-point sweep
    # (Mehrstellen Laplacian, 56 algorithmic B/LUP: x r/w, b, 2 axis + 2 diagonal coefficient arrays)
    # and the eikonal fast-sweeping pass (24 B/LUP: u r/w, slowness), per-pass time and HBM fraction
    n = 4096
    g9 = binding.Grid(2, (n, n), binding.COEF_FACES).decompose((64, 64))
    F9 = [np.full(tuple(reversed((n + (a == 0), n + (a == 1)))), 4.0) for a in range(2)]
    g9.set_faces_global(F9)
    del F9
    g9.set_diagonals(np.ones((n + 1, n + 1)), np.ones((n + 1, n + 1)))
    g9.set_vector(binding.B, gen.uniform_field(args.seed, gen.STREAM_RHS, (n, n)) / float((n + 1) ** 2))
    ms = _time_sweeps(g9, [1.0], 20)
    out["n3_sweep9"] = {"n": [n, n], "tile": [64, 64], "stencil": "Mehrstellen 9-point", "ms_per_sweep": round(ms, 4),
                        "glups": round(n * n / (ms * 1e-3) / 1e9, 2), "algorithmic_B_per_lup": 56,
                        "frac_of_measured_hbm": round(56 * n * n / (ms * 1e-3) / 1e9 / peaks()[0], 3)}
    del g9
    ge = binding.Grid(2, (n, n)).decompose((64, 64))
    ge.set_slowness(0.5 + gen.uniform_field(args.seed, gen.STREAM_TEST, (n, n)) ** 2, 1.0 / n)
    u0 = np.full((n, n), np.inf)
    u0[n // 3, n // 2] = 0.0
    ge.set_vector(binding.X, u0)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    ph = ge.eikonal_sweep(8, 0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 8
    t0 = time.perf_counter()
    while ge.eikonal_changes() > 0 and ph < 4000:
        ph = ge.eikonal_sweep(8, ph)
    t_fix = time.perf_counter() - t0
    # the same passes once every box has been reached (the full per-node work: no box is skipped as
    # all +inf)
    torch.cuda.synchronize()
    e0.record()
    ge.eikonal_sweep(8, ph)
    e1.record()
    torch.cuda.synchronize()
    ms_all = e0.elapsed_time(e1) / 8
    out["n4_eikonal"] = {"n": [n, n], "tile": [64, 64], "ms_per_pass": round(ms, 4),
                         "glups": round(n * n / (ms * 1e-3) / 1e9, 2), "algorithmic_B_per_lup": 24,
                         "frac_of_measured_hbm": round(24 * n * n / (ms * 1e-3) / 1e9 / peaks()[0], 3),
                         "ms_per_pass_all_reached": round(ms_all, 4),
                         "glups_all_reached": round(n * n / (ms_all * 1e-3) / 1e9, 2),
                         "passes_to_fixed_point": ph, "seconds_to_fixed_point": round(t_fix, 3)}
    del ge, u0
    # ---- config 1: 1D Poisson n = 1024, 4 boxes, SOR at omega_opt until relres < 1e-8
    n1 = 1024
    g1d = binding.Grid(1, (n1,)).decompose((256,))
    g1d.set_vector(binding.B, gen.uniform_field(args.seed, gen.STREAM_RHS, (n1,)) / float((n1 + 1) ** 2))
    from paper_1008_3699_b200 import omega as OM
    t0 = time.perf_counter()
    c1 = OM.sweeps_to_tol(g1d, [OM.omega_opt_poisson(n1)], 1e-8, 100000, 1)
    out["c1_sweeps_to_1e-8"] = {"n": n1, "tile": 256, "omega": round(OM.omega_opt_poisson(n1), 6), "sweeps": c1,
                                "seconds": round(time.perf_counter() - t0, 3)}
    del g1d
    # ---- config 2 iteration counts (256^2 Poisson, 64 x 64 boxes)
    n2 = 256
    g = binding.Grid(2, (n2, n2)).decompose((64, 64))
    b = gen.uniform_field(args.seed, gen.STREAM_RHS, (n2, n2)) / float((n2 + 1) ** 2)
    g.set_vector(binding.B, b)
    res = {}
    for name, pc in (("ilu0", binding.PC_ILU0), ("ssor", binding.PC_SSOR), ("none", binding.PC_NONE)):
        it, rel, ok = g.pcg_solve(pc, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 20000)
        res[f"pcg_{name}"] = it
    # the PAPER pairing (nonsymmetric) with the flexible (Polak-Ribiere) beta it needs
    res["pcg_ilu0_paper_pairing_flexible"], _, _ = g.pcg_solve(binding.PC_ILU0, 1.0, binding.PAIR_PAPER, 1e-8, 20000)
    w = 2.0 / (1.0 + np.sin(np.pi / (n2 + 1)))
    g.set_vector(binding.X, np.zeros((n2, n2)))
    ph, sweeps = 0, 0
    while sweeps < 20000:
        ph = g.sor_sweep([w], 10, ph)
        sweeps += 10
        if g.residual_norm() < 1e-8:
            break
    res["sor_sweeps_to_1e-8 (checked every 10)"] = sweeps
    # m-step SSOR preconditioning, theta = 1/2 (lambda_max(P^-1 A) = 2)
    for m in (2, 3, 4):
        g.set_precond_steps(m, 0.5)
        it, rel, ok = g.pcg_solve(binding.PC_SSOR, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 20000)
        res[f"pcg_ssor_{m}step"] = it
    g.set_precond_steps(1, 1.0)
    g.mg_setup(4, 1, 0.5, 16, 1.2)
    res["pcg_mg"], _, _ = g.pcg_solve(binding.PC_MG, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 20000)
    # the same V-cycle with one box per level (the sequential sweep as smoother): the paper's
    # "no convergence decay" claim for smoothing
    g1 = binding.Grid(2, (n2, n2)).decompose((n2, n2)).mg_setup(4, 1, 0.5, 16, 1.2)
    g1.set_vector(binding.B, b)
    res["pcg_mg_one_box_smoother"], _, _ = g1.pcg_solve(binding.PC_MG, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 20000)
    del g1
    out["c2_iterations"] = res
    # ---- the relaxation-factor search of PAPER:1996-1998 on config 2
    from paper_1008_3699_b200 import omega as OM
    evals = []

    def count(v):
        evals.append(1)
        return OM.sweeps_to_tol(g, v, 1e-8, 20000, 10)
    t0 = time.perf_counter()
    w_best, c_best = OM.refine_search(count, 1.90, 1.999, accuracy=1e-3, coarse=0.01)
    dt = time.perf_counter() - t0
    w_y = OM.omega_opt_poisson(n2)
    out["c2_omega_search"] = {"range": [1.90, 1.999], "accuracy": 1e-3, "best_omega": w_best,
                              "sweeps_at_best": c_best, "young_omega_opt": round(w_y, 6),
                              "sweeps_at_young": OM.sweeps_to_tol(g, [w_y], 1e-8, 20000, 10),
                              "evaluations": len(evals), "seconds": round(dt, 3)}
    return out


def k_slab_c5(seed, n3, z0, nz):
    """Config 5's node diffusivities k = exp(0.5 N(0,1)) on the (n3 + 2)^3 ring grid (gen.lognormal_k),
    cut to the layout sw_set_coefficients_k wants for the z slab [z0, z0 + nz): the one-node ring on
    x and y, z coordinates z0 - 2 .. z0 + nz + 1 (ring rows outside 0 .. n3 + 1 are ignored: 1.0)."""
    from paper_1008_3699_b200 import gen
    m = n3 + 2
    out = np.ones((nz + 4, m, m))
    lo, hi = max(z0 - 1, 0), min(z0 + nz + 3, m)          # ring rows = coordinate + 1
    rows = gen.normal(seed, gen.STREAM_LOGK, (hi - lo) * m * m, start=lo * m * m).reshape(hi - lo, m, m)
    out[lo - (z0 - 1):hi - (z0 - 1)] = np.exp(0.5 * rows)
    return out


def run_secondary_slabs(args, world, rank, dev, comm):
    """Config 5 slab-sharded over the N GPUs (BASELINE.json: "slab-sharded over 8 GPUs, SSOR- and
    ILU(0)-preconditioned CG"): z slabs of 512 / N planes, boxes TILE5 (512 x 8 x 4), the library's
    communicator for the ghost layers and the rank-ordered reductions.  Sweep GLUP/s (all ranks'
    nodes / max-over-ranks time), then ILU(0)- and SSOR(1)-PCG to 1e-8."""
    import torch

    from paper_1008_3699_b200 import binding, gen
    n3 = 512
    g = binding.Grid(3, (n3, n3, n3), binding.COEF_FACES, 0.0, dev).decompose(TILE5, rank, world, comm)
    z0, nz = g.slab_offset, g.n_local[2]
    g.set_coefficients_k(k_slab_c5(args.seed, n3, z0, nz), (1.0, 0.1, 0.01))
    b = gen.uniform(args.seed, gen.STREAM_RHS, nz * n3 * n3, start=z0 * n3 * n3).reshape(nz, n3, n3)
    g.set_vector(binding.B, b / float((n3 + 1) ** 2))
    out = {}
    g.sor_sweep([1.0], 3, 0)
    barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    g.sor_sweep([1.0], 8, 3)
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world) / 8
    out["c5_sweep_slabs"] = {"n": [n3] * 3, "tile": list(TILE5), "ranks": world, "planes_per_rank": nz,
                             "ms_per_sweep": round(ms, 3), "glups": round(n3 ** 3 / (ms * 1e-3) / 1e9, 2),
                             "glups_per_gpu": round(n3 ** 3 / world / (ms * 1e-3) / 1e9, 2)}
    if not args.no_c5_pcg:
        for name, pc in (("ilu0", binding.PC_ILU0), ("ssor", binding.PC_SSOR)):
            barrier(world)
            t0 = time.perf_counter()
            it, rel, ok = g.pcg_solve(pc, 1.0, binding.PAIR_SYMMETRIC, 1e-8, 5000)
            torch.cuda.synchronize()
            dt = max_over_ranks(time.perf_counter() - t0, world)
            out[f"c5_pcg_{name}_slabs"] = {"ranks": world, "iterations": it, "relres": rel, "converged": ok,
                                           "seconds": round(dt, 3), "ms_per_iteration": round(dt / max(it, 1) * 1e3, 3)}
    del g
    return out


def host_cpu():
    """CPU model and thread count of the host the oracle ran on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def cpu_baseline(seed, n, sweeps):
    """The oracle as it stands, single-threaded, on an n x n sample of the same workload."""
    import oracle as O
    pb = O.tiled((n, n), (64, 64))
    h = 1.0 / (NX + 1)
    b = rhs_slab(seed, n, 0, n, h)
    x = np.zeros(pb.shape)
    t0 = time.perf_counter()
    for k in range(sweeps):
        x = O.sweep(pb, [2.0 / (1.0 + np.sin(np.pi * h))], x, b, phase=k)
    dt = time.perf_counter() - t0
    return {"value": round(n * n * sweeps / dt / 1e9, 6), "unit": "GLUP/s", "cores": 1, "kind": "oracle",
            "sample": f"{sweeps} decomposed SOR sweeps on a {n}x{n} sub-grid (64x64 boxes), same per-node work",
            "seconds": round(dt, 3), "host": host_cpu()}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    n = args.ref_n
    pb = O.tiled((n, n), (64, 64))
    h = 1.0 / (NX + 1)
    b = rhs_slab(args.seed, n, 0, n, h)
    w = [2.0 / (1.0 + np.sin(np.pi * h))]
    x = np.zeros(pb.shape)
    for k in range(args.warmup):
        x = O.sweep(pb, w, x, b, phase=k)
    t0 = time.perf_counter()
    for k in range(args.steps):
        x = O.sweep(pb, w, x, b, phase=k)
    dt = time.perf_counter() - t0
    v = n * n * args.steps / dt / 1e9
    line = {"impl": "reference", "metric": "lattice-point sweep updates/sec (GLUP/s), decomposed SOR sweep",
            "value": round(v, 6), "unit": "GLUP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded U[-1,1) rhs, gen.py)",
            "config": {"workload": "BASELINE config 4 sweep, bounded CPU sample", "n": [n, n], "tile": [64, 64]},
            "cpu_baseline": {"value": round(v, 6), "unit": "GLUP/s", "cores": 1, "kind": "oracle",
                             "sample": f"each step = 1 sweep of a {n}x{n} sub-grid of config 4", "host": host_cpu()},
            "e2e": {"value": round(v, 6), "unit": "GLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-n", type=int, default=4096)
    ap.add_argument("--cpu-sweeps", type=int, default=2)
    ap.add_argument("--ref-n", type=int, default=1024)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-c5-pcg", action="store_true", help="skip config 5's 512^3 PCG solves (about a minute)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="config 4 over N GPUs: weak = 16384 x 16384 per GPU, strong = 16384^2 split over N")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "host"],
                    help="N > 1 transport: nccl (one GPU per rank) or host (gloo staging; ranks may share a GPU, tests)")
    ap.add_argument("--nx", type=int, default=NX, help="config 4 edge (tests only; the bench line is 16384)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
