"""bench.py's JSON contract on the CPU (-m "not gpu"): the reference arm (the oracle timed on the
host cores) prints one line with the keys the driver reads, and the ours-arm flags parse."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_the_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--ref-n", "128"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "GLUP/s" and d["value"] > 0
    assert d["steps"] == 1 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_bench_help_lists_the_driver_flags():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True,
                         timeout=120, cwd=ROOT)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl"):
        assert flag in out.stdout


def test_c5_slab_coefficients_match_the_single_grid_layout():
    """bench.k_slab_c5 (config 5's k for one z slab, generated with counter offsets) equals the cut of
    the single-grid array bench.py's one-GPU leg builds (gen.lognormal_k padded by one z layer)."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    from paper_1008_3699_b200 import gen
    n3 = 8
    full = np.pad(gen.lognormal_k(3, (n3 + 2,) * 3, 0.5), [(1, 1), (0, 0), (0, 0)], constant_values=1.0)
    for z0, nz in ((0, 4), (4, 4), (2, 2), (0, 8)):
        assert np.array_equal(bench.k_slab_c5(3, n3, z0, nz), full[z0:z0 + nz + 4])
