"""Race detection without compute-sanitizer (closed on the GPU pool): the parity suites re-run on
the race-exposure build libsweep_jitter.so (-DSW_JITTER, csrc/common.cuh), in which every thread
sleeps a pseudo-random 0-1023 ns after every barrier, mbarrier wait and flag acquire and at kernel
start, under three seeds.  Warps, and the lanes of a warp, then reach the shared-memory hand-offs
of the wavefronts (k_sweep2p / k_sweep2v in-place predicated updates, k_sweep3's release/acquire
x-edge hand-off and named barrier, k_sweep3s's producer/consumer batches behind a named barrier
and its TMA chunk ring, the k_tri2t / k_tri3t lane groups, k_generic's levels) in
orders the normal build never produces; a missing barrier shows up as a result that is no longer
bitwise equal to the oracle.  (SURVEY.md §5 race detection.)"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["tests/test_gpu_parity.py", "tests/test_gpu_degenerate.py", "tests/test_gpu_msteps.py", "tests/test_gpu_eikonal.py",
          "tests/test_gpu_ninepoint.py", "tests/test_gpu_sweep3s.py"]


@pytest.mark.parametrize("seed", [1, 7, 12345])
def test_parity_suites_under_schedule_jitter(seed):
    lib = os.path.join(ROOT, "paper_1008_3699_b200", "libsweep_jitter.so")
    assert os.path.exists(lib), "race-exposure build missing: run paper_1008_3699_b200.build.build()"
    env = dict(os.environ, SW_LIBRARY="libsweep_jitter.so", SW_JITTER_SEED=str(seed), SW_NO_GRAPH="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider", *SUITES]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT, env=env)
    out = os.path.join(ROOT, "gpurun_out", "jitter")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, f"seed{seed}.log"), "w") as f:
        f.write(res.stdout + res.stderr)
    assert res.returncode == 0, (res.stdout + res.stderr)[-4000:]
    assert " passed" in res.stdout
