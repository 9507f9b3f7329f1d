"""Race detection: compute-sanitizer racecheck, synccheck and memcheck over every
hot-path kernel on small grids (tools/sanitize_case.py), failing on any reported hazard or error.
The shared-memory wavefronts (k_sweep2p / k_sweep2v in-place predicated updates, k_sweep3's
release/acquire hand-off between warps, k_tri2t / k_tri3t lane groups) are exactly what bitwise
parity on one schedule cannot prove race-free.  Logs go to gpurun_out/sanitizer/ (copied to
profiles/ by hand)."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
GROUPS = ["2d", "3d", "generic", "blas", "mg"]
TOOLS = ["racecheck", "synccheck", "memcheck"]


@pytest.mark.parametrize("tool", TOOLS)
@pytest.mark.parametrize("group", GROUPS)
def test_sanitizer_clean(tool, group):
    if not os.path.exists(CS):
        pytest.fail("compute-sanitizer not found")
    outdir = os.path.join(ROOT, "gpurun_out", "sanitizer")
    os.makedirs(outdir, exist_ok=True)
    cmd = [CS, "--tool", tool, "--error-exitcode", "99"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py"), group]
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT, env=env)
    log = res.stdout + res.stderr
    with open(os.path.join(outdir, f"{tool}_{group}.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + log)
    assert f"sanitize case {group} done" in log, log[-3000:]
    if tool == "racecheck":
        m = re.search(r"RACECHECK SUMMARY: (\d+) hazards? displayed \((\d+) errors?, (\d+) warnings?\)", log)
        assert m is not None or "ERROR SUMMARY: 0 errors" in log, log[-3000:]
        if m:
            assert m.group(1) == "0", log[-3000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in log, log[-3000:]
    assert res.returncode == 0, log[-3000:]
