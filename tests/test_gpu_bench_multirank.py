"""bench.py's N > 1 path, run as torchrun would launch it (2 ranks), on the one GPU of the test box:
the ranks share the GPU, so the library's host transport (gloo staging, --comm host) stands in for
NCCL; everything else -- the slab split, one sw_sor_sweep call per timed region with the exchange
behind the interior rows, max-over-ranks timing, the e2e job, config 5 slab-sharded -- is the code
the 8-GPU run executes.  Checks the JSON contract of the line rank 0 prints."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks_host_transport(scaling):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--comm", "host", "--steps", "4",
           "--warmup", "3", "--no-cpu", "--nx", "4096", "--scaling", scaling, "--no-c5-pcg"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-4000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 4 and d["scaling"] == scaling and d["value"] > 0
    assert d["config"]["n"] == ([4096, 8192] if scaling == "weak" else [4096, 4096])
    assert d["gpu_launches"] >= 4 * 3                        # boundary rows x 2 + interior per sweep
    assert d["e2e"]["value"] > 0
    sec = d["secondary"]["c5_sweep_slabs"]
    assert sec["ranks"] == 2 and sec["planes_per_rank"] == 256 and sec["glups"] > 0
