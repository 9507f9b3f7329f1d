#!/bin/bash
# eikonal register wavefront: parity (normal + jitter), timing, phase clocks
set -u
TAG=${1:-expd}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "from paper_1008_3699_b200 import build as b; b.build(force=True)" > $OUT/build.log 2>&1 || { echo "BUILD FAILED"; tail -5 $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_eikonal.py -m gpu -q 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_jitter.py -m gpu -q -k "eik" 2>&1 | tail -3
timeout 200 python tools/time_next.py 2>&1 | tail -4
SW_TRACE=1 python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build_t.log 2>&1
timeout 120 python tools/phase_trace_eik.py reached 2>&1 | tail -5
