#!/bin/bash
# phase clocks of k_sweep2v (look-ahead on / off) and k_sweep9; look-ahead distances; k_sweep9<64> timing
set -u
TAG=${1:-expb}
OUT=gpurun_out/$TAG; mkdir -p $OUT
bld() { SW_TRACE=${2:-0} SW_DEFINES="$1" python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build.log 2>&1 || { echo "BUILD FAILED $1"; tail -5 $OUT/build.log; }; }
echo "== trace, defaults"; bld "" 1
timeout 120 python tools/phase_trace.py 4096 faces 2>&1 | tail -12
timeout 120 python tools/phase_trace9.py 2>&1 | tail -7
timeout 120 python tools/phase_trace_eik.py reached 2>&1 | tail -8
echo "== trace, SW_V2_AHEAD=0"; bld "SW_V2_AHEAD=0" 1
timeout 120 python tools/phase_trace.py 4096 faces 2>&1 | tail -12
for a in 222 259 333 370; do echo "== SW_V2_AHEAD=$a"; bld "SW_V2_AHEAD=$a"; timeout 200 python tools/t2v.py 2>&1 | tail -2; done
echo "== defaults"; bld ""
timeout 200 python tools/t2v.py 2>&1 | tail -2
timeout 200 python tools/time_next.py 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_ninepoint.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
