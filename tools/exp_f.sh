#!/bin/bash
# k_sweep9 producer ring variants: parity then timing / phase clocks per variant
set -u
TAG=${1:-expf}
OUT=gpurun_out/$TAG; mkdir -p $OUT
bld() { SW_TRACE=${2:-0} SW_DEFINES="$1" python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build.log 2>&1 || { echo "BUILD FAILED $1"; tail -5 $OUT/build.log; }; }
bld ""
timeout 600 python -m pytest tests/test_gpu_ninepoint.py tests/test_gpu_eikonal.py -m gpu -q 2>&1 | tail -3
for d in "" "SW_S9_AHEAD=0" "SW_S9_OLDCHAIN" "SW_S9_AHEAD_AT=4" "SW_S9_AHEAD_AT=8" "SW_EK_AHEAD=0"; do
echo "== [$d]"; bld "$d"
timeout 200 python tools/time_next.py 2>&1 | grep -v "fixed point"
done
for d in "" "SW_S9_OLDCHAIN"; do
echo "== trace [$d]"; bld "$d" 1
timeout 120 python tools/phase_trace9.py 2>&1 | tail -6
done
