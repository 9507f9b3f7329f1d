#!/bin/bash
# k_sweep9: keeping the producer / explicit-part work off the scheduler of the serial warp
set -u
TAG=${1:-expg}
OUT=gpurun_out/$TAG; mkdir -p $OUT
bld() { SW_TRACE=${2:-0} SW_DEFINES="$1" python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build.log 2>&1 || { echo "BUILD FAILED $1"; tail -5 $OUT/build.log; }; }
for d in "" "SW_S9_SKIPW4=0" "SW_S9_EXPL6=1"; do
echo "== [$d]"; bld "$d"
timeout 300 python -m pytest tests/test_gpu_ninepoint.py -m gpu -q 2>&1 | tail -1
timeout 200 python tools/time_next.py 2>&1 | head -1
done
for d in "" "SW_S9_EXPL6=1"; do
echo "== trace [$d]"; bld "$d" 1
timeout 120 python tools/phase_trace9.py 2>&1 | tail -6
done
