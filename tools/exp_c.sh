#!/bin/bash
# k_sweep9 wavefront: what the per-lane cp.async coefficient ring costs (timing-only builds)
set -u
TAG=${1:-expc}
OUT=gpurun_out/$TAG; mkdir -p $OUT
bld() { SW_TRACE=${2:-0} SW_DEFINES="$1" python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build.log 2>&1 || { echo "BUILD FAILED $1"; tail -5 $OUT/build.log; }; }
for d in "" "SW_S9_NOFETCH" "SW_S9_NOWAIT" $EXTRA; do
echo "== trace [$d]"; bld "$d" 1
timeout 120 python tools/phase_trace9.py 2>&1 | tail -7
done
