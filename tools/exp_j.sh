#!/bin/bash
# look-ahead distances of k_sweep9 / k_eik2
set -u
TAG=${1:-expj}
OUT=gpurun_out/$TAG; mkdir -p $OUT
bld() { SW_DEFINES="$1" python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build.log 2>&1 || { echo "BUILD FAILED $1"; tail -5 $OUT/build.log; }; }
for d in "SW_S9_AHEAD=148 SW_EK_AHEAD=222" "SW_S9_AHEAD=296 SW_EK_AHEAD=444" "SW_S9_AHEAD=185 SW_EK_AHEAD=278" "SW_S9_AHEAD=259 SW_EK_AHEAD=388"; do
echo "== [$d]"; bld "$d"
timeout 200 python tools/time_next.py 2>&1 | grep -v "fixed point"
done
