#!/bin/bash
# streaming 3D engine: ncu of one 512x8x4 launch + phase trace (usage under gpurun)
set -u
TAG=${1:-e3t}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
ARGS="--dim 3 --n 512 --tile 512 8 4 --faces --sweeps 4"
#timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep3s -s 2 -c 1 -o $OUT/prof python tools/profile_case.py $ARGS > $OUT/ncu.log 2>&1; echo "ncu exit $?"
SW_TRACE=1 python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build_trace.log 2>&1 || { echo TRACE BUILD FAILED; exit 1; }
timeout 60 python tools/phase_trace3s.py 512 512x8x4 2>&1 | tail -14
