#!/bin/bash
# streaming 3D kernel: phase trace (SW_TRACE build) and timings by box shape (usage under gpurun)
set -u
TAG=${1:-e3t}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
for T in "256 8 4" "128 8 4" "512 8 4" "64 8 4"; do
  timeout 120 python tools/profile_case.py --dim 3 --n 512 --tile $T --faces --sweeps 8 2>&1 | tail -1
done
SW_TRACE=1 python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build_trace.log 2>&1 || { echo TRACE BUILD FAILED; tail -5 $OUT/build_trace.log; exit 1; }
for T in 256x8x4 32x8x4; do timeout 120 python tools/phase_trace3s.py 512 $T 2>&1 | tail -16; done
