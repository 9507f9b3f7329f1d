#!/bin/bash
# N3 / N4 kernels: parity subset, timing (tools/time_next.py), then the SW_TRACE phase clocks
set -u
TAG=${1:-n34}; K=${2:-"ninepoint or eikonal"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q --timeout 180 -k "$K" > $OUT/pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python tools/time_next.py 2>&1 | tail -5 | tee $OUT/time_next.txt
SW_TRACE=1 python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build_trace.log 2>&1 || { echo TRACE BUILD FAILED; tail -5 $OUT/build_trace.log; exit 1; }
timeout 60 python tools/phase_trace9.py 2>&1 | tail -6 | tee $OUT/trace9.txt
timeout 60 python tools/phase_trace_eik.py 2>&1 | tail -6 | tee $OUT/trace_eik.txt; timeout 120 python tools/phase_trace_eik.py reached 2>&1 | tail -6 | tee $OUT/trace_eik_reached.txt
