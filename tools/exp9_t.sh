#!/bin/bash
set -u
TAG=${1:-e9t}
OUT=gpurun_out/$TAG; mkdir -p $OUT
SW_TRACE=1 python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build_trace.log 2>&1 || { echo TRACE BUILD FAILED; tail -5 $OUT/build_trace.log; exit 1; }
timeout 60 python tools/phase_trace9.py 2>&1 | tail -6
