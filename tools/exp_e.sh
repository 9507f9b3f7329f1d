#!/bin/bash
# k_sweep9 with producer warps filling the coefficient ring: parity (normal + jitter), timing, phase clocks
set -u
TAG=${1:-expe}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "from paper_1008_3699_b200 import build as b; b.build(force=True)" > $OUT/build.log 2>&1 || { echo "BUILD FAILED"; tail -5 $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_ninepoint.py -m gpu -q 2>&1 | tail -5
timeout 200 python tools/time_next.py 2>&1 | head -1
for sd in 1 7; do SW_LIBRARY=libsweep_jitter.so SW_JITTER_SEED=$sd SW_NO_GRAPH=1 timeout 600 python -m pytest tests/test_gpu_ninepoint.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2; done
SW_TRACE=1 python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build_t.log 2>&1
timeout 120 python tools/phase_trace9.py 2>&1 | tail -6
