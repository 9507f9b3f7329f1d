#!/bin/bash
set -u
TAG=${1:-expi}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "from paper_1008_3699_b200 import build as b; b.build(force=True)" > $OUT/build.log 2>&1 || { echo "BUILD FAILED"; tail -5 $OUT/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_ninepoint.py -m gpu -q 2>&1 | tail -1
timeout 200 python tools/time_next.py 2>&1 | head -1
for sd in 1 7; do SW_LIBRARY=libsweep_jitter.so SW_JITTER_SEED=$sd SW_NO_GRAPH=1 timeout 600 python -m pytest tests/test_gpu_ninepoint.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1; done
timeout 200 python tools/time_next.py 2>&1 | head -1
