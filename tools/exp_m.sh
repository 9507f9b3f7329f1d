#!/bin/bash
# k_sweep3s: ring entries split into two arrays of 16-byte halves (bank groups)
set -u
TAG=${1:-expm}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "from paper_1008_3699_b200 import build as b; b.build(force=True)" > $OUT/build.log 2>&1 || { echo "BUILD FAILED"; tail -5 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_sweep3s.py -m gpu -q 2>&1 | tail -2
timeout 300 python tools/profile_case.py --dim 3 --n 512 --tile 512 8 4 --faces --sweeps 8 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q 2>&1 | tail -2
for sd in 7; do SW_LIBRARY=libsweep_jitter.so SW_JITTER_SEED=$sd SW_NO_GRAPH=1 timeout 600 python -m pytest tests/test_gpu_sweep3s.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1; done
