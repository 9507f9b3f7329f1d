#!/bin/bash
set -u
TAG=${1:-eeik}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 400 python -m pytest tests/test_gpu_eikonal.py -q -x --timeout 200 > $OUT/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $OUT/pytest.log
timeout 60 python tools/time_eik.py 2>&1 | tail -1
