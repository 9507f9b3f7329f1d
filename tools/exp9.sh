#!/bin/bash
set -u
TAG=${1:-e9}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 400 python -m pytest tests/test_gpu_ninepoint.py -q -x --timeout 200 > $OUT/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $OUT/pytest.log
bash tools/exp9_t.sh ${TAG}t
