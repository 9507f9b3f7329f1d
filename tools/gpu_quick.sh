#!/bin/bash
# quick GPU check: build, parity tests (-k filter), one timing case
set -u
TAG=${1:-q}; K=${2:-""}; shift 2 || true
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q --timeout 180 -k "$K" > $OUT/pytest_gpu.log 2>&1; else timeout 900 python -m pytest tests -m gpu -x -q --timeout 180 > $OUT/pytest_gpu.log 2>&1; fi
echo "pytest exit $?"; tail -15 $OUT/pytest_gpu.log
for c in "$@"; do echo "== $c"; timeout 300 python tools/profile_case.py $c 2>&1 | tail -3; done
