#!/bin/bash
# GPU session: build, parity tests (optionally -k filter), then sanitizer tests.
# usage (under gpurun): bash tools/gpu_check.sh TAG [pytest -k expr] [extra pytest files...]
set -u
TAG=${1:-chk}; K=${2:-""}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1; lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
if [ -n "$K" ]; then
  timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -k "$K" > $OUT/pytest_gpu.log 2>&1
else
  timeout 1800 python -m pytest tests -m gpu -q --timeout 300 --ignore=tests/test_gpu_sanitizer.py > $OUT/pytest_gpu.log 2>&1
fi
echo "pytest exit $?"; tail -25 $OUT/pytest_gpu.log
