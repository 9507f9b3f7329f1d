#!/bin/bash
set -u
TAG=${1:-e3tri}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep3s.py tests/test_gpu_degenerate.py tests/test_gpu_msteps.py -q -x --timeout 200 > $OUT/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $OUT/pytest.log
timeout 120 python tools/profile_case.py --dim 3 --n 512 --tile 512 8 4 --faces --pcg --pc 2 --maxit 5000 2>&1 | tail -1
SW_PCG_HOSTLOOP=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/profile_case.py --dim 3 --n 512 --tile 512 8 4 --faces --pcg --pc 2 --maxit 4 > $OUT/ncu.log 2>&1; echo "ncu exit $?"
