#!/bin/bash
# streaming 3D engine with the x-edge warp: parity subset, timings, ILU(0)-PCG at 512x8x4 (under gpurun)
set -u
TAG=${1:-e3x}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_sweep3s.py -q -x --timeout 120 > $OUT/pytest.log 2>&1; echo "pytest sweep3s exit $?"; tail -3 $OUT/pytest.log
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_degenerate.py tests/test_gpu_msteps.py -q -x --timeout 120 -k "3" > $OUT/pytest3.log 2>&1; echo "pytest 3d exit $?"; tail -3 $OUT/pytest3.log
for T in "512 8 4" "256 8 4" "64 8 4"; do
  timeout 60 python tools/profile_case.py --dim 3 --n 512 --tile $T --faces --sweeps 8 2>&1 | tail -1
done
timeout 120 python tools/profile_case.py --dim 3 --n 512 --tile 512 8 4 --faces --pcg --pc 2 --maxit 5000 2>&1 | tail -1
