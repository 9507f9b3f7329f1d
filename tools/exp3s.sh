#!/bin/bash
# streaming 3D kernel: parity subset + timing against k_sweep3 (usage under gpurun: bash tools/exp3s.sh TAG [pytest files])
set -u
TAG=${1:-e3s}; shift || true
FILES=${@:-tests/test_gpu_parity.py tests/test_gpu_degenerate.py}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest $FILES -q -x --timeout 600 > $OUT/pytest.log 2>&1; echo "pytest exit $?"; tail -15 $OUT/pytest.log
for T in "32 8 4" "16 8 4"; do
  timeout 120 python tools/profile_case.py --dim 3 --n 512 --tile $T --faces --sweeps 8 2>&1 | tail -1
  SW_SWEEP3=old timeout 120 python tools/profile_case.py --dim 3 --n 512 --tile $T --faces --sweeps 8 2>&1 | tail -1
done
timeout 120 python tools/profile_case.py --dim 3 --n 256 --tile 32 8 4 --sweeps 8 2>&1 | tail -1
