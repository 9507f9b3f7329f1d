#!/bin/bash
# config-5 box shapes: decomposed SOR sweep rate and ILU(0)-/SSOR-PCG (usage under gpurun)
set -u
TAG=${1:-e3b}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
for T in "32 8 4" "512 8 4" "256 8 4" "128 8 4" "512 4 8"; do
  echo "== tile $T"
  timeout 60 python tools/profile_case.py --dim 3 --n 512 --tile $T --faces --sweeps 8 2>&1 | tail -1
  timeout 120 python tools/profile_case.py --dim 3 --n 512 --tile $T --faces --pcg --pc 2 --maxit 5000 2>&1 | tail -1
done
