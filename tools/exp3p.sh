#!/bin/bash
# config-5 ILU(0)-PCG at 512x8x4: per-kernel launch list of a few iterations (ncu durations, under gpurun)
set -u
TAG=${1:-e3p}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
ARGS="--dim 3 --n 512 --tile 512 8 4 --faces --pcg --pc 2 --maxit 4"
timeout 120 python tools/profile_case.py $ARGS > $OUT/plain.log 2>&1; cat $OUT/plain.log | tail -1
SW_PCG_HOSTLOOP=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/profile_case.py $ARGS > $OUT/ncu.log 2>&1; echo "ncu exit $?"
