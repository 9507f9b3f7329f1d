#!/bin/bash
# ncu --set full of k_sweep9 and of k_eik2 (every box reached): bash tools/exp_ncu_next.sh TAG
set -u
TAG=${1:-ncn}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python tools/prof_next.py nine > $OUT/nine.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep9 -s 2 -c 1 -o $OUT/sweep9 python tools/prof_next.py nine > $OUT/ncu9.log 2>&1
echo "ncu9 exit $?"
timeout 300 python tools/prof_next.py eik > $OUT/eik.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eik2 -s 472 -c 1 -o $OUT/eik2 python tools/prof_next.py eik > $OUT/ncue.log 2>&1
echo "ncue exit $?"; tail -2 $OUT/eik.log
