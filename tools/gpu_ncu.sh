#!/bin/bash
# ncu --set full of one kernel on one profile_case invocation: bash tools/gpu_ncu.sh TAG REGEX "profile_case args"
set -u
TAG=$1; RX=$2; ARGS=$3; SKIP=${4:-2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python tools/profile_case.py $ARGS > $OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -s $SKIP -c 1 -o $OUT/prof python tools/profile_case.py $ARGS > $OUT/ncu.log 2>&1
echo "ncu exit $?"; cat $OUT/plain.log | tail -2
