#!/bin/bash
# One GPU session: parity tests, smoke, bench, launch list, ncu --set full of the bench's top kernel.
# usage (under gpurun): bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"; tail -2 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"; cat $OUT/bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref exit $?"; cat $OUT/bench_ref.json
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-secondary"
timeout 300 $CMD > $OUT/plain_launch.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "ncu launches exit $?"
timeout 300 $CMD > $OUT/plain_prof.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep2p -s 4 -c 1 -o $OUT/sweep2p $CMD > $OUT/ncu_full.log 2>&1
echo "ncu full exit $?"
# config 5's engine: one k_sweep3s launch at 512^3 with 512x8x4 boxes
ARGS5="--dim 3 --n 512 --tile 512 8 4 --faces --sweeps 4"
timeout 120 python tools/profile_case.py $ARGS5 > $OUT/plain_c5.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep3s -s 2 -c 1 -o $OUT/sweep3s $(echo python tools/profile_case.py $ARGS5) > $OUT/ncu_c5.log 2>&1
echo "ncu c5 exit $?"
