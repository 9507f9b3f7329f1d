#!/bin/bash
# Look-ahead L2 prefetch experiments (k_sweep2v: SW_V2_AHEAD) and 16 prologue warps.  The k_sweep2p switches
# (SW_P2_AHEAD, SW_P2_SWAP) measured slower and were removed from the kernel (profiles/r02_ahead_experiments.txt);
# the script is kept as the record of what was run.
# usage (under gpurun): bash tools/exp_ahead.sh TAG
set -u
TAG=${1:-ahead}
OUT=gpurun_out/$TAG; mkdir -p $OUT
run() {  # name, defines
    SW_DEFINES="$2" python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build_$1.log 2>&1 || { echo "BUILD FAILED $1"; tail -5 $OUT/build_$1.log; return; }
    echo "== $1: $2"
    timeout 300 python tools/t2v.py 2>&1 | tail -4
    timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('2p', d['value'], d['roofline']['frac'], d['clocks'])"
}
run base "SW_V2_AHEAD=0 SW_P2_AHEAD=0"
run a296 "SW_V2_AHEAD=296 SW_P2_AHEAD=888"
run a148 "SW_V2_AHEAD=148 SW_P2_AHEAD=1776"
run a592 "SW_V2_AHEAD=592 SW_P2_AHEAD=444"
run nw16 "SW_V2_AHEAD=296 SW_V2_NW=16 SW_V2_RING=2 SW_P2_AHEAD=2664"
run swap "SW_V2_AHEAD=0 SW_P2_SWAP=1"
run swap_a "SW_V2_AHEAD=296 SW_V2_RING=2 SW_P2_SWAP=1 SW_P2_AHEAD=888"
# parity of the default build
python -c "from paper_1008_3699_b200 import build as b; b.build(force=True, jitter=False)" > $OUT/build_default.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_degenerate.py -m gpu -q -x 2>&1 | tail -3
