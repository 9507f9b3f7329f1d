#!/bin/bash
for v in "SW_RB=2" "SW_RB=3" "SW_RB=4" "SW_RB=6" "SW_RB=3 SW_KB=3"; do
  SW_DEFINES="$v" python -c "from paper_1008_3699_b200 import build; build.build(force=True, jitter=False)" || exit 1
  grep -A3 "k_sweep3ILb1ELi1" paper_1008_3699_b200/ptxas.log | grep -E "spill|Used" | tr '\n' ' '
  echo "== [$v] $(SW_NO_ROLL=1 python tools/profile_case.py --dim 3 --n 512 --tile 32 8 4 --faces --sweeps 8 2>&1 | tail -1)"
done
