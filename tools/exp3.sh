#!/bin/bash
# timing-only variants of k_sweep3 (tools: wrong results), 512^3 faces 32x8x4
mkdir -p gpurun_out/exp3
for v in "" "SW_EXP_NOWAIT" "SW_EXP_NOCORNER" "SW_EXP_NOSHEET" "SW_EXP_NOLOAD" "SW_EXP_NOWAIT SW_EXP_NOCORNER SW_EXP_NOSHEET" "SW_EXP_NOWAIT SW_EXP_NOCORNER SW_EXP_NOSHEET SW_EXP_NOLOAD"; do
  SW_DEFINES="$v" python -c "from paper_1008_3699_b200 import build; build.build(force=True, jitter=False)" || exit 1
  echo "== [$v] $(python tools/profile_case.py --dim 3 --n 512 --tile 32 8 4 --faces --sweeps 8 2>&1 | tail -1)"
done
