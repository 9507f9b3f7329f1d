#!/bin/bash
mkdir -p gpurun_out/exp3r
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep3r -s 1 -c 1 -o gpurun_out/exp3r/k3r python tools/profile_case.py --dim 3 --n 512 --tile 32 8 4 --faces --sweeps 2 > gpurun_out/exp3r/ncu.log 2>&1
for v in "SW_EXP_NOSTG"; do
  SW_DEFINES="$v" python -c "from paper_1008_3699_b200 import build; build.build(force=True, jitter=False)" || exit 1
  echo "== [$v] $(python tools/profile_case.py --dim 3 --n 512 --tile 32 8 4 --faces --sweeps 8 2>&1 | tail -1)"
done
