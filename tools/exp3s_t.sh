#!/bin/bash
set -u
python -c "import __graft_entry__ as g; g.build()" > /tmp/b.log 2>&1 || { echo BUILD FAILED; tail -20 /tmp/b.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_degenerate.py -q --timeout 300 -k "${1:-n1}" 2>&1 | grep -E "passed|failed|FAILED|Error" | head -30
