#!/bin/bash
# one GPU iteration: parity tests (optionally a -k filter), smoke, then a bench sweep (SWEEP as in gpu_sweep.sh)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
grep -E "passed|failed|Error|assert" gpurun_out/gpu_tests.log | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
[ -n "$SWEEP" ] && bash scripts/gpu_sweep.sh
python -c "
import json; d=json.load(open('gpurun_out/parity_errors.json')); print('max parity err', max(v['max_norm_err'] for v in d.values() if 'fallback_points' not in v))"
