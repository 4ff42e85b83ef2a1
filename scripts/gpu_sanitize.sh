#!/bin/bash
# compute-sanitizer over every operator (scripts/sanitize_smoke.py: both precisions, direction
# blocks, the differentiable path) with memcheck / synccheck / racecheck, and memcheck +
# synccheck over the whole GPU suite. Summaries into gpurun_out/sanitizer/.
cd "$(dirname "$0")/.."
S=gpurun_out/sanitizer
mkdir -p $S
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 python scripts/sanitize_smoke.py > $S/smoke_$tool.txt 2>&1
  echo "smoke $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $S/smoke_$tool.txt | tail -1)"
done
for tool in memcheck synccheck; do
  timeout 2400 $CS --tool $tool --print-limit 20 python -m pytest tests -q -m gpu -p no:cacheprovider -x \
    > $S/pytest_$tool.txt 2>&1
  echo "pytest $tool rc=$? $(grep -E 'ERROR SUMMARY' $S/pytest_$tool.txt | tail -1) $(grep -E 'passed|failed' $S/pytest_$tool.txt | tail -1)"
done
