#!/bin/bash
# batch sweep (C1, eager + CUDA graph), C0 oracle timing + GPU parity, compute-sanitizer passes
cd "$(dirname "$0")/.."
E=gpurun_out/misc
mkdir -p $E
timeout 600 python scripts/batch_sweep.py > $E/batch_sweep_laplacian.json 2> $E/batch_sweep_laplacian.err
timeout 600 python scripts/batch_sweep.py --op biharmonic_nested > $E/batch_sweep_nested.json 2> $E/batch_sweep_nested.err
timeout 300 python scripts/c0_oracle_timing.py > $E/c0_oracle_timing.json 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_smoke.py > $E/$tool.log 2>&1
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $E/$tool.log > $E/$tool.summary.txt
done
ls -la $E; cat $E/*.summary.txt
