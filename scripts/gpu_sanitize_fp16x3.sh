#!/bin/bash
# compute-sanitizer (memcheck, synccheck, racecheck) over the fp16x3 mode: its test file and the
# sanitizer smoke with every handle in the mode (CTM_PRECISION=fp16x3). Into gpurun_out/sanitizer_f16/.
cd "$(dirname "$0")/.."
S=gpurun_out/sanitizer_f16
mkdir -p $S
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 20 python -m pytest tests/test_gpu_fp16x3.py -q -p no:cacheprovider \
    > $S/fp16x3_tests_$tool.txt 2>&1
  echo "fp16x3 tests $tool rc=$? $(grep -E 'ERROR SUMMARY' $S/fp16x3_tests_$tool.txt | tail -1) $(grep -E 'passed|failed' $S/fp16x3_tests_$tool.txt | tail -1)"
done
for tool in memcheck synccheck; do  # fp16x3 training (the full-size C1 shard test is left out: hours under memcheck)
  timeout 1500 $CS --tool $tool --print-limit 20 python -m pytest tests/test_gpu_grad_fp16x3.py -q -p no:cacheprovider \
    -k "not full_size" > $S/grad16_tests_$tool.txt 2>&1
  echo "fp16x3 grad tests $tool rc=$? $(grep -E 'ERROR SUMMARY' $S/grad16_tests_$tool.txt | tail -1) $(grep -E 'passed|failed' $S/grad16_tests_$tool.txt | tail -1)"
done
for tool in memcheck synccheck racecheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 python scripts/sanitize_smoke.py > $S/smoke_$tool.txt 2>&1
  echo "smoke(fp16x3) $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $S/smoke_$tool.txt | tail -1)"
done
grep "Race reported" $S/smoke_racecheck.txt | sed 's/+0x[0-9a-f]*//g' | sort | uniq -c | head
grep -A2 "Race reported" $S/smoke_racecheck.txt | grep "and " | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head
