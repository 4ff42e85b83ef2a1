#!/bin/bash
# fp16x3 training: its tests, the whole gradient suite with every handle in the fp16x3 mode
# (fixed sets in grad mode run fp16x3), a gradient fuzz soak in the mode, the full GPU suite.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grad_fp16x3.py -q --timeout 300 -p no:cacheprovider > gpurun_out/t16.log 2>&1; echo "grad16 rc=$?" >> gpurun_out/t16.log
tail -3 gpurun_out/t16.log
cp gpurun_out/grad_errors.json gpurun_out/grad_errors_fp16x3_tests.json 2>/dev/null
CTM_PRECISION=fp16x3 CTM_FUZZ_GRAD=60 timeout 1200 python -m pytest tests/test_gpu_grad.py -q --timeout 600 -p no:cacheprovider > gpurun_out/t16suite.log 2>&1; echo "grad suite fp16x3 rc=$?" >> gpurun_out/t16suite.log
tail -3 gpurun_out/t16suite.log
cp gpurun_out/grad_errors.json gpurun_out/grad_errors_fp16x3_suite.json 2>/dev/null
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
