#!/bin/bash
# GPU suite in the default mode, then in the fp16x3 mode, then the fuzz soak in the fp16x3 mode
mkdir -p gpurun_out/s3check
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/s3check/gpu_tests.log 2>&1; echo "default rc=$?"; tail -2 gpurun_out/s3check/gpu_tests.log
CTM_PRECISION=fp16x3 timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/s3check/gpu_tests_fp16x3.log 2>&1; echo "fp16x3 rc=$?"; tail -2 gpurun_out/s3check/gpu_tests_fp16x3.log
CTM_PRECISION=fp16x3 CTM_FUZZ_SHAPES=150 CTM_FUZZ_DSUM=120 CTM_FUZZ_K4=80 CTM_FUZZ_GRAD=60 timeout 1800 python -m pytest tests -q -m gpu -k fuzz --timeout 600 -p no:cacheprovider > gpurun_out/s3check/soak_fp16x3.log 2>&1; echo "soak fp16x3 rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/s3check/soak_fp16x3.log | tail -5
cp gpurun_out/parity_errors.json gpurun_out/s3check/soak_parity_errors_fp16x3.json
