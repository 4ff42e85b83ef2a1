#!/bin/bash
# The GPU suite with every new handle in the fp16x3 mode (CTM_PRECISION=fp16x3), the suite in
# the default mode, the fuzz soak in fp16x3 (incl. the 60-case gradient fuzz: fp16x3 training),
# and bench lines of the mode; logs and error records into gpurun_out/f16s/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/f16s
CTM_PRECISION=fp16x3 timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/f16s/gpu_tests_fp16x3.log 2>&1; echo "fp16x3 suite rc=$?"; tail -3 gpurun_out/f16s/gpu_tests_fp16x3.log
cp gpurun_out/parity_errors.json gpurun_out/f16s/parity_errors_fp16x3.json 2>/dev/null
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/f16s/gpu_tests_default.log 2>&1; echo "default suite rc=$?"; tail -3 gpurun_out/f16s/gpu_tests_default.log
if [ -z "$NOSOAK" ]; then
CTM_PRECISION=fp16x3 CTM_FUZZ_SHAPES=150 CTM_FUZZ_DSUM=120 CTM_FUZZ_K4=80 CTM_FUZZ_GRAD=60 timeout 1800 python -m pytest tests -q -m gpu -k fuzz --timeout 600 -p no:cacheprovider > gpurun_out/f16s/soak_fp16x3.log 2>&1; echo "soak rc=$?"; tail -3 gpurun_out/f16s/soak_fp16x3.log
cp gpurun_out/parity_errors.json gpurun_out/f16s/soak_parity_errors_fp16x3.json 2>/dev/null
fi
cp gpurun_out/grad_errors.json gpurun_out/f16s/soak_grad_errors_fp16x3.json 2>/dev/null
for a in "--precision fp16x3" "--precision fp16x3 --op randomized --S 8" "--precision fp16x3 --op laplacian_train" \
         "--precision fp16x3 --op stochastic_biharmonic --S 16"; do
  python bench.py --no-cpu-baseline --steps 30 $a > gpurun_out/f16s/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/f16s/b.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$a', round(d['value']), round(d['ms_per_step'],3), d['config']['precision_ran'], round(r['frac'],3), d['clocks']['sm_mhz'])"
done
