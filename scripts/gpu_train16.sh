#!/bin/bash
# fp16x3 training check: the new gradient tests, the fp32-mode gradient suite, the fp16x3
# forward tests, the training bench line in both modes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grad_fp16x3.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/t16.log 2>&1; echo "grad16 rc=$?" >> gpurun_out/t16.log
tail -25 gpurun_out/t16.log
cp gpurun_out/grad_errors.json gpurun_out/grad_errors_fp16x3.json 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_grad.py tests/test_gpu_fp16x3.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/t32.log 2>&1; echo "grad32+fwd16 rc=$?" >> gpurun_out/t32.log
tail -3 gpurun_out/t32.log
for p in fp16x3 fp32; do
  timeout 600 python bench.py --op laplacian_train --precision $p --no-cpu-baseline --steps 20 > gpurun_out/train_$p.json 2> gpurun_out/train_$p.err
  python - gpurun_out/train_$p.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[1], round(d["value"]), round(d["ms_per_step"], 2), d["dtype"][:40], {k: round(v, 2) for k, v in r["kernel_ms_per_step"].items() if v}, d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "failed", e); print(open(sys.argv[1].replace(".json", ".err")).read()[-2000:])
PY
done
