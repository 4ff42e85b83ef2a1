#!/bin/bash
# Round-2 GPU iteration: smoke, the GPU suite, and bench lines for the given configs.
#   EXTRA="--precision,bf16x3 --op,randomized,--S,8" bash scripts/gpu_r2.sh
# (each EXTRA word is one bench line; commas become spaces)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
if [ -z "$NOTESTS" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -q -m gpu -x --timeout 300 -p no:cacheprovider $PYTEST_ARGS > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
  tail -5 gpurun_out/gpu_tests.log
fi
i=0
for args in "" $EXTRA; do
  i=$((i+1))
  timeout 600 python bench.py --no-cpu-baseline ${args//,/ } > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err
  python - "$args" $i <<'PY'
import json, sys
try:
    d = json.load(open(f"gpurun_out/bench_{sys.argv[2]}.json")); r = d["roofline"]
    print(sys.argv[1] or "C1", round(d["value"]), "pts/s", round(d["ms_per_step"], 3), "ms", "layer", round(r["achieved"], 1), "TF",
          round(r["frac"], 3), "burst", round(r.get("frac_vs_burst") or 0, 3), {k: round(v, 3) for k, v in r["kernel_ms_per_step"].items()}, d["clocks"]["sm_mhz"], "MHz")
except Exception as e:
    print(sys.argv[1], "FAILED", e); print(open(f"gpurun_out/bench_{sys.argv[2]}.err").read()[-1500:])
PY
done
