#!/bin/bash
# quick GPU iteration: parity tests, smoke, C1 bench line (+ optional extra bench args)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for args in "" $EXTRA; do
  timeout 600 python bench.py --no-cpu-baseline ${args//,/ } > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
  python - "$args" <<'PY'
import json, sys
d = json.load(open("gpurun_out/bench_q.json")); r = d["roofline"]
print(sys.argv[1] or "C1", round(d["value"]), "pts/s", round(d["ms_per_step"], 3), "ms", "layer", round(r["achieved"], 1), "TF",
      round(r["frac"], 3), {k: round(v, 3) for k, v in r["kernel_ms_per_step"].items()}, d["clocks"]["sm_mhz"], "MHz")
PY
done
python -c "
import json; d=json.load(open('gpurun_out/parity_errors.json')); print('max parity err', max(v['max_norm_err'] for v in d.values()))"
