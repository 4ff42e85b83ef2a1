#!/bin/bash
# sweep bench configurations (1 GPU): SWEEP="args1 args2 ..." with commas for spaces
mkdir -p gpurun_out
for args in $SWEEP; do
  timeout 300 python bench.py --no-cpu-baseline --steps ${STEPS:-20} ${args//,/ } > gpurun_out/sweep_q.json 2> gpurun_out/sweep_q.err || { echo "$args FAILED"; tail -3 gpurun_out/sweep_q.err; continue; }
  python - "$args" <<'PY'
import json, sys
d = json.load(open("gpurun_out/sweep_q.json")); r = d["roofline"]
print(sys.argv[1] or "C1", round(d["value"]), "pts/s", round(d["ms_per_step"], 3), "ms", "layer", round(r["achieved"], 1), "TF",
      round(r["frac"], 3), {k: round(v, 3) for k, v in r["kernel_ms_per_step"].items() if v}, d["clocks"]["sm_mhz"], "MHz", {k: d["config"].get(k) for k in ("slots_per_point", "points_per_tile", "mma_n")})
PY
done
