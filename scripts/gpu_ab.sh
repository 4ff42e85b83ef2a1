#!/bin/bash
# A/B: bench lines of the tree in _ab/old vs this tree, alternating (AB_ARGS as SWEEP in gpu_sweep.sh)
mkdir -p gpurun_out
for rep in 1 2; do
for tree in ${TREES:-_ab/old .}; do
  for args in $AB_ARGS; do
    (cd $tree && timeout 300 python bench.py --no-cpu-baseline --steps ${STEPS:-20} ${args//,/ } > /tmp/ab.json 2>/dev/null)
    python - "$tree $args" <<'PY'
import json, sys
d = json.load(open("/tmp/ab.json")); r = d["roofline"]
print(sys.argv[1], round(d["value"]), "pts/s", round(d["ms_per_step"], 3), "ms frac", round(r["frac"], 3),
      {k: round(v, 3) for k, v in r["kernel_ms_per_step"].items() if v}, d["clocks"]["sm_mhz"], "MHz")
PY
  done
done
done
