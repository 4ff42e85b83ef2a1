#!/bin/bash
# A/B of bench lines across build variants under abtest/<name> (scripts/make_variant.sh), alternating.
#   VARIANTS="r1 NP2" ARGS="--precision,bf16x3" bash scripts/gpu_ab_r2.sh
mkdir -p gpurun_out
b() { python - "$1" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d["roofline"]
    print(sys.argv[1], round(d["value"]), round(d["ms_per_step"],3), {k: round(v,3) for k,v in r["kernel_ms_per_step"].items() if v}, d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
}
for i in 1 2; do
  for a in ${ARGS:-""}; do
    tag=$(echo "$a" | tr -c 'a-zA-Z0-9' '_')
    python bench.py --no-cpu-baseline --steps 30 ${a//,/ } > gpurun_out/ab_head_${tag}_$i.json 2>/dev/null; b gpurun_out/ab_head_${tag}_$i.json
    for v in $VARIANTS; do
      va=${a//,/ }; [ "$v" = "r1" ] && va=$(echo "$va" | sed 's/--precision bf16x3//')
      (cd abtest/$v && python bench.py --no-cpu-baseline --steps 30 $va > ../../gpurun_out/ab_${v}_${tag}_$i.json 2>/dev/null); b gpurun_out/ab_${v}_${tag}_$i.json
    done
  done
done
