#!/bin/bash
# Session-3 evidence pass (fp16x3 headline, fp16x3 training): every bench line, sweeps, suites,
# soaks, ncu summaries (gpu_evidence.sh), then the roofline traffic per workload and precision.
cd "$(dirname "$0")/.."
# (two gpurun calls: PART=1 the evidence pass, PART=2 the ratio tables in both modes and the traffic)
if [ "${PART:-1}" = 1 ]; then
  TAG=${TAG:-r02s3} bash scripts/gpu_evidence.sh
else
  mkdir -p gpurun_out/${TAG:-r02s3}
  for p in fp16x3 fp32; do
    timeout 1500 python scripts/ratio_table.py --precision $p > gpurun_out/${TAG:-r02s3}/ratio_table_$p.json 2> gpurun_out/${TAG:-r02s3}/ratio_table_$p.log
  done
  bash scripts/layer_traffic.sh
fi
