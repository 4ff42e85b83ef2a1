#!/bin/bash
# Session-3 check: smoke, GPU suite, bench lines (default, fp16x3), ncu --set full of the fp16x3
# and fp32-mode C1 layer kernels.
mkdir -p gpurun_out
EXTRA="--precision,fp16x3" bash scripts/gpu_r2.sh
for p in fp16x3 fp32; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:jet_layer -c 3 \
    -o gpurun_out/full_$p python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-other-precisions --precision $p > gpurun_out/ncu_$p.log 2>&1
  echo "ncu $p rc=$?"
done
