#!/bin/bash
# sanitizers over the fp16x3 paths (incl. training) and the fp16x3 training launch list
mkdir -p gpurun_out
CTM_PRECISION=fp16x3 bash scripts/gpu_sanitize_fp16x3.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_fp16x3.csv \
  python bench.py --op laplacian_train --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu train rc=$?"
