#!/bin/bash
# Session-3 evidence pass (fp16x3 headline, fp16x3 training): every bench line, sweeps, suites,
# soaks, ncu summaries (gpu_evidence.sh), then the roofline traffic per workload and precision.
cd "$(dirname "$0")/.."
TAG=r02s3 bash scripts/gpu_evidence.sh
bash scripts/layer_traffic.sh
