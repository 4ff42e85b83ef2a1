#!/bin/bash
# One gpurun session: tests, smoke, bench, ncu launch list + full capture of the top kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.txt
nproc > gpurun_out/host_cores.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host_cores.txt
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 3 \
  -o gpurun_out/prof_layer -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_layer.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seed_layer -s 1 -c 1 \
  -o gpurun_out/prof_seed -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_seed.log 2>&1
fi
ls -la gpurun_out
