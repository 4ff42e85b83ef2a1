#!/bin/bash
# bench every §8 operator (1 GPU) + ncu evidence for the default (C1) line
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_laplacian.json 2> gpurun_out/bench_laplacian.err
for op in weighted biharmonic; do python bench.py --op $op --no-cpu-baseline > gpurun_out/bench_$op.json 2>/dev/null; done
for S in 8 32 128; do python bench.py --op randomized --S $S --no-cpu-baseline > gpurun_out/bench_randomized_S$S.json 2>/dev/null; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 3 \
  -o gpurun_out/prof_layer -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_layer.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seed_layer -s 1 -c 1 \
  -o gpurun_out/prof_seed -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_seed.log 2>&1
