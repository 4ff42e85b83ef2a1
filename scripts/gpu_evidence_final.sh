#!/bin/bash
# Final-build evidence (round 1, session 3): C1 launch list and ncu --set full summaries of
# the layer and seed kernels, plus the randomized S=8 launch list.
cd "$(dirname "$0")/.."
E=gpurun_out/final
mkdir -p $E
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_laplacian.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $E/under_ncu_laplacian.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_randomized_S_8.csv \
  python bench.py --op randomized --S 8 --steps 2 --warmup 1 --no-cpu-baseline > $E/under_ncu_s8.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 3 \
  -o $E/prof_layer_c1 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $E/ncu_c1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seed_layer -s 1 -c 1 \
  -o $E/prof_seed_c1 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $E/ncu_seed.log 2>&1
for r in $E/prof_*.ncu-rep; do python scripts/ncu_summary.py $r > ${r%.ncu-rep}.json 2>/dev/null; done
ls -la $E
