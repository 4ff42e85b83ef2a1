#!/bin/bash
# ncu --set full of one layer launch per NCU_CASES entry "name|bench args|skip"
E=gpurun_out/ncu
mkdir -p $E
IFS=';' read -ra CASES <<< "$NCU_CASES"
for c in "${CASES[@]}"; do
  IFS='|' read -r name args skip <<< "$c"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s $skip -c 1 \
    -o $E/$name -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline $args > $E/$name.log 2>&1
  ncu -i $E/$name.ncu-rep --page details --csv > $E/$name.details.csv 2>/dev/null
  ncu -i $E/$name.ncu-rep --page raw --csv > $E/$name.raw.csv 2>/dev/null
done
ls -la $E
