#!/bin/bash
# DRAM bytes per launch of the layer kernel (the roofline's `traffic`), per bench workload and
# precision: one ncu pass per workload over a bench run of 1 warm-up + 1 timed step. Parse the
# CSVs with scripts/layer_traffic.py into profiles/layer_traffic.json.
cd "$(dirname "$0")/.."
D=gpurun_out/traffic
mkdir -p $D
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for spec in "laplacian" "weighted" "standard" "biharmonic" "biharmonic_nested" "randomized --S 8" \
            "randomized --S 32" "randomized --S 128" "stochastic_biharmonic --S 16" "laplacian_train"; do
  for prec in fp32 fp16x3 bf16x3; do
    name=$(echo $spec | tr ' ' '_' | tr -d '-')_$prec
    timeout 600 ncu --metrics $M --clock-control none -k regex:jet_layer --csv --log-file $D/$name.csv \
      python bench.py --op $spec --precision $prec --steps 1 --warmup 1 --no-cpu-baseline --no-other-precisions > $D/$name.json 2> $D/$name.err
  done
done
ls $D | wc -l
