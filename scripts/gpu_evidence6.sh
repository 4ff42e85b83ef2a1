#!/bin/bash
# Evidence pass 6 (round 1, session 2 final: + 128-byte operand rows / SWIZZLE_128B): every bench line, the torchrun path, the
# CPU reference arm, launch lists, ncu --set full of the layer kernel for C1, C3 S=128 (now
# in direction blocks) and standard mode, and the parity sweep.
cd "$(dirname "$0")/.."
E=gpurun_out/ev6
mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $E/gpu_info.txt
python bench.py > $E/bench_laplacian.json 2> $E/bench_laplacian.err
for spec in "weighted" "standard" "biharmonic" "biharmonic_nested" "randomized --S 8" "randomized --S 32" \
            "randomized --S 128" "stochastic_biharmonic --S 16" "laplacian_train" "biharmonic_standard" \
            "randomized_standard --S 8" "randomized_standard --S 32" "stochastic_biharmonic_standard --S 16"; do
  name=$(echo $spec | tr ' ' '_' | tr -d '-')
  python bench.py --no-cpu-baseline --op $spec > $E/bench_$name.json 2>> $E/bench_other.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > $E/bench_torchrun1.json 2> $E/bench_torchrun1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $E/bench_reference.json 2>&1
timeout 900 python scripts/parity_sweep.py 2048 > $E/parity_sweep.log 2>&1
cp gpurun_out/parity_sweep.json $E/ 2>/dev/null
for spec in "laplacian" "randomized --S 128" "randomized --S 8" "biharmonic"; do
  name=$(echo $spec | tr ' ' '_' | tr -d '-')
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_$name.csv \
    python bench.py --op $spec --steps 2 --warmup 1 --no-cpu-baseline > $E/under_ncu_$name.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 3 \
  -o $E/prof_layer_c1 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $E/ncu_c1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 4 -c 4 \
  -o $E/prof_layer_s128 -f python bench.py --op randomized --S 128 --steps 1 --warmup 1 --no-cpu-baseline > $E/ncu_s128.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 3 \
  -o $E/prof_layer_bih -f python bench.py --op biharmonic --steps 1 --warmup 1 --no-cpu-baseline > $E/ncu_bih.log 2>&1
for r in $E/prof_*.ncu-rep; do python scripts/ncu_summary.py $r > ${r%.ncu-rep}.json 2>/dev/null; done
ls -la $E
timeout 900 python scripts/ratio_table.py > $E/ratio_table.json 2> $E/ratio_table.err; bash scripts/gpu_misc.sh
