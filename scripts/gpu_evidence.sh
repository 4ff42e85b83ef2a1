#!/bin/bash
# Evidence pass: bench every operator, torchrun path, parity sweep, ncu (launch list + full captures).
mkdir -p gpurun_out/ev
cd "$(dirname "$0")/.."
python bench.py > gpurun_out/ev/bench_laplacian.json 2> gpurun_out/ev/bench_laplacian.err
for spec in "weighted" "standard" "biharmonic" "randomized --S 8" "randomized --S 32" "randomized --S 128" "stochastic_biharmonic --S 16"; do
  name=$(echo $spec | tr ' ' '_' | tr -d '-')
  python bench.py --no-cpu-baseline --op $spec > gpurun_out/ev/bench_$name.json 2>> gpurun_out/ev/bench_other.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ev/bench_torchrun1.json 2> gpurun_out/ev/bench_torchrun1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_reference.json 2>&1
timeout 900 python scripts/parity_sweep.py 2048 > gpurun_out/ev/parity_sweep.log 2>&1
cp gpurun_out/parity_sweep.json gpurun_out/ev/ 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ev/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 3 \
  -o gpurun_out/ev/prof_layer -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ev/ncu_layer.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seed_layer -s 1 -c 1 \
  -o gpurun_out/ev/prof_seed -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ev/ncu_seed.log 2>&1
ls gpurun_out/ev
