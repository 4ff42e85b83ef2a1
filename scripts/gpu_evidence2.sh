#!/bin/bash
# Evidence pass 2 (round 1, after NEXT-2/3/4): every bench line, the torchrun path, the CPU
# reference arm, the parity sweep, launch lists and ncu --set full captures of the C1
# layer kernel, the nested-biharmonic layer kernel, the adjoint layer kernel and the top
# adjoint kernel.
cd "$(dirname "$0")/.."
E=gpurun_out/ev2
mkdir -p $E
python bench.py > $E/bench_laplacian.json 2> $E/bench_laplacian.err
for spec in "weighted" "standard" "biharmonic" "biharmonic_nested" "randomized --S 8" "randomized --S 32" \
            "randomized --S 128" "stochastic_biharmonic --S 16" "laplacian_train"; do
  name=$(echo $spec | tr ' ' '_' | tr -d '-')
  python bench.py --no-cpu-baseline --op $spec > $E/bench_$name.json 2>> $E/bench_other.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > $E/bench_torchrun1.json 2> $E/bench_torchrun1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $E/bench_reference.json 2>&1
timeout 900 python scripts/parity_sweep.py 2048 > $E/parity_sweep.log 2>&1
cp gpurun_out/parity_sweep.json $E/ 2>/dev/null
for op in laplacian biharmonic_nested laplacian_train; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_$op.csv \
    python bench.py --op $op --steps 2 --warmup 1 --no-cpu-baseline > $E/under_ncu_$op.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 3 \
  -o $E/prof_layer -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $E/ncu_layer.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 3 \
  -o $E/prof_nested -f python bench.py --op biharmonic_nested --steps 1 --warmup 1 --no-cpu-baseline > $E/ncu_nested.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:jet_layer_kernel<6' -s 3 -c 3 \
  -o $E/prof_bwd -f python bench.py --op laplacian_train --steps 1 --warmup 1 --no-cpu-baseline > $E/ncu_bwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:top_bwd -s 1 -c 1 \
  -o $E/prof_topbwd -f python bench.py --op laplacian_train --steps 1 --warmup 1 --no-cpu-baseline > $E/ncu_topbwd.log 2>&1
ls $E
