#!/bin/bash
# One evidence pass on a B200 into gpurun_out/$TAG (default r02): smoke, the GPU suite, every
# operator's bench line (both precisions for C1, the torchrun path, the reference arm), the
# 2048-point parity sweep, the fuzz soak, ncu launch lists and ncu --set full summaries of the
# top kernels. Steps can be skipped: SKIP="tests bench sweep soak ncu".
cd "$(dirname "$0")/.."
E=gpurun_out/${TAG:-r02}
mkdir -p $E
skip() { [[ " $SKIP " == *" $1 "* ]]; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $E/gpu_info.txt 2>&1
{ nproc; grep -m1 "model name" /proc/cpuinfo; } > $E/host_cores.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; echo "smoke rc=$?" >> $E/smoke.log
if ! skip tests; then
  timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $E/gpu_tests.log 2>&1
  echo "pytest rc=$?" >> $E/gpu_tests.log
  cp gpurun_out/parity_errors.json gpurun_out/grad_errors.json $E/ 2>/dev/null
fi
if ! skip bench; then
  timeout 600 python bench.py > $E/bench_laplacian.json 2> $E/bench_laplacian.err
  # (the default line is the fp16x3 mode; "precision fp32" lines time the 24-bit mode)
  for spec in "precision fp32" "precision bf16x3" "precision fp32 --op weighted" \
              "precision fp32 --op randomized --S 8" "precision fp32 --op randomized --S 32" \
              "precision fp32 --op randomized --S 128" "precision fp32 --op biharmonic" \
              "precision fp32 --op laplacian_train" "precision fp32 --op biharmonic_nested" \
              "precision fp32 --op stochastic_biharmonic --S 16" "precision fp32 --op standard" \
              "precision fp32 --op biharmonic_standard" "precision fp32 --op randomized_standard --S 8" \
              "precision fp32 --op randomized_standard --S 32" \
              "precision fp32 --op stochastic_biharmonic_standard --S 16" \
              "op weighted" "op standard" "op biharmonic" "op biharmonic_nested" \
              "op randomized --S 8" "op randomized --S 32" "op randomized --S 128" \
              "op stochastic_biharmonic --S 16" "op laplacian_train" "op biharmonic_standard" \
              "op randomized_standard --S 8" "op randomized_standard --S 32" \
              "op stochastic_biharmonic_standard --S 16"; do
    name=$(echo $spec | tr ' ' '_' | tr -d '-')
    timeout 600 python bench.py --no-cpu-baseline --no-other-precisions --$spec > $E/bench_$name.json 2>> $E/bench_other.err
  done
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29555 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > $E/bench_torchrun1.json 2> $E/bench_torchrun1.err
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29556 bench.py --gpus 1 --scaling strong --steps 20 --warmup 3 --no-cpu-baseline \
    > $E/bench_strong1.json 2> $E/bench_strong1.err
  timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $E/bench_reference.json 2>&1
  for f in $E/bench_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    print(sys.argv[1].split("/")[-1], round(d["value"]), d["unit"], "frac", r.get("frac") and round(r["frac"], 3),
          "e2e", d.get("e2e", {}).get("value") and round(d["e2e"]["value"]), d.get("clocks", {}).get("sm_mhz"))
except Exception as e:
    print(sys.argv[1], "unparsed", e)
PY
  done
fi
if ! skip sweep; then
  timeout 900 python scripts/parity_sweep.py 2048 > $E/parity_sweep.log 2>&1
  cp gpurun_out/parity_sweep.json $E/ 2>/dev/null
  CTM_PRECISION=fp16x3 timeout 900 python scripts/parity_sweep.py 2048 > $E/parity_sweep_fp16x3.log 2>&1
  cp gpurun_out/parity_sweep.json $E/parity_sweep_fp16x3.json 2>/dev/null
fi
if ! skip f16suite; then
  CTM_PRECISION=fp16x3 timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider \
    > $E/gpu_tests_fp16x3.log 2>&1; echo "pytest rc=$?" >> $E/gpu_tests_fp16x3.log
fi
if ! skip soak; then
  CTM_FUZZ_SHAPES=150 CTM_FUZZ_DSUM=120 CTM_FUZZ_K4=80 CTM_FUZZ_GRAD=60 timeout 1800 python -m pytest tests -q -m gpu \
    -k fuzz --timeout 600 -p no:cacheprovider > $E/soak.log 2>&1; echo "soak rc=$?" >> $E/soak.log
  cp gpurun_out/parity_errors.json $E/soak_parity_errors.json 2>/dev/null
  cp gpurun_out/grad_errors.json $E/soak_grad_errors.json 2>/dev/null
  CTM_PRECISION=fp16x3 CTM_FUZZ_SHAPES=150 CTM_FUZZ_DSUM=120 CTM_FUZZ_K4=80 CTM_FUZZ_GRAD=60 timeout 1800 \
    python -m pytest tests -q -m gpu -k fuzz --timeout 600 -p no:cacheprovider > $E/soak_fp16x3.log 2>&1
  echo "soak rc=$?" >> $E/soak_fp16x3.log
  cp gpurun_out/parity_errors.json $E/soak_parity_errors_fp16x3.json 2>/dev/null
fi
if ! skip ncu; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_laplacian.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-other-precisions > $E/under_ncu_laplacian.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_randomized_S_8.csv \
    python bench.py --op randomized --S 8 --steps 2 --warmup 1 --no-cpu-baseline > $E/under_ncu_s8.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_laplacian_train.csv \
    python bench.py --op laplacian_train --steps 2 --warmup 1 --no-cpu-baseline > $E/under_ncu_train.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 3 \
    -o $E/prof_layer_c1 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-other-precisions > $E/ncu_layer.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 3 \
    -o $E/prof_layer_c1_fp32 -f python bench.py --precision fp32 --steps 1 --warmup 1 --no-cpu-baseline \
    --no-other-precisions > $E/ncu_layer_fp32.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_laplacian_fp32.csv \
    python bench.py --precision fp32 --steps 2 --warmup 1 --no-cpu-baseline --no-other-precisions > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:wgrad_kernel -s 2 -c 1 \
    -o $E/prof_wgrad -f python bench.py --op laplacian_train --steps 1 --warmup 1 --no-cpu-baseline > $E/ncu_wgrad.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:seed -s 1 -c 1 \
    -o $E/prof_seed_c1 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-other-precisions > $E/ncu_seed.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:jet_layer_kernel<.int.6" -s 3 -c 1 \
    -o $E/prof_bwd -f python bench.py --op laplacian_train --steps 1 --warmup 1 --no-cpu-baseline > $E/ncu_bwd.log 2>&1
  for r in $E/prof_*.ncu-rep; do python scripts/ncu_summary.py $r > ${r%.ncu-rep}.json 2>/dev/null; done
  # the reports themselves stay on the box unless KEEP_REPS=1 (gpurun brings back <= 64 MiB)
  [ -n "$KEEP_REPS" ] || rm -f $E/*.ncu-rep
fi
ls -la $E
