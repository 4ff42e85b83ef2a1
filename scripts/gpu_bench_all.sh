#!/bin/bash
# Every operator's bench line (one B200) into gpurun_out/$1 (default final): the default
# C1 line with the CPU baseline, the others without, the torchrun path and the reference arm.
cd "$(dirname "$0")/.."
E=gpurun_out/${1:-final}
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
