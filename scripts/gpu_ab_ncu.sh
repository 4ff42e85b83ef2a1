#!/bin/bash
# A/B of build variants (scripts/make_variant.sh): bench lines alternating (gpu_ab_r2.sh), then
# per variant one ncu pass over the layer kernels with time, DRAM bytes and tensor-pipe activity.
#   VARIANTS="SPREAD CS" ARGS="" bash scripts/gpu_ab_ncu.sh
mkdir -p gpurun_out
bash scripts/gpu_ab_r2.sh
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second
for v in head $VARIANTS; do
  d=.; [ "$v" = head ] || d=abtest/$v
  (cd $d && timeout 600 ncu --metrics $M --clock-control none -k regex:${KREGEX:-jet_layer|seed} --csv \
     --log-file $GRAFT_REPO_ROOT/gpurun_out/abncu_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${NCU_ARGS:-} > /dev/null 2>&1)
  python - gpurun_out/abncu_$v.csv <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; rows = rows[1:]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
iid = h.index("ID")
per = collections.OrderedDict()
for r in rows:
    per.setdefault(r[iid], {"k": r[ik][:40]})[r[im]] = float(r[iv].replace(",", ""))
for i, d in per.items():
    print(sys.argv[1].split("_")[-1], d["k"], {k.split("__")[1][:28]: round(v, 3) for k, v in d.items() if k != "k"})
PY
done
