M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
for v in head NOST 1PL; do
  d=.; [ "$v" = head ] || d=abtest/$v
  (cd $d && timeout 300 ncu --metrics $M --clock-control none -k regex:jet_layer --csv --log-file $GRAFT_REPO_ROOT/gpurun_out/s8_$v.csv python bench.py --op randomized --S 8 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1)
  (cd $d && timeout 300 ncu --metrics $M --clock-control none -k regex:jet_layer --csv --log-file $GRAFT_REPO_ROOT/gpurun_out/c1_$v.csv python bench.py --op laplacian --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1)
done
for f in gpurun_out/s8_*.csv gpurun_out/c1_*.csv; do python3 - $f <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; per={}
for r in rows[1:]:
    per.setdefault(int(r[h.index("ID")]),{})[r[h.index("Metric Name")]]=float(r[h.index("Metric Value")].replace(",",""))
L=list(per.values())[-8:]
print(sys.argv[1], [(round(d["gpu__time_duration.sum"]/1e3,1), round(d["smsp__inst_executed.sum"]/1e6,1), round(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"],1)) for d in L])
PY
done
