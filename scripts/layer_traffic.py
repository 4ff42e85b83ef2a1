"""Parse the ncu CSVs of scripts/layer_traffic.sh into profiles/layer_traffic.json: for each
bench workload and precision, the DRAM bytes (read + write) per launch of the layer kernel in
the timed step, averaged over the step's layer launches, next to the algorithmic bytes of
the same launches (bf16 planes of the input block read once, of the output block written
once). bench.py reads `dram_bytes_per_launch` as roofline.traffic."""
import csv
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "traffic")
out = {}
for f in sorted(glob.glob(os.path.join(src, "*.csv"))):
    name = os.path.basename(f)[:-4]  # e.g. randomized_S_8_fp32
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows:
        continue
    h = rows[0]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[1:]:
        per.setdefault(int(r[iid]), {"kernel": r[ik]})[r[im]] = float(r[iv].replace(",", ""))
    launches = [per[i] for i in sorted(per)]
    key = name.replace("randomized_S_", "randomized_S").replace("stochastic_biharmonic_S_16", "stochastic_biharmonic")
    rec = {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none over "
                     f"`bench.py --op ... --steps 1 --warmup 1` ({os.path.basename(f)}); every jet_layer_kernel "
                     f"launch of the run (all steps launch the same shapes)"}
    for tag, sel in (("", lambda k: "jet_layer_kernel<6" not in k), ("bwd_", lambda k: "jet_layer_kernel<6" in k)):
        ls = [d for d in launches if sel(d["kernel"].replace("(int)", "").replace(" ", ""))]
        if not ls:
            continue
        b = [d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in ls]
        rec[f"{tag}dram_bytes_per_launch"] = sum(b) / len(b)
        rec[f"{tag}launches"] = len(b)
        rec[f"{tag}dram_read_per_launch"] = sum(d["dram__bytes_read.sum"] for d in ls) / len(b)
        rec[f"{tag}dram_write_per_launch"] = sum(d["dram__bytes_write.sum"] for d in ls) / len(b)
    out[key] = rec
dst = os.path.join(ROOT, "profiles", "layer_traffic.json")
json.dump(out, open(dst, "w"), indent=1, sort_keys=True)
print(f"{len(out)} workloads -> {dst}")
