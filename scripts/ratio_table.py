"""The paper's collapsed/standard time ratios (Table `tab:benchmark-ratios`)
on one B200: each (collapsed, standard) bench pair is run back to back, alternating, REPS
times; the ratio of the medians of ms/step is reported with the clocks. One JSON object.
usage: python scripts/ratio_table.py [--reps 3] [--steps 20] [--precision fp16x3|fp32]
(both members of a pair run in the same arithmetic; every operator of the table has both
modes)"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAIRS = [
    ("exact Laplacian (C1)", ["--op", "laplacian"], ["--op", "standard"], "52/101", "0.55 (0.51)"),
    ("randomized Laplacian S=8", ["--op", "randomized", "--S", "8"], ["--op", "randomized_standard", "--S", "8"],
     "10/17", "0.54 per sample (0.50)"),
    ("randomized Laplacian S=32", ["--op", "randomized", "--S", "32"], ["--op", "randomized_standard", "--S", "32"],
     "34/65", "0.54 per sample (0.50)"),
    ("exact biharmonic (C4)", ["--op", "biharmonic"], ["--op", "biharmonic_standard"], "107/141", "0.88 (0.77)"),
    ("stochastic biharmonic S=16", ["--op", "stochastic_biharmonic", "--S", "16"],
     ["--op", "stochastic_biharmonic_standard", "--S", "16"], "50/65", "0.76 (0.75)"),
]


def bench(args, steps, precision):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline", "--no-other-precisions",
                          "--steps", str(steps), "--precision", precision, *args], capture_output=True, text=True,
                         cwd=ROOT)
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert d["config"]["precision_ran"] == precision, (args, d["config"]["precision_ran"])
    return d["ms_per_step"], d["clocks"]["sm_mhz"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--precision", default="fp16x3", choices=["fp16x3", "fp32", "bf16x3"])
    a = ap.parse_args()
    rows = []
    for name, col, std, vec, paper in PAIRS:
        c, s, cm, sm = [], [], [], []
        for _ in range(a.reps):
            t, m = bench(col, a.steps, a.precision)
            c.append(t), cm.append(m)
            t, m = bench(std, a.steps, a.precision)
            s.append(t), sm.append(m)
        num, den = (int(x) for x in vec.split("/"))
        rows.append({"operator": name, "collapsed_ms": c, "standard_ms": s, "collapsed_mhz": cm, "standard_mhz": sm,
                     "ratio_of_medians": statistics.median(c) / statistics.median(s), "vectors": vec,
                     "vector_ratio": num / den, "paper_measured_theory": paper})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    print(json.dumps({"reps": a.reps, "steps": a.steps, "N": 16384, "precision": a.precision, "rows": rows}))


if __name__ == "__main__":
    main()
