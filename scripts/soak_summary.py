"""Summarise a fuzz soak's parity records (gpurun_out/parity_errors.json, written by
tests/test_gpu_parity.py check()): operator checks, points, the worst normalised error, and
every check with points above the north_star bar (1e-4) with their condition numbers and
whether plain fp32 also misses there (reading R9). Analysis tool, not product.
    python scripts/soak_summary.py parity_errors.json [label] > soak_summary.json"""
import json
import sys

d = json.load(open(sys.argv[1]))
label = sys.argv[2] if len(sys.argv) > 2 else ""
checks = len(d)
points = sum(int(v.get("n", 0)) for v in d.values())
worst = max((v.get("max_norm_err", 0.0) for v in d.values()), default=0.0)
above = {k: v for k, v in d.items() if v.get("max_norm_err", 0.0) > 1e-4}
print(json.dumps({
    "what": label,
    "operator_checks": checks,
    "points": points,
    "worst_err_over_norm": worst,
    "checks_above_1e-4": len(above),
    "above": {k: {kk: vv for kk, vv in v.items()} for k, v in above.items()},
}, indent=1))
