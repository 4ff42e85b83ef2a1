"""Experiment harness (CTM_EXP_STATS build): per-role cycle counters of the layer kernel.
usage: python scripts/exp_stats.py <op> [S] [precision]   (run from a tree built with -DCTM_EXP_STATS)"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2505_13644_b200 as ctm  # noqa: E402
from synth import mlp_params, points, widths_for  # noqa: E402

op = sys.argv[1]
S = int(sys.argv[2]) if len(sys.argv) > 2 else 8
D = 5 if "biharmonic" in op else 50
params = mlp_params(widths_for(D), 0)
mlp = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0)
if len(sys.argv) > 3 and hasattr(mlp, "set_precision"):
    mlp.set_precision(sys.argv[3])
X = torch.from_numpy(points(16384, D)).cuda()
fn = getattr(mlp, op)
kw = {"S": S, "seed": 2} if op in ("randomized_laplacian", "stochastic_biharmonic") else {}
lib = ctm.lib()
lib.ctm_debug_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((256, 8), dtype=np.uint64)
for _ in range(3):
    fn(X, **kw)
torch.cuda.synchronize()
lib.ctm_debug_stats(buf.ctypes.data, 1)
fn(X, **kw)
torch.cuda.synchronize()
lib.ctm_debug_stats(buf.ctypes.data, 1)
b = buf[:148].astype(np.float64)
lead = b[0::2]  # leaders (MMA issuer)
life = lead[:, 3].mean()
print(f"{op} S={S} plan={mlp.last_plan()}")
print(f"  MMA issuer lifetime {life:.0f} cyc, tiles/pair {lead[:, 7].mean():.1f}")
print(f"  MMA wait tmem_empty {lead[:, 1].mean() / life:.3f}  wait TMA full {lead[:, 2].mean() / life:.3f}")
print(f"  producer wait empty (all CTAs) {b[:, 0].mean() / life:.3f}")
print(f"  epilogue warp2: wait tmem_full {b[:, 4].mean() / life:.3f}  work {b[:, 5].mean() / life:.3f}")
print(f"  epilogue other warps mean work {b[:, 6].mean() / life / 7:.3f} (of 7 or 15 warps, assuming 7)")
