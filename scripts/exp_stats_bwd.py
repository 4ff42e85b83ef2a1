"""Experiment harness (CTM_EXP_STATS build): cycle counters of the adjoint layer kernel
(jet_layer_kernel<kBwd2>) during ctm_backward at C1, N = 16384."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2505_13644_b200 as ctm  # noqa: E402
from synth import mlp_params, points, widths_for  # noqa: E402

params = mlp_params(widths_for(50), 0)
mlp = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0)
mlp.grad_enable()
X = torch.from_numpy(points(16384, 50)).cuda()
gop = torch.ones(16384, device="cuda") / 16384
lib = ctm.lib()
lib.ctm_debug_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((256, 8), dtype=np.uint64)
for _ in range(2):
    mlp.laplacian(X)
    mlp.backward(gop)
torch.cuda.synchronize()
mlp.laplacian(X)
torch.cuda.synchronize()
lib.ctm_debug_stats(buf.ctypes.data, 1)
mlp.backward(gop)
torch.cuda.synchronize()
lib.ctm_debug_stats(buf.ctypes.data, 1)
b = buf[:148].astype(np.float64)
lead = b[0::2]
life = lead[:, 3].mean()
print(f"adjoint layers: MMA issuer lifetime {life:.0f} cyc, tiles/pair {lead[:, 7].mean():.1f}")
print(f"  MMA wait tmem_empty {lead[:, 1].mean() / life:.3f}  wait TMA full {lead[:, 2].mean() / life:.3f}")
print(f"  producer wait empty {b[:, 0].mean() / life:.3f}")
print(f"  epilogue warp2: wait tmem_full {b[:, 4].mean() / life:.3f}  work {b[:, 5].mean() / life:.3f}")
