"""Diagnose test_fuzz_directional_sums_blocks_activations[94] (the soak point fp16x3 misses):
per check, the normalised error of the fp16x3 and fp32 modes and of plain fp32 (vanilla32)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_2505_13644_b200 as ctm
from tests._util import magnitude_k2, magnitude_k4, ref32
from tests.test_gpu_parity import nets
from synth import gaussian_directions, points, sigma_field, signed_weights

case = int(sys.argv[1]) if len(sys.argv) > 1 else 94
rng = np.random.default_rng(3000 + case)
D = int(rng.integers(1, 24))
hidden = [int(rng.integers(65, 300)) for _ in range(int(rng.integers(1, 4)))]
widths = [D] + hidden + [1]
act = ["tanh", "sin"][case % 2]
N = int(rng.integers(1, 50))
params, _ = nets(widths, seed=100 + case)
onet = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params], act)
X = points(N, D, seed=case)
Xc = torch.from_numpy(X).cuda(); Xd = X.astype(np.float64)
ms = {p: ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0, act=act, precision=p)
      for p in ("fp16x3", "fp32")}
rb = int(rng.integers(0, 40))
for m in ms.values(): m.set_direction_block(rb)
print("widths", widths, "act", act, "N", N, "rb", rb)
for K in (2, 4):
    J = int(rng.integers(1, 120 if K == 2 else 50))
    w = signed_weights(J, seed=case)
    per_point = bool(rng.integers(0, 2))
    dirs = gaussian_directions(N, J, D, seed=case) if per_point else gaussian_directions(1, J, D, seed=case)[0]
    if K == 4 and per_point and J * D > 12288:
        continue
    want, _, norm = O.directional_sum(onet, Xd, K, dirs.astype(np.float64), w.astype(np.float64))
    r32 = ref32(params, X, dirs, w, K, act)(np.arange(N))
    e32 = np.abs(np.asarray(r32, np.float64) - want) / norm
    for p, m in ms.items():
        got = m.directional_sum(Xc, K, torch.from_numpy(dirs).cuda(), torch.from_numpy(w).cuda())[0]
        e = np.abs(got.double().cpu().numpy() - want) / norm
        i = int(e.argmax())
        print(f"K={K} J={J} per_point={per_point} {p}({m.last_precision()}) max {e.max():.3e} at {i}; vanilla32 there {e32[i]:.3e}; plan {m.last_plan()}")
R = int(rng.integers(1, 80))
sx = sigma_field(X, R, seed=case)
want, _, norm = O.weighted_laplacian_pointwise(onet, Xd, sx.astype(np.float64))
for p, m in ms.items():
    got = m.weighted_laplacian_pointwise(Xc, torch.from_numpy(sx).cuda())[0]
    e = np.abs(got.double().cpu().numpy() - want) / norm
    print(f"sigma(x) R={R} {p}({m.last_precision()}) max {e.max():.3e} at {int(e.argmax())}")
