"""GPU vs fp64 oracle over LARGE samples: the error distribution (quantiles) of the
normalised parity metric for every BASELINE config. Writes gpurun_out/parity_sweep.json.
Diagnostic companion of tests/test_gpu_parity.py (same inputs and metric)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2505_13644_b200 as ctm  # noqa: E402
from synth import mlp_params, points, sigma as make_sigma, widths_for  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
res = {}


def run(name, D, fn_gpu, fn_or):
    params = mlp_params(widths_for(D), 0)
    net = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params])
    mlp = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0)
    X = points(N, D)
    got = fn_gpu(mlp, torch.from_numpy(X).cuda())[0].double().cpu().numpy()
    t = time.time()
    want, _, norm = fn_or(net, X.astype(np.float64))
    e = np.abs(got - want) / norm
    q = {f"q{p}": float(np.quantile(e, p / 100)) for p in (50, 90, 99, 99.9)}
    res[name] = {"N": N, "max": float(e.max()), **q, "frac_over_1e-4": float((e > 1e-4).mean()),
                 "oracle_s": time.time() - t}
    print(name, res[name], flush=True)
    mlp.close()


sig = make_sigma(50, 50, kind="dense")
run("C1 laplacian", 50, lambda m, X: m.laplacian(X), lambda n, X: O.laplacian(n, X))
run("C2 weighted dense", 50, lambda m, X: m.weighted_laplacian(X, torch.from_numpy(sig).cuda()),
    lambda n, X: O.weighted_laplacian(n, X, sig.astype(np.float64)))
for S in (8, 128):
    V = O.rademacher(2, 0, N, S, 50)
    run(f"C3 randomized S={S}", 50, lambda m, X, S=S: m.randomized_laplacian(X, S=S, seed=2),
        lambda n, X, V=V: O.randomized_laplacian(n, X, V))
run("C4 biharmonic", 5, lambda m, X: m.biharmonic(X), lambda n, X: O.biharmonic(n, X))
run("C1 standard Taylor mode", 50, lambda m, X: m.laplacian_standard(X), lambda n, X: O.laplacian(n, X))
Vg = np.random.default_rng(7).standard_normal((N, 16, 5)).astype(np.float32)
run("stochastic biharmonic S=16", 5, lambda m, X: m.stochastic_biharmonic(X, V=torch.from_numpy(Vg).cuda()),
    lambda n, X: O.stochastic_biharmonic(n, X, Vg.astype(np.float64)))
run("C4 biharmonic, nested Laplacians", 5, lambda m, X: m.biharmonic_nested(X), lambda n, X: O.biharmonic(n, X))
sx = None


def _pw_gpu(m, X):
    global sx
    from synth import sigma_field
    sx = sigma_field(X.cpu().numpy(), 50)
    return m.weighted_laplacian_pointwise(X, torch.from_numpy(sx).cuda())


run("C2 weighted, sigma(x)", 50, _pw_gpu, lambda n, X: O.weighted_laplacian_pointwise(n, X, sx.astype(np.float64)))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "parity_sweep.json"), "w"), indent=1)
