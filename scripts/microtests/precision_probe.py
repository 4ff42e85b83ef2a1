"""Parity of one precision mode on C1 / S=8 / C4-nested samples against the fp64 oracle
(normalised metric, max and quantiles). usage: python scripts/microtests/precision_probe.py MODE [npts]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.getcwd())  # a variant tree (abtest/<name>) run from its own directory wins
import oracle as O  # noqa: E402
import paper_2505_13644_b200 as ctm  # noqa: E402
from synth import mlp_params, points, widths_for  # noqa: E402

mode = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
res = {}
for name, D in (("C1", 50), ("S8", 50)):
    params = mlp_params(widths_for(D), 0)
    net = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params])
    mlp = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0)
    mlp.set_precision(mode)
    X = points(n, D)
    if name == "C1":
        got = mlp.laplacian(torch.from_numpy(X).cuda())[0].double().cpu().numpy()
        want, _, norm = O.laplacian(net, X.astype(np.float64))
    else:
        got = mlp.randomized_laplacian(torch.from_numpy(X).cuda(), S=8, seed=2)[0].double().cpu().numpy()
        want, _, norm = O.randomized_laplacian(net, X.astype(np.float64), O.rademacher(2, 0, n, 8, D))
    e = np.abs(got - want) / norm
    res[name] = {"max": float(e.max()), "q99": float(np.quantile(e, 0.99)), "median": float(np.median(e))}
    res[name]["ran"] = mlp.last_precision()
    mlp.close()
print(json.dumps({mode: res}))
