"""Small runs of every operator for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13644_b200 as ctm  # noqa: E402
from synth import gaussian_directions, mlp_params, points, sigma, sigma_field, signed_weights  # noqa: E402

for widths, prec in (([5, 16, 16, 1], "fp32"), ([50, 64, 64, 1], "fp32"), ([50, 64, 64, 1], "bf16x3"),
                     ([3, 16, 130, 1], "fp32"), ([5, 16, 16, 1], "fp16x3"), ([50, 64, 64, 1], "fp16x3")):
    D = widths[0]
    params = mlp_params(widths, 0)
    mlp = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0)
    mlp.set_precision(prec)
    X = torch.from_numpy(points(9, D)).cuda()
    outs = [mlp.laplacian(X)[0], mlp.laplacian_standard(X)[0],
            mlp.weighted_laplacian(X, torch.from_numpy(sigma(D, D)).cuda())[0],
            mlp.randomized_laplacian(X, S=4, seed=1)[0],
            mlp.randomized_laplacian(X, V=torch.from_numpy(gaussian_directions(9, 3, D)).cuda(), dist="gaussian")[0]]
    if D <= 7:
        outs += [mlp.biharmonic(X)[0], mlp.stochastic_biharmonic(X, S=3, seed=2)[0]]
    outs += [mlp.biharmonic_nested(X)[0] if D <= 20 else X[:, 0],
             mlp.weighted_laplacian_pointwise(X, torch.from_numpy(sigma_field(X.cpu().numpy(), 3)).cuda())[0]]
    w = torch.from_numpy(signed_weights(3)).cuda()
    for K in (2, 4):
        outs.append(mlp.directional_sum(X, K, torch.from_numpy(gaussian_directions(1, 3, D)[0]).cuda(), w)[0])
        outs.append(mlp.directional_sum(X, K, torch.from_numpy(gaussian_directions(9, 3, D)).cuda(), w)[0])
    # direction blocks (forced small blocks: many sub-points, padded last block)
    mlp.set_direction_block(2)
    outs += [mlp.laplacian(X)[0], mlp.laplacian_standard(X)[0], mlp.randomized_laplacian(X, S=7, seed=1)[0],
             mlp.weighted_laplacian(X, torch.from_numpy(sigma(D, D)).cuda())[0]]
    if D <= 7:
        outs += [mlp.biharmonic(X)[0], mlp.stochastic_biharmonic(X, S=5, seed=2)[0]]
    for K in (2, 4):
        outs.append(mlp.directional_sum(X, K, torch.from_numpy(gaussian_directions(9, 5, D)).cuda(),
                                        torch.from_numpy(signed_weights(5)).cuda())[0])
    mlp.set_direction_block(0)
    # differentiable path: forward in grad mode, backward, weight update
    mlp.grad_enable()
    for call in (lambda: mlp.laplacian(X), lambda: mlp.randomized_laplacian(X, S=4, seed=1),
                 lambda: mlp.weighted_laplacian(X, torch.from_numpy(sigma(D, D)).cuda()),
                 lambda: mlp.directional_sum(X, 2, torch.from_numpy(gaussian_directions(1, 3, D)[0]).cuda(), w)):
        call()
        g = mlp.backward(torch.ones(9, device="cuda"), torch.ones(9, device="cuda"))
        outs.append(g[0][0].reshape(-1))
    mlp.set_weights([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params])
    outs.append(mlp.laplacian(X)[0])
    torch.cuda.synchronize()
    print(widths, prec, [float(o.abs().max()) for o in outs])
    mlp.close()
