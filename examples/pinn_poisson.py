"""PINN for a Poisson problem, trained through the collapsed Laplacian (the paper's use
case): find u_theta on [-1, 1]^D with

    -Laplacian u = g  in the cube,   u = u*  on its boundary,

for the manufactured solution u*(x) = sum_d sin(pi x_d / 2), g = (pi^2 / 4) u*.
Every step evaluates Laplacian u and u at interior collocation points with ONE call
(ctm_laplacian in grad mode), u at boundary points with a second call, and gets the
parameter gradients of

    loss = mean_int (Laplacian u + g)^2 + mean_bnd (u - u*)^2

from ctm_backward (the second backward accumulates). Adam runs on torch copies of the
parameters, which go back with ctm_set_weights. Usage:
    python examples/pinn_poisson.py [--D 5] [--steps 300] [--N 4096]
"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13644_b200 as ctm  # noqa: E402


def u_star(x):
    return torch.sin(0.5 * math.pi * x).sum(1)


def train(D=5, steps=300, N=4096, Nb=1024, width=128, lr=3e-3, seed=0, log_every=50, device=0):
    g = torch.Generator().manual_seed(seed)
    widths = [D, width, width, 1]
    params = []
    for fi, fo in zip(widths[:-1], widths[1:]):
        bound = 1.0 / math.sqrt(fi)
        params.append([((torch.rand(fo, fi, generator=g) * 2 - 1) * bound).cuda(device).requires_grad_(),
                       ((torch.rand(fo, generator=g) * 2 - 1) * bound).cuda(device).requires_grad_()])
    flat = [p for layer in params for p in layer]
    opt = torch.optim.Adam(flat, lr=lr)
    mlp = ctm.MLP([(W.detach(), b.detach()) for W, b in params], device=device)
    mlp.grad_enable()
    history = []
    for step in range(steps):
        xi = (torch.rand(N, D, device=f"cuda:{device}") * 2 - 1).contiguous()
        xb = (torch.rand(Nb, D, device=f"cuda:{device}") * 2 - 1)
        face = torch.randint(0, D, (Nb,), device=xb.device)
        xb[torch.arange(Nb, device=xb.device), face] = torch.sign(torch.rand(Nb, device=xb.device) - 0.5)
        xb = xb.contiguous()
        lap, _ = mlp.laplacian(xi)                                  # forward, records the tape
        res = lap + (math.pi ** 2 / 4) * u_star(xi)                 # Laplacian u + g
        grads = mlp.backward(2.0 * res / N)                         # d/dtheta mean(res^2)
        _, ub = mlp.laplacian(xb)                                   # u on the boundary
        bres = ub - u_star(xb)
        mlp.backward(torch.zeros(Nb, device=xb.device), 2.0 * bres / Nb, grads=grads, accumulate=True)
        loss = float((res ** 2).mean() + (bres ** 2).mean())
        history.append(loss)
        for (W, b), (dW, db) in zip(params, grads):
            W.grad, b.grad = dW, db
        opt.step()
        mlp.set_weights([(W.detach(), b.detach()) for W, b in params])
        if log_every and step % log_every == 0:
            print(f"step {step:5d}  loss {loss:.4e}", flush=True)
    # relative L2 error against u* on fresh points
    xt = (torch.rand(8192, D, device=f"cuda:{device}") * 2 - 1).contiguous()
    mlp.grad_enable(False)
    _, u = mlp.laplacian(xt)
    err = float(torch.linalg.norm(u - u_star(xt)) / torch.linalg.norm(u_star(xt)))
    mlp.close()
    return history, err


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--D", type=int, default=5)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--N", type=int, default=4096)
    a = ap.parse_args()
    hist, err = train(D=a.D, steps=a.steps, N=a.N)
    print(f"final loss {hist[-1]:.4e} (first {hist[0]:.4e}); relative L2 error of u vs u*: {err:.3e}")
