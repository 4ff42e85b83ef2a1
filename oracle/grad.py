"""fp64 oracle for the DIFFERENTIABLE path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline leg may
import this module; the product package never does, and nothing here is shared with the
CUDA path.

Plain PyTorch CPU ops in fp64 (no blocking, no fusion). The K = 2 operators are
evaluated by VANILLA Taylor mode (Eq. D1): the primal is shared,
each direction u_j carries its own 2-jet (x1 = u_j, x2 = 0), through every layer

    affine:  z0 = W h0 + b,  z1 = W h1,  z2 = W h2
    activation (Eq. 1, Faa di Bruno K = 2):
                     h0 = s(z0),  h1 = s'(z0) z1,  h2 = s''(z0) z1^2 + s'(z0) z2

and the output's top coefficients f_{2,j} are sliced and combined,
op = sum_j w_j f_{2,j} (Eq. 5 with weights; w = 1 for the exact and weighted
Laplacians, 1/S for the randomized one). The parameter gradient of
L = sum_n gop[n] op[n] + gf[n] f[n] is torch.autograd's reverse mode of exactly
this computation — the plain definition of d L / d theta.

Pins (tests/test_oracle_grad.py): the values equal the C oracle (ctmo.c, route O1);
the gradients equal central finite differences of the C oracle's L(theta) (independent
code) and the closed form of a one-hidden-layer net.
"""
from __future__ import annotations

import numpy as np
import torch

_ACTS = ("tanh", "identity", "square", "sin", "exp")


def _derivs(act: str, z: torch.Tensor):
    """s, s', s'' of the activation (textbook derivatives)."""
    if act == "tanh":
        t = torch.tanh(z)
        return t, 1 - t * t, -2 * t * (1 - t * t)
    if act == "sin":
        return torch.sin(z), torch.cos(z), -torch.sin(z)
    if act == "square":
        return z * z, 2 * z, torch.full_like(z, 2.0)
    if act == "exp":
        e = torch.exp(z)
        return e, e, e
    if act == "identity":
        return z, torch.ones_like(z), torch.zeros_like(z)
    raise ValueError(act)


def k2_operator(Ws, bs, X, dirs, w, act: str = "tanh"):
    """(op [N], f [N]) as differentiable fp64 torch functions of Ws, bs.

    Ws[l]: [w_{l+1}, w_l] (nn.Linear layout), bs[l]: [w_{l+1}]; X [N, D];
    dirs [J, D] (the same for every point) or [N, J, D]; w [J]."""
    X = torch.as_tensor(X, dtype=torch.float64)
    dirs = torch.as_tensor(dirs, dtype=torch.float64)
    w = torch.as_tensor(w, dtype=torch.float64)
    N = X.shape[0]
    if dirs.dim() == 2:
        dirs = dirs.unsqueeze(0).expand(N, -1, -1)
    h0, h1 = X, dirs                       # [N, D], [N, J, D]
    h2 = torch.zeros_like(dirs)
    L = len(Ws)
    for l in range(L):
        W, b = Ws[l], bs[l]
        z0 = h0 @ W.T + b
        z1 = h1 @ W.T
        z2 = h2 @ W.T
        if l == L - 1:
            return (z2[..., 0] * w).sum(-1), z0[:, 0]
        s0, s1, s2 = _derivs(act, z0)
        h0 = s0
        h1 = s1.unsqueeze(1) * z1
        h2 = s2.unsqueeze(1) * z1 * z1 + s1.unsqueeze(1) * z2


def k2_grad(Ws, bs, X, dirs, w, gop, gf=None, act: str = "tanh"):
    """Gradients of L = sum_n gop[n] op[n] + gf[n] f[n] w.r.t. every W_l, b_l (fp64 numpy).
    Returns (op, f, [dW_l], [db_l])."""
    Wt = [torch.tensor(np.asarray(W, dtype=np.float64), requires_grad=True) for W in Ws]
    bt = [torch.tensor(np.asarray(b, dtype=np.float64).reshape(-1), requires_grad=True) for b in bs]
    op, f = k2_operator(Wt, bt, X, dirs, w, act)
    loss = (torch.as_tensor(gop, dtype=torch.float64) * op).sum()
    if gf is not None:
        loss = loss + (torch.as_tensor(gf, dtype=torch.float64) * f).sum()
    grads = torch.autograd.grad(loss, Wt + bt, allow_unused=True)
    grads = [torch.zeros_like(p) if g is None else g for g, p in zip(grads, Wt + bt)]
    L = len(Ws)
    return (op.detach().numpy(), f.detach().numpy(), [g.numpy() for g in grads[:L]],
            [g.numpy() for g in grads[L:]])


def k2_grad_magnitude(Ws, bs, X, dirs, w, gop, gf=None, act: str = "tanh"):
    """Per-element magnitude of the parameter gradients (the gradient analogue of the
    north_star normaliser, reading R10 of DESIGN.md §3): the same vanilla computation as
    k2_operator, and for every affine layer z_k = W h_k (+ b for k = 0) the sum of the
    ABSOLUTE values of the terms of its final contraction,
        M_W[l] = |z0_bar|^T |h0| + sum_j (|z1_bar_j|^T |h1_j| + |z2_bar_j|^T |h2_j|),
        M_b[l] = sum_n |z0_bar|,
    with z_bar the fp64 adjoints dL/dz of that layer. M >= |dL/dtheta| elementwise, with
    equality when no two terms of an element differ in sign. Returns ([M_W], [M_b])."""
    X = torch.as_tensor(X, dtype=torch.float64)
    dirs = torch.as_tensor(dirs, dtype=torch.float64)
    w = torch.as_tensor(w, dtype=torch.float64)
    Wt = [torch.as_tensor(np.asarray(W, dtype=np.float64)) for W in Ws]
    bt = [torch.as_tensor(np.asarray(b, dtype=np.float64).reshape(-1)) for b in bs]
    N = X.shape[0]
    if dirs.dim() == 2:
        dirs = dirs.unsqueeze(0).expand(N, -1, -1)
    h0, h1 = X, dirs
    h2 = torch.zeros_like(dirs)
    ins, zs = [], []
    L = len(Wt)
    for l in range(L):
        z0 = (h0 @ Wt[l].T + bt[l]).requires_grad_(True)
        z1 = (h1 @ Wt[l].T).requires_grad_(True)
        z2 = (h2 @ Wt[l].T).requires_grad_(True)
        ins.append((h0.detach(), h1.detach(), h2.detach()))
        zs.append((z0, z1, z2))
        if l == L - 1:
            op, f = (z2[..., 0] * w).sum(-1), z0[:, 0]
            break
        s0, s1, s2 = _derivs(act, z0)
        h0 = s0
        h1 = s1.unsqueeze(1) * z1
        h2 = s2.unsqueeze(1) * z1 * z1 + s1.unsqueeze(1) * z2
    loss = (torch.as_tensor(gop, dtype=torch.float64) * op).sum()
    if gf is not None:
        loss = loss + (torch.as_tensor(gf, dtype=torch.float64) * f).sum()
    flat = [z for t in zs for z in t]
    bars = torch.autograd.grad(loss, flat, allow_unused=True)
    bars = [torch.zeros_like(z) if g is None else g for g, z in zip(bars, flat)]
    MW, Mb = [], []
    for l in range(L):
        zb0, zb1, zb2 = (bars[3 * l + k].abs() for k in range(3))
        a0, a1, a2 = (t.abs() for t in ins[l])
        MW.append((zb0.T @ a0 + torch.einsum("njo,nji->oi", zb1, a1) + torch.einsum("njo,nji->oi", zb2, a2)).numpy())
        Mb.append(zb0.sum(0).numpy())
    return MW, Mb
