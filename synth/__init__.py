"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This module holds NONE of the method's arithmetic: it only draws numbers.
Recipe:

* weights ``W_l, b_l ~ U(-1/sqrt(fan_in), +1/sqrt(fan_in))`` (the PyTorch
  ``nn.Linear`` default init), drawn in fp64 with numpy PCG64 and rounded once
  to fp32 — both sides consume the same fp32 values;
* points ``X ~ U(-1, 1)^D`` (PINN collocation cube);
* full-rank weighting ``sigma = Q diag(s)``, Q orthogonal (QR of a Gaussian),
  ``s ~ U(0.5, 1.5)``, or the paper-faithful diagonal ``sigma = diag(s)``;
* Gaussian directions ``V ~ N(0, 1)`` passed explicitly.

Seeds: weights 0, points 1, directions 2 (by convention of the callers).
"""
from __future__ import annotations

import numpy as np

# The paper's benchmark MLP: D -> 768 -> 768 -> 512 -> 512 -> 1, tanh.
PAPER_HIDDEN = (768, 768, 512, 512)


def widths_for(D: int, hidden=PAPER_HIDDEN) -> list[int]:
    return [D, *hidden, 1]


def mlp_params(widths, seed: int = 0):
    """[(W_l [w_l, w_{l-1}] fp32, b_l [w_l] fp32)] for the given widths."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for fan_in, fan_out in zip(widths[:-1], widths[1:]):
        bound = 1.0 / np.sqrt(fan_in)
        W = rng.uniform(-bound, bound, size=(fan_out, fan_in)).astype(np.float32)
        b = rng.uniform(-bound, bound, size=(fan_out,)).astype(np.float32)
        out.append((W, b))
    return out


def points(N: int, D: int, seed: int = 1) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-1.0, 1.0, size=(N, D)).astype(np.float32)


def sigma(D: int, R: int | None = None, seed: int = 3, kind: str = "dense") -> np.ndarray:
    """Weighting sigma [D, R]: 'dense' = Q diag(s) (R = D), 'diag' = diag(s),
    'rect' = Gaussian [D, R] / sqrt(R)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    R = D if R is None else R
    if kind == "diag":
        assert R == D
        return np.diag(rng.uniform(0.5, 1.5, size=D)).astype(np.float32)
    if kind == "dense":
        assert R == D
        Q, _ = np.linalg.qr(rng.standard_normal((D, D)))
        return (Q * rng.uniform(0.5, 1.5, size=D)[None, :]).astype(np.float32)
    if kind == "rect":
        return (rng.standard_normal((D, R)) / np.sqrt(R)).astype(np.float32)
    raise ValueError(kind)


def gaussian_directions(N: int, S: int, Rv: int, seed: int = 2) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((N, S, Rv)).astype(np.float32)


def sylvester_hadamard(order: int) -> np.ndarray:
    """The Sylvester-Hadamard matrix of size 2^k (entries +-1) — an exact
    Rademacher design for the unbiasedness pin."""
    H = np.array([[1.0]])
    while H.shape[0] < order:
        H = np.block([[H, H], [H, -H]])
    assert H.shape[0] == order
    return H


def sigma_field(X: np.ndarray, R: int, seed: int = 4) -> np.ndarray:
    """A smooth point-dependent weighting sigma(x) [N, D, R] ("sigma can depend on
    x0"): sigma(x)[d, r] = A[d, r] (1 + 0.5 sin(x_d + phi_r)), A Gaussian / sqrt(R)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    N, D = X.shape
    A = rng.standard_normal((D, R)) / np.sqrt(R)
    phi = rng.uniform(-np.pi, np.pi, size=R)
    return (A[None] * (1.0 + 0.5 * np.sin(X.astype(np.float64)[:, :, None] + phi[None, None, :]))).astype(np.float32)


def signed_weights(J: int, seed: int = 5) -> np.ndarray:
    """Direction weights for general directional sums: U(-1, 1), both signs."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-1.0, 1.0, size=J).astype(np.float32)
