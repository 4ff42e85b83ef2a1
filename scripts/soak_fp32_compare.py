"""Soak analysis: are the fuzz points that miss the north_star metric arithmetic-limited?

For the fuzz cases the expanded GPU soak flagged (CTM_FUZZ_* env, profiles/r01/soak/),
rebuild the same seeded nets, points and directions as tests/test_gpu_parity.py and
evaluate every operator of the case twice on the CPU:
  - the fp64 oracle (oracle/, the reference value and the north_star normaliser);
  - a plain fp32 evaluation of the same vanilla Taylor rules (Eq. 3, per direction,
    numpy float32 end to end, BLAS sgemm).
It prints the worst fp32 err/norm per operator. If plain fp32 also misses 1e-4 at these
points, the miss comes from the conditioning of the point, not from the kernels.
Analysis tool (imports oracle/), not part of the product."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from synth import gaussian_directions, mlp_params, points, sigma as make_sigma, sigma_field, signed_weights  # noqa: E402


from tests._util import vanilla32  # noqa: E402  (plain fp32 vanilla Taylor rules)


def report(tag, got32, want, norm):
    e = np.abs(got32 - want) / norm
    print(f"  {tag:28s} fp32 max err/norm {e.max():.2e}  points > 1e-4: {int((e > 1e-4).sum())}/{e.size}")


def shapes_case(case):
    rng = np.random.default_rng(1000 + case)
    D = int(rng.integers(1, 41))
    depth = int(rng.integers(1, 4))
    hidden = [int(rng.integers(8, 321)) for _ in range(depth)]
    widths = [D] + hidden + [1]
    N = int(rng.integers(1, 71))
    params = mlp_params(widths, case)
    net = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params], "tanh")
    X = points(N, D, seed=case)
    Xd = X.astype(np.float64)
    print(f"shapes[{case}] widths {widths} N {N}")
    want, _, norm = O.laplacian(net, Xd)
    report("laplacian", vanilla32(params, "tanh", X, np.eye(D), 1.0, 2), want, norm)
    R = int(rng.integers(1, 300))
    sig = make_sigma(D, R, kind="rect")
    want, _, norm = O.weighted_laplacian(net, Xd, sig.astype(np.float64))
    report("weighted", vanilla32(params, "tanh", X, sig.T, 1.0, 2), want, norm)
    S = int(rng.integers(1, 300))
    V = O.rademacher(7, 0, N, S, D)
    want, _, norm = O.randomized_laplacian(net, Xd, V)
    report("randomized", vanilla32(params, "tanh", X, V, 1.0 / S, 2), want, norm)
    if D <= 8:
        want, _, norm = O.biharmonic(net, Xd)
        dirs, c = O.biharmonic_set(D)
        report("biharmonic", vanilla32(params, "tanh", X, dirs, c, 4), want, norm)
        Sg = int(rng.integers(1, 40))
        Vg = gaussian_directions(N, Sg, D, seed=case)
        want, _, norm = O.stochastic_biharmonic(net, Xd, Vg.astype(np.float64), O.O1)
        report("stochastic biharmonic", vanilla32(params, "tanh", X, Vg, 1.0 / (3 * Sg), 4), want, norm)


def dsum_case(case):
    rng = np.random.default_rng(3000 + case)
    D = int(rng.integers(1, 24))
    hidden = [int(rng.integers(65, 300)) for _ in range(int(rng.integers(1, 4)))]
    widths = [D] + hidden + [1]
    act = ["tanh", "sin"][case % 2]
    N = int(rng.integers(1, 50))
    params = mlp_params(widths, 100 + case)
    net = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params], act)
    X = points(N, D, seed=case)
    Xd = X.astype(np.float64)
    print(f"dsum[{case}] widths {widths} N {N} act {act}")
    rng.integers(0, 40)  # the forced block size (GPU only)
    for K in (2, 4):
        J = int(rng.integers(1, 120 if K == 2 else 50))
        w = signed_weights(J, seed=case)
        per_point = bool(rng.integers(0, 2))
        dirs = gaussian_directions(N, J, D, seed=case) if per_point else gaussian_directions(1, J, D, seed=case)[0]
        if K == 4 and per_point and J * D > 12288:
            continue
        want, _, norm = O.directional_sum(net, Xd, K, dirs.astype(np.float64), w.astype(np.float64))
        report(f"directional K={K} J={J}", vanilla32(params, act, X, dirs, w, K), want, norm)
    R = int(rng.integers(1, 80))
    sx = sigma_field(X, R, seed=case)
    want, _, norm = O.weighted_laplacian_pointwise(net, Xd, sx.astype(np.float64))
    report("sigma(x)", vanilla32(params, act, X, sx.transpose(0, 2, 1), 1.0, 2), want, norm)


def k4_case(case):
    rng = np.random.default_rng(4000 + case)
    D = int(rng.integers(1, 13))
    hidden = [int(rng.integers(65, 300)) for _ in range(int(rng.integers(1, 4)))]
    widths = [D] + hidden + [1]
    N = int(rng.integers(1, 40))
    params = mlp_params(widths, 200 + case)
    net = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params], "tanh")
    X = points(N, D, seed=case)
    Xd = X.astype(np.float64)
    print(f"k4[{case}] widths {widths} N {N}")
    want, _, norm = O.biharmonic(net, Xd)
    dirs, c = O.biharmonic_set(D)
    report("biharmonic", vanilla32(params, "tanh", X, dirs, c, 4), want, norm)


if __name__ == "__main__":
    for c in (95, 115, 148):
        shapes_case(c)
    for c in (12, 14, 94, 103):
        dsum_case(c)
    for c in (14, 37, 45, 59, 62):
        k4_case(c)
