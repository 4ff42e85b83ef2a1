"""Pins for the condition-aware fallback bound used by the small-net GPU edge tests
(tests/_util.magnitude_k2, DESIGN.md §5 reading R9). CPU only."""
import numpy as np
import pytest

import oracle as O
from tests._util import magnitude_k2, magnitude_k4, random_params


def test_magnitude_equals_value_when_nothing_cancels():
    """One hidden layer, D = 1: f'' = sum_j w2_j s''(z_j) w1_j^2. Choosing
    w2_j = sign(s''(z_j)) makes every term non-negative, so the magnitude must equal
    the exact Laplacian the oracle computes (no cancellation, nothing to bound)."""
    Ws, bs = random_params([1, 9, 1], seed=3)
    x = np.array([[0.37]])
    z = Ws[0] @ x[0] + bs[0]
    t = np.tanh(z)
    s2 = -2.0 * t * (1.0 - t * t)
    Ws[1] = np.sign(s2)[None, :] * np.abs(Ws[1])
    want, _, norm = O.laplacian(O.Net(Ws, bs), x)
    M = magnitude_k2(Ws, bs, x, np.eye(1), 1.0)
    assert want[0] > 0
    np.testing.assert_allclose(M, want, rtol=1e-13)
    np.testing.assert_allclose(M, norm, rtol=1e-13)


def test_magnitude_bounds_the_north_star_normaliser():
    """Triangle inequality: M >= sum_r |c_r f_{2,r}| for shared (Laplacian, weighted)
    and per-point (randomized) direction sets, deep nets, any signs."""
    rng = np.random.default_rng(0)
    for trial in range(12):
        D = int(rng.integers(1, 6))
        widths = [D] + [int(rng.integers(4, 40)) for _ in range(int(rng.integers(1, 4)))] + [1]
        Ws, bs = random_params(widths, seed=trial)
        net = O.Net(Ws, bs)
        X = rng.uniform(-1, 1, size=(4, D))
        _, _, norm = O.laplacian(net, X)
        assert np.all(magnitude_k2(Ws, bs, X, np.eye(D), 1.0) >= norm * (1 - 1e-12))
        sig = rng.normal(size=(D, 3))
        _, _, norm = O.weighted_laplacian(net, X, sig)
        assert np.all(magnitude_k2(Ws, bs, X, sig.T, 1.0) >= norm * (1 - 1e-12))
        V = O.rademacher(trial, 0, 4, 5, D)
        _, _, norm = O.randomized_laplacian(net, X, V)
        assert np.all(magnitude_k2(Ws, bs, X, V, 1.0 / 5) >= norm * (1 - 1e-12))


def test_magnitude_is_homogeneous_and_catches_a_dropped_term():
    """M scales with |c|; and a plausible bug (dropping the s' x2 term of Eq. 3 in one
    layer) changes the result by far more than 1e-5 M, so the fallback cannot hide it."""
    Ws, bs = random_params([3, 20, 16, 1], seed=5)
    X = np.random.default_rng(1).uniform(-1, 1, size=(6, 3))
    M = magnitude_k2(Ws, bs, X, np.eye(3), 1.0)
    np.testing.assert_allclose(magnitude_k2(Ws, bs, X, np.eye(3), -2.5), 2.5 * M, rtol=1e-14)
    want, _, _ = O.laplacian(O.Net(Ws, bs), X)
    # same propagation without the s' x2 term in the second hidden layer
    bad = np.empty(len(X))
    for n, x in enumerate(X):
        z = Ws[0] @ x + bs[0]
        t = np.tanh(z); d1 = 1 - t * t; d2 = -2 * t * d1
        x1 = d1[None, :] * Ws[0].T                      # [D, h1]
        x2 = d2[None, :] * Ws[0].T ** 2
        z0 = Ws[1] @ t + bs[1]
        z1, z2 = x1 @ Ws[1].T, x2 @ Ws[1].T
        t = np.tanh(z0); d1 = 1 - t * t; d2 = -2 * t * d1
        x2 = d2 * z1 ** 2                               # dropped: + d1 * z2
        bad[n] = float((x2 @ Ws[2][0]).sum())
    assert np.all(np.abs(bad - want) > 1e-3 * M)


def test_magnitude_k4_equals_value_when_nothing_cancels():
    """One hidden layer, D = 1: f'''' = sum_j w2_j s''''(z_j) w1_j^4. With
    w2_j = sign(s''''(z_j)) every term is non-negative, so M equals the exact f''''."""
    Ws, bs = random_params([1, 9, 1], seed=4)
    x = np.array([[0.21]])
    z = Ws[0] @ x[0] + bs[0]
    t = np.tanh(z)
    s4 = 8 * t * (1 - t * t) * (2 - 3 * t * t)
    Ws[1] = np.sign(s4)[None, :] * np.abs(Ws[1])
    want, _, _ = O.biharmonic(O.Net(Ws, bs), x)
    assert want[0] > 0
    np.testing.assert_allclose(magnitude_k4(Ws, bs, x, np.eye(1), 1.0), want, rtol=1e-12)


@pytest.mark.parametrize("act", ["tanh", "sin"])
def test_magnitude_k4_bounds_the_normaliser(act):
    """Triangle inequality: M >= sum_j |c_j f_{4,j}| for the biharmonic family and for
    random weighted jets (shared and per point), deep nets, any signs."""
    rng = np.random.default_rng(2)
    for trial in range(8):
        D = int(rng.integers(1, 5))
        widths = [D] + [int(rng.integers(4, 30)) for _ in range(int(rng.integers(1, 4)))] + [1]
        Ws, bs = random_params(widths, seed=trial)
        net = O.Net(Ws, bs, act)
        X = rng.uniform(-1, 1, size=(3, D))
        dirs, coef = O.biharmonic_set(D)
        _, _, norm = O.biharmonic(net, X)
        assert np.all(magnitude_k4(Ws, bs, X, dirs, coef, act) >= norm * (1 - 1e-12))
        U = rng.normal(size=(3, 4, D))
        w = rng.normal(size=4)
        _, _, norm = O.directional_sum(net, X, 4, U, w)
        assert np.all(magnitude_k4(Ws, bs, X, U, w, act) >= norm * (1 - 1e-12))


def test_magnitude_k4_catches_a_dropped_term():
    """Dropping any one term of the K = 4 rule in one layer moves f'''' by more than
    10x the fallback tolerance (1e-5 M), so the fallback cannot hide that bug."""
    Ws, bs = random_params([1, 12, 10, 1], seed=9)
    x = np.array([0.3])
    want = O.biharmonic(O.Net(Ws, bs, "tanh"), x[None, :])[0][0]

    def derivs(z):
        t = np.tanh(z)
        s1 = 1 - t * t
        return t, s1, -2 * t * s1, s1 * (6 * t * t - 2), 8 * t * s1 * (2 - 3 * t * t)

    t, s1, s2, s3, s4 = derivs(Ws[0] @ x + bs[0])
    u = Ws[0][:, 0]
    x1, x2, x3, x4 = s1 * u, s2 * u**2, s3 * u**3, s4 * u**4
    z1, z2, z3, z4 = Ws[1] @ x1, Ws[1] @ x2, Ws[1] @ x3, Ws[1] @ x4
    _, s1, s2, s3, s4 = derivs(Ws[1] @ t + bs[1])
    good = s4 * z1**4 + 6 * s3 * z1**2 * z2 + 4 * s2 * z1 * z3 + 3 * s2 * z2**2 + s1 * z4
    np.testing.assert_allclose(Ws[2][0] @ good, want, rtol=1e-10)  # the restated rule is the oracle's
    M = magnitude_k4(Ws, bs, x[None, :], np.eye(1), 1.0)[0]
    for term in (s4 * z1**4, 6 * s3 * z1**2 * z2, 4 * s2 * z1 * z3, 3 * s2 * z2**2, s1 * z4):
        bad = Ws[2][0] @ (good - term)
        assert abs(bad - want) > 1e-4 * M  # 10x the fallback tolerance 1e-5 M


@pytest.mark.parametrize("K,act", [(2, "tanh"), (4, "tanh"), (2, "sin"), (4, "sin")])
def test_vanilla32_is_the_vanilla_rules_in_fp32(K, act):
    """The plain-fp32 reference of reading R9 (tests/_util.vanilla32) computes the operator:
    on a well-conditioned small net it matches the fp64 oracle to fp32 accuracy, and it is
    genuinely fp32 (not bitwise the fp64 value)."""
    from synth import mlp_params, points
    from tests._util import vanilla32

    params = mlp_params([3, 24, 16, 1], 5)
    net = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params], act)
    X = points(6, 3, seed=5)
    dirs = np.random.default_rng(5).standard_normal((4, 3)).astype(np.float32)
    w = np.array([0.5, -1.0, 2.0, 0.25], np.float32)
    want, _, norm = O.directional_sum(net, X.astype(np.float64), K, dirs.astype(np.float64), w.astype(np.float64))
    got = vanilla32(params, act, X, dirs, w, K)
    err = np.abs(got - want) / norm
    assert err.max() <= 1e-4
    assert np.any(got != want)
