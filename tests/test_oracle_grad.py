"""Pins of the differentiable-path oracle (oracle/grad.py), CPU only."""
import numpy as np
import pytest

import oracle as O
from oracle import grad as OG
from tests._util import random_params


def _pts(N, D, seed=5):
    return np.random.default_rng(seed).uniform(-1, 1, size=(N, D))


@pytest.mark.parametrize("act", ["tanh", "sin", "exp"])
def test_values_match_the_c_oracle(act):
    D = 4
    Ws, bs = random_params([D, 9, 7, 1], 3, scale=1.5)
    net = O.Net(Ws, bs, act)
    X = _pts(5, D)
    rng = np.random.default_rng(6)
    sig = rng.standard_normal((D, 3))
    op, f, _, _ = OG.k2_grad(Ws, bs, X, sig.T, np.ones(3), np.ones(5), act=act)
    want, fw, _ = O.weighted_laplacian(net, X, sig)
    np.testing.assert_allclose(op, want, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(f, fw, rtol=1e-13)
    V = rng.standard_normal((5, 6, D))
    op, _, _, _ = OG.k2_grad(Ws, bs, X, V, np.full(6, 1 / 6), np.ones(5), act=act)
    np.testing.assert_allclose(op, O.randomized_laplacian(net, X, V)[0], rtol=1e-12, atol=1e-14)


def test_gradients_match_finite_differences_of_the_c_oracle():
    """Central differences (Richardson) of L(theta) = sum gop*op + gf*f through ctmo.c,
    every parameter of a small net: independent code, same definition."""
    D = 3
    Ws, bs = random_params([D, 5, 4, 1], 7, scale=1.5)
    X = _pts(4, D)
    gop = np.array([0.7, -1.2, 0.4, 2.0])
    gf = np.array([0.3, 0.1, -0.5, 0.8])
    _, _, dW, db = OG.k2_grad(Ws, bs, X, np.eye(D), np.ones(D), gop, gf)

    def L(Ws_, bs_):
        op, f, _ = O.laplacian(O.Net(Ws_, bs_), X)
        return float(gop @ op + gf @ f)

    def fd(get, setv):
        def g(h):
            setv(+h); a = L(Ws, bs)
            setv(-2 * h); b = L(Ws, bs)
            setv(+h)
            return (a - b) / (2 * h)
        return (4 * g(1e-4) - g(2e-4)) / 3

    for l in range(len(Ws)):
        for idx in np.ndindex(Ws[l].shape):
            def setv(dh, l=l, idx=idx):
                Ws[l][idx] += dh
            assert abs(fd(None, setv) - dW[l][idx]) < 1e-7 * max(1.0, abs(dW[l][idx])), (l, idx)
        for i in range(bs[l].size):
            def setv(dh, l=l, i=i):
                bs[l][i] += dh
            assert abs(fd(None, setv) - db[l][i]) < 1e-7 * max(1.0, abs(db[l][i])), (l, i)


def test_one_hidden_layer_closed_form_gradient():
    """f = sum_j c_j tanh(w_j.x + b_j) + b2: Laplacian = sum_j c_j tanh''(z_j) |w_j|^2,
    so d op / d c_j = tanh''(z_j) |w_j|^2 and d op / d b2 = 0, d f / d b2 = 1."""
    D, H = 3, 6
    Ws, bs = random_params([D, H, 1], 11, scale=2.0)
    X = _pts(1, D)
    _, _, dW, db = OG.k2_grad(Ws, bs, X, np.eye(D), np.ones(D), np.ones(1), np.zeros(1))
    z = Ws[0] @ X[0] + bs[0]
    t = np.tanh(z)
    np.testing.assert_allclose(dW[1][0], -2 * t * (1 - t * t) * np.sum(Ws[0] ** 2, 1), rtol=1e-12)
    assert db[1][0] == 0.0
    _, _, _, db = OG.k2_grad(Ws, bs, X, np.eye(D), np.ones(D), np.zeros(1), np.ones(1))
    assert db[1][0] == 1.0


# ------------------------------------------------------------------ gradient magnitude (R10)
@pytest.mark.parametrize("act", ["tanh", "sin"])
def test_gradient_magnitude_bounds_every_element(act):
    """M = sum of |terms| of each gradient element's final contraction bounds |g| elementwise
    (triangle inequality), and is strictly larger where terms cancel."""
    D = 4
    Ws, bs = random_params([D, 9, 7, 1], 11, scale=1.5)
    X = _pts(6, D, seed=8)
    rng = np.random.default_rng(12)
    dirs, w = rng.standard_normal((5, D)), rng.standard_normal(5)
    gop, gf = rng.standard_normal(6), rng.standard_normal(6)
    _, _, dW, db = OG.k2_grad(Ws, bs, X, dirs, w, gop, gf, act=act)
    MW, Mb = OG.k2_grad_magnitude(Ws, bs, X, dirs, w, gop, gf, act=act)
    strict = 0
    for g, m in zip(dW + db, MW + Mb):
        assert g.shape == np.shape(m)
        assert np.all(m >= np.abs(g) * (1 - 1e-12) - 1e-300)
        strict += int(np.sum(m > 1.01 * np.abs(g)))
    assert strict > 0


def test_gradient_magnitude_equals_the_gradient_when_no_term_can_cancel():
    """All weights, biases, inputs, directions and cotangents positive with the square
    activation (s, s', s'' >= 0 on z > 0): every term of every element is >= 0, so M = |g|
    exactly. A dropped or sign-flipped term in M breaks this equality."""
    rng = np.random.default_rng(0)
    Ws = [np.abs(rng.standard_normal((6, 3))), np.abs(rng.standard_normal((5, 6))), np.abs(rng.standard_normal((1, 5)))]
    bs = [np.abs(rng.standard_normal(6)), np.abs(rng.standard_normal(5)), np.abs(rng.standard_normal(1))]
    X = np.abs(rng.standard_normal((4, 3)))
    dirs = np.abs(rng.standard_normal((2, 3)))
    gop, gf = np.abs(rng.standard_normal(4)), np.abs(rng.standard_normal(4))
    _, _, dW, db = OG.k2_grad(Ws, bs, X, dirs, np.ones(2), gop, gf, act="square")
    MW, Mb = OG.k2_grad_magnitude(Ws, bs, X, dirs, np.ones(2), gop, gf, act="square")
    for g, m in zip(dW + db, MW + Mb):
        np.testing.assert_allclose(m, np.abs(g), rtol=1e-13, atol=0)
        assert np.all(m > 0)


def test_gradient_magnitude_is_homogeneous_in_the_cotangents():
    D = 3
    Ws, bs = random_params([D, 8, 6, 1], 4)
    X = _pts(5, D, seed=2)
    gop, gf = np.linspace(-1, 1, 5), np.linspace(0.3, -0.7, 5)
    a = OG.k2_grad_magnitude(Ws, bs, X, np.eye(D), np.ones(D), gop, gf)
    b = OG.k2_grad_magnitude(Ws, bs, X, np.eye(D), np.ones(D), -2.5 * gop, -2.5 * gf)
    for x, y in zip(a[0] + a[1], b[0] + b[1]):
        np.testing.assert_allclose(y, 2.5 * np.asarray(x), rtol=1e-13)
