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
