"""Pins for the fp64 oracle (oracle/ctmo.c) against things other than itself:
the paper's printed numbers (tests/golden/), closed forms, finite differences,
torch fp64 autograd, exact designs and statistical unbiasedness.

All CPU-only (-m "not gpu").
"""
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle as O
from synth import sylvester_hadamard
from tests._util import golden, random_params, rel_err

ROUTES = [O.O1, O.O2, O.O3]


@pytest.fixture(scope="module", autouse=True)
def _build():
    O.build()


# --------------------------------------------------------------------------
# Bookkeeping pins
# --------------------------------------------------------------------------
def test_splitmix64_reference_vectors():
    for seed, idx, hexval in ((r[0].split()[0], r[0].split()[1], r[1]) for r in golden("splitmix64.txt")):
        assert O.splitmix64(int(seed), int(idx)) == int(hexval, 16)


def test_rademacher_values_and_shard_invariance():
    V = O.rademacher(7, 0, 10, 3, 5)
    assert set(np.unique(V)) <= {-1.0, 1.0}
    # global-index keyed: the shard starting at point 4 sees the same draws
    V2 = O.rademacher(7, 4, 6, 3, 5)
    np.testing.assert_array_equal(V[4:], V2)
    # the sign is the top bit of splitmix64(seed, ((n*S)+s)*Rv+d)
    n, s, d = 3, 2, 4
    top = O.splitmix64(7, (n * 3 + s) * 5 + d) >> 63
    assert V[n, s, d] == (-1.0 if top else 1.0)
    big = O.rademacher(11, 0, 2000, 4, 8)
    assert abs(big.mean()) < 4.0 / math.sqrt(big.size)


def test_partition_counts():
    # the partition numbers p(k), OEIS A000041
    assert [len(O.partitions(k)) for k in range(1, 9)] == [1, 2, 3, 5, 7, 11, 15, 22]


def test_nu_matches_paper_cheatsheet():
    rows = golden("faa_di_bruno_nu.txt")
    want = {}
    for k, parts, nu, _src in rows:
        want.setdefault(int(k), {})[tuple(int(p) for p in parts.split())] = int(nu)
    for k in range(1, 9):
        got = {parts: nu for parts, nu in O.partitions(k)}
        assert got == want[k], k


def test_nu_sums_to_bell_numbers():
    # sum_sigma nu(sigma) counts the set partitions of a k-set (Bell numbers)
    bell = [1, 2, 5, 15, 52, 203, 877, 4140]
    assert [sum(nu for _, nu in O.partitions(k)) for k in range(1, 9)] == bell


def test_gamma_matches_fig3():
    for j, num, den, _src in golden("gamma_biharmonic.txt"):
        j1, j2 = (int(x) for x in j.split())
        assert O.gamma((2, 2), (j1, j2)) == Fraction(int(num), int(den))


def test_gamma_reproduces_pure_power_and_unit_index():
    # i = (K, 0): the only member with nonzero weight is j = i, gamma = K! / K^K * K^K/K! ... :
    # <d^K f, v^K> = gamma_{i,i}/K! <d^K f, (K v)^K>  =>  gamma_{(K,0),(K,0)} = K!/K^K
    for K in (1, 2, 3, 4):
        assert O.gamma((K, 0), (K, 0)) == Fraction(math.factorial(K), K**K)
        for j1 in range(K):
            assert O.gamma((K, 0), (j1, K - j1)) == 0


def test_vector_counts_match_table():
    for op, D, std, col, ratio, _src in golden("vector_counts.txt"):
        D, std, col = int(D), int(std), int(col)
        if op in ("laplacian", "weighted"):
            R = D
            assert (1 + 2 * R, 2 + R) == (std, col)
        else:
            dirs, _ = O.biharmonic_set(D)
            J = dirs.shape[0]
            assert J == D * (3 * D - 1) // 2
            # standard: 1 + 4J ; paper's collapse: 1 + 3J + one per interpolation group (3)
            assert (1 + 4 * J, 1 + 3 * J + 3) == (std, col)
        assert round(col / std, 2) == float(ratio)


def test_biharmonic_set_1d_is_fourth_derivative():
    # D = 1: only 4 e_1 with c = (2 g40 + 2 g31 + g22)/24; c * 4^4 must be 1
    dirs, coef = O.biharmonic_set(1)
    assert dirs.shape == (1, 1) and dirs[0, 0] == 4.0
    assert abs(coef[0] * 256.0 - 1.0) < 1e-15


# --------------------------------------------------------------------------
# Activation derivatives: central differences
# --------------------------------------------------------------------------
@pytest.mark.parametrize("act", ["tanh", "sin", "exp", "square", "identity"])
def test_act_derivs_finite_differences(act):
    ref0 = {"tanh": np.tanh, "sin": np.sin, "exp": np.exp, "square": np.square, "identity": lambda z: z}[act]
    h = 1e-4
    for z in (-1.3, -0.2, 0.0, 0.4, 1.1, 2.2):
        d = O.act_derivs(act, z)
        assert abs(d[0] - ref0(z)) < 1e-15
        for k in range(4):
            fd = (O.act_derivs(act, z + h)[k] - O.act_derivs(act, z - h)[k]) / (2 * h)
            assert abs(fd - d[k + 1]) < 1e-7, (act, z, k)


# --------------------------------------------------------------------------
# Closed forms through MLP-shaped nets (all three routes)
# --------------------------------------------------------------------------
def _pts(N, D, seed=5):
    return np.random.default_rng(seed).uniform(-1, 1, size=(N, D))


@pytest.mark.parametrize("route", ROUTES)
def test_linear_net_has_zero_operators(route):
    Ws, bs = random_params([4, 7, 5, 1], 1)
    net = O.Net(Ws, bs, "identity")
    X = _pts(3, 4)
    sig = np.random.default_rng(2).standard_normal((4, 3))
    for op in (O.laplacian(net, X, route)[0], O.weighted_laplacian(net, X, sig, route)[0],
               O.biharmonic(net, X, route)[0]):
        assert np.max(np.abs(op)) < 1e-13


@pytest.mark.parametrize("route", ROUTES)
def test_quadratic_net_known_hessian(route):
    # f = sum_j c_j (w_j^T x + b_j)^2 + b2  =>  H = 2 sum_j c_j w_j w_j^T
    D, H = 5, 6
    Ws, bs = random_params([D, H, 1], 3, scale=2.0)
    net = O.Net(Ws, bs, "square")
    X = _pts(4, D)
    W1, c = Ws[0], Ws[1][0]
    Hess = 2 * (W1.T * c) @ W1
    sig = np.random.default_rng(4).standard_normal((D, 3))
    np.testing.assert_allclose(O.laplacian(net, X, route)[0], np.trace(Hess), rtol=1e-13)
    np.testing.assert_allclose(O.weighted_laplacian(net, X, sig, route)[0], np.sum(Hess * (sig @ sig.T)), rtol=1e-13)
    assert np.max(np.abs(O.biharmonic(net, X, route)[0])) < 1e-12
    f = O.forward(net, X)
    np.testing.assert_allclose(f, ((X @ W1.T + bs[0]) ** 2) @ c + bs[1][0], rtol=1e-13)


def _norm4_net(D):
    # square(1^T square(x)) = ||x||^4, then an identity output layer
    Ws = [np.eye(D), np.ones((1, D)), np.ones((1, 1))]
    bs = [np.zeros(D), np.zeros(1), np.zeros(1)]
    return O.Net(Ws, bs, "square")


@pytest.mark.parametrize("route", ROUTES)
@pytest.mark.parametrize("D", [2, 3, 5])
def test_norm4_closed_forms(route, D):
    net = _norm4_net(D)
    X = _pts(3, D)
    r2 = np.sum(X**2, axis=1)
    np.testing.assert_allclose(O.forward(net, X), r2**2, rtol=1e-14)
    np.testing.assert_allclose(O.laplacian(net, X, route)[0], 4 * (D + 2) * r2, rtol=1e-13)
    np.testing.assert_allclose(O.biharmonic(net, X, route)[0], 8 * D * (D + 2), rtol=1e-12)


@pytest.mark.parametrize("route", ROUTES)
def test_mixed_quartic_x1sq_x2sq(route):
    # x1^2 x2^2 = ((x1+x2)^4 + (x1-x2)^4 - 2 x1^4 - 2 x2^4) / 12  as a square-square net
    W1 = np.array([[1.0, 1.0], [1.0, -1.0], [1.0, 0.0], [0.0, 1.0]])
    W2 = np.eye(4)
    W3 = np.array([[1.0, 1.0, -2.0, -2.0]]) / 12.0
    net = O.Net([W1, W2, W3], [np.zeros(4), np.zeros(4), np.zeros(1)], "square")
    X = _pts(4, 2)
    np.testing.assert_allclose(O.forward(net, X), X[:, 0] ** 2 * X[:, 1] ** 2, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(O.laplacian(net, X, route)[0], 2 * X[:, 0] ** 2 + 2 * X[:, 1] ** 2, rtol=1e-12)
    np.testing.assert_allclose(O.biharmonic(net, X, route)[0], 8.0, rtol=1e-12)


@pytest.mark.parametrize("route", ROUTES)
def test_sum_of_sines(route):
    rng = np.random.default_rng(9)
    D = 4
    bvec, phi, a = rng.uniform(0.5, 2, D), rng.uniform(-1, 1, D), rng.uniform(-1, 1, D)
    net = O.Net([np.diag(bvec), a[None, :]], [phi, np.array([0.3])], "sin")
    X = _pts(5, D)
    s = np.sin(X * bvec + phi)
    np.testing.assert_allclose(O.laplacian(net, X, route)[0], -(s * a * bvec**2).sum(1), rtol=1e-12)
    np.testing.assert_allclose(O.biharmonic(net, X, route)[0], (s * a * bvec**4).sum(1), rtol=1e-11)
    sig = rng.standard_normal((D, 2))
    diagD = np.sum(sig**2, axis=1)  # (sigma sigma^T)_dd ; H is diagonal
    np.testing.assert_allclose(O.weighted_laplacian(net, X, sig, route)[0], -(s * a * bvec**2 * diagD).sum(1), rtol=1e-12)



@pytest.mark.parametrize("route", ROUTES)
def test_sum_of_exponentials(route):
    # f = sum_j c_j exp(a_j^T x + b_j) (exp activation): every derivative of
    # exp is exp, so Laplacian = sum_j c_j e_j ||a_j||^2, weighted: ||sigma^T a_j||^2,
    # biharmonic = sum_j c_j e_j ||a_j||^4.
    rng = np.random.default_rng(10)
    D, H = 3, 4
    A, b, c = rng.uniform(-0.8, 0.8, (H, D)), rng.uniform(-0.5, 0.5, H), rng.uniform(-1, 1, H)
    net = O.Net([A, c[None, :]], [b, np.array([0.2])], "exp")
    X = _pts(5, D)
    e = np.exp(X @ A.T + b)
    n2 = np.sum(A**2, 1)
    np.testing.assert_allclose(O.forward(net, X), e @ c + 0.2, rtol=1e-13)
    np.testing.assert_allclose(O.laplacian(net, X, route)[0], e @ (c * n2), rtol=1e-12)
    np.testing.assert_allclose(O.biharmonic(net, X, route)[0], e @ (c * n2**2), rtol=1e-11)
    sig = rng.standard_normal((D, 2))
    np.testing.assert_allclose(O.weighted_laplacian(net, X, sig, route)[0], e @ (c * np.sum((A @ sig) ** 2, 1)),
                               rtol=1e-12)


def _tanh_derivs_autograd(z, k):
    """k-th derivative of tanh at z by torch autograd (independent of the oracle)."""
    zt = torch.tensor(z, dtype=torch.float64, requires_grad=True)
    y = torch.tanh(zt)
    for _ in range(k):
        (y,) = torch.autograd.grad(y.sum(), zt, create_graph=True)
    return y.detach().numpy()


@pytest.mark.parametrize("route", ROUTES)
def test_one_hidden_layer_tanh_closed_forms(route):
    # f = sum_j c_j tanh(w_j^T x + b_j) + b2:
    #   Laplacian = sum_j c_j tanh''(z_j) ||w_j||^2,  weighted: ||sigma^T w_j||^2,
    #   biharmonic = sum_j c_j tanh''''(z_j) ||w_j||^4
    D, H = 5, 7
    Ws, bs = random_params([D, H, 1], 11, scale=2.0)
    net = O.Net(Ws, bs, "tanh")
    X = _pts(4, D)
    W1, c = Ws[0], Ws[1][0]
    Z = X @ W1.T + bs[0]
    t2, t4 = _tanh_derivs_autograd(Z, 2), _tanh_derivs_autograd(Z, 4)
    sig = np.random.default_rng(12).standard_normal((D, 3))
    nw = np.sum(W1**2, 1)
    np.testing.assert_allclose(O.laplacian(net, X, route)[0], (t2 * c * nw).sum(1), rtol=1e-12)
    np.testing.assert_allclose(O.weighted_laplacian(net, X, sig, route)[0],
                               (t2 * c * np.sum((W1 @ sig) ** 2, 1)).sum(1), rtol=1e-12)
    np.testing.assert_allclose(O.biharmonic(net, X, route)[0], (t4 * c * nw**2).sum(1), rtol=1e-11)


# --------------------------------------------------------------------------
# torch fp64 autograd on deeper tanh nets
# --------------------------------------------------------------------------
def _torch_f(Ws, bs):
    Wt = [torch.tensor(W) for W in Ws]
    bt = [torch.tensor(b) for b in bs]

    def f(x):
        h = x
        for l, (W, b) in enumerate(zip(Wt, bt)):
            h = h @ W.T + b
            if l < len(Wt) - 1:
                h = torch.tanh(h)
        return h[..., 0]

    return f


@pytest.mark.parametrize("route", ROUTES)
def test_second_order_operators_vs_autograd_hessian(route):
    D = 4
    Ws, bs = random_params([D, 12, 12, 9, 1], 21, scale=1.5)
    net = O.Net(Ws, bs, "tanh")
    X = _pts(3, D, seed=22)
    f = _torch_f(Ws, bs)
    Hs = np.stack([torch.autograd.functional.hessian(f, torch.tensor(x)).numpy() for x in X])
    sig = np.random.default_rng(23).standard_normal((D, 6))
    V = np.random.default_rng(24).standard_normal((3, 5, 6))
    U = V @ sig.T  # u_{n,s} = sigma v_{n,s}
    op_l, fval, _ = O.laplacian(net, X, route)
    np.testing.assert_allclose(fval, f(torch.tensor(X)).numpy(), rtol=1e-14)
    np.testing.assert_allclose(op_l, np.trace(Hs, axis1=1, axis2=2), rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(O.weighted_laplacian(net, X, sig, route)[0],
                               np.einsum("nab,ab->n", Hs, sig @ sig.T), rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(O.randomized_laplacian(net, X, V, sig, route)[0],
                               np.einsum("nab,nsa,nsb->n", Hs, U, U) / 5, rtol=1e-11, atol=1e-13)


@pytest.mark.parametrize("route", ROUTES)
def test_biharmonic_vs_nested_autograd_laplacian(route):
    D = 3
    Ws, bs = random_params([D, 10, 8, 1], 31, scale=1.5)
    net = O.Net(Ws, bs, "tanh")
    X = _pts(2, D, seed=32)
    f = _torch_f(Ws, bs)

    def lap(g, x):
        x = x.requires_grad_(True) if not x.requires_grad else x
        (gr,) = torch.autograd.grad(g(x), x, create_graph=True)
        return sum(torch.autograd.grad(gr[i], x, create_graph=True)[0][i] for i in range(D))

    want = []
    for x in X:
        xt = torch.tensor(x, requires_grad=True)
        want.append(lap(lambda y: lap(f, y), xt).item())
    np.testing.assert_allclose(O.biharmonic(net, X, route)[0], want, rtol=1e-10)


# --------------------------------------------------------------------------
# Finite differences of f along a direction (pins O1's per-direction jets)
# --------------------------------------------------------------------------
def test_second_directional_derivative_fd():
    D = 5
    Ws, bs = random_params([D, 16, 16, 1], 41, scale=1.5)
    net = O.Net(Ws, bs, "tanh")
    x = _pts(1, D, seed=42)[0]
    v = np.random.default_rng(43).standard_normal(D)

    def g(h):
        F = O.forward(net, np.stack([x + h * v, x, x - h * v]))
        return (F[0] - 2 * F[1] + F[2]) / h**2

    fd = (4 * g(5e-4) - g(1e-3)) / 3
    got, _, norm = O.weighted_laplacian(net, x[None], v[:, None], O.O1)
    assert abs(got[0] - fd) < 1e-7 * max(1.0, abs(norm[0]))


def test_fourth_derivative_fd_1d():
    # D = 1: the biharmonic family is the single jet (4 e_1), so op = f''''(x)
    Ws, bs = random_params([1, 16, 16, 1], 51, scale=2.0)
    net = O.Net(Ws, bs, "tanh")
    x = 0.3

    def g(h):
        F = O.forward(net, np.array([[x + 2 * h], [x + h], [x], [x - h], [x - 2 * h]]))
        return (F[0] - 4 * F[1] + 6 * F[2] - 4 * F[3] + F[4]) / h**4

    fd = (4 * g(5e-3) - g(1e-2)) / 3
    for route in ROUTES:
        got = O.biharmonic(net, np.array([[x]]), route)[0][0]
        assert abs(got - fd) < 1e-5 * max(1.0, abs(got)), route


# --------------------------------------------------------------------------
# Invariants between routes (Eq. 7: collapsed == vanilla-then-summed)
# --------------------------------------------------------------------------
def _mid_net(D, seed):
    Ws, bs = random_params([D, 24, 20, 16, 1], seed, scale=1.5)
    return O.Net(Ws, bs, "tanh")


def test_routes_agree_second_order():
    D = 6
    net = _mid_net(D, 61)
    X = _pts(4, D, seed=62)
    sig = np.random.default_rng(63).standard_normal((D, 9))
    V = np.sign(np.random.default_rng(64).standard_normal((4, 7, 9)))
    for fn, args in ((O.laplacian, ()), (O.weighted_laplacian, (sig,)), (O.randomized_laplacian, (V, sig))):
        o1, f1, norm = fn(net, X, *args, route=O.O1)
        o2, f2, _ = fn(net, X, *args, route=O.O2)
        o3, f3, _ = fn(net, X, *args, route=O.O3)
        assert rel_err(o3, o1, norm) < 1e-12
        assert rel_err(o2, o1, norm) < 1e-11
        np.testing.assert_array_equal(f1, f3)


def test_routes_agree_biharmonic():
    D = 4
    net = _mid_net(D, 71)
    X = _pts(3, D, seed=72)
    o1, _, norm = O.biharmonic(net, X, O.O1)
    o2 = O.biharmonic(net, X, O.O2)[0]
    o3 = O.biharmonic(net, X, O.O3)[0]
    assert rel_err(o3, o1, norm) < 1e-12
    assert rel_err(o2, o1, norm) < 1e-11


def test_weighted_identity_equals_laplacian():
    D = 6
    net = _mid_net(D, 81)
    X = _pts(3, D, seed=82)
    for route in ROUTES:
        a = O.laplacian(net, X, route)[0]
        b = O.weighted_laplacian(net, X, np.eye(D), route)[0]
        np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-14)


def test_randomized_exact_designs_reproduce_laplacian():
    # (i) Sylvester-Hadamard: rows of H64[:, :50] are legal Rademacher draws with
    #     sum_s v_s v_s^T = 64 I, so the estimator is exact (D = 50)
    D = 50
    Ws, bs = random_params([D, 32, 24, 1], 91, scale=1.5)
    net = O.Net(Ws, bs, "tanh")
    X = _pts(2, D, seed=92)
    H = sylvester_hadamard(64)[:, :D]
    V = np.broadcast_to(H, (2, 64, D)).copy()
    exact, _, norm = O.laplacian(net, X, O.O1)
    for route in (O.O1, O.O3):
        est = O.randomized_laplacian(net, X, V, route=route)[0]
        assert rel_err(est, exact, norm) < 1e-12
    # (ii) all 2^D sign vectors (D = 4)
    D = 4
    net4 = _mid_net(D, 93)
    X4 = _pts(3, D, seed=94)
    signs = np.array([[1.0 if (m >> d) & 1 else -1.0 for d in range(D)] for m in range(2**D)])
    V4 = np.broadcast_to(signs, (3, 2**D, D)).copy()
    e4, _, n4 = O.laplacian(net4, X4, O.O1)
    for route in ROUTES:
        assert rel_err(O.randomized_laplacian(net4, X4, V4, route=route)[0], e4, n4) < 1e-12


def test_rademacher_estimator_unbiased_and_variance():
    D = 4
    net = _mid_net(D, 101)
    x = _pts(1, D, seed=102)
    f = _torch_f(net.Ws, net.bs)
    H = torch.autograd.functional.hessian(f, torch.tensor(x[0])).numpy()
    T = 4000
    V = np.concatenate([O.rademacher(seed, 0, 1, 1, D) for seed in range(T)], axis=0)  # [T, 1, D]
    X = np.repeat(x, T, axis=0)
    est = O.randomized_laplacian(net, X, V, route=O.O3)[0]
    exact = np.trace(H)
    var_theory = 2 * (np.sum(H**2) - np.sum(np.diag(H) ** 2))  # S = 1
    se = math.sqrt(var_theory / T)
    assert abs(est.mean() - exact) < 4 * se
    assert abs(est.var() / var_theory - 1) < 0.15


# --------------------------------------------------------------------------
# Stochastic biharmonic (Eq. 12 stochastic case, unbiased 1/(3S) scale: reading Q1)
# --------------------------------------------------------------------------
def test_stochastic_biharmonic_routes_agree():
    D = 4
    net = _mid_net(D, 111)
    X = _pts(3, D, seed=112)
    V = np.random.default_rng(113).standard_normal((3, 5, D))
    o1, _, norm = O.stochastic_biharmonic(net, X, V, O.O1)
    assert rel_err(O.stochastic_biharmonic(net, X, V, O.O3)[0], o1, norm) < 1e-12
    assert rel_err(O.stochastic_biharmonic(net, X, V, O.O2)[0], o1, norm) < 1e-11


@pytest.mark.parametrize("route", ROUTES)
def test_stochastic_biharmonic_norm4_closed_form(route):
    # f = ||x||^4: d^4/dt^4 ||x + t v||^4 = 24 ||v||^4, so the estimator is 8/S sum_s ||v_s||^4
    D = 3
    net = _norm4_net(D)
    X = _pts(2, D)
    V = np.random.default_rng(121).standard_normal((2, 6, D))
    want = 8.0 / 6 * np.sum(np.sum(V**2, axis=2) ** 2, axis=1)
    np.testing.assert_allclose(O.stochastic_biharmonic(net, X, V, route)[0], want, rtol=1e-12)


def test_stochastic_biharmonic_unbiased_for_gaussian():
    # E <d^4 f, v^4> = 3 Laplacian^2 f for v ~ N(0, I) (Isserlis); mean within 4 SE
    D = 3
    net = _mid_net(D, 131)
    x = _pts(1, D, seed=132)
    exact = O.biharmonic(net, x, O.O2)[0][0]
    T = 20000
    V = np.random.default_rng(133).standard_normal((T, 1, D))
    est = O.stochastic_biharmonic(net, np.repeat(x, T, axis=0), V, O.O3)[0]
    assert abs(est.mean() - exact) < 4 * est.std() / math.sqrt(T)


# --------------------------------------------------------------------------
# Nested collapsed Laplacians: Laplacian(Laplacian f)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("D", [1, 2, 3, 5])
def test_nested_biharmonic_norm4_and_x1sq_x2sq(D):
    net = _norm4_net(D)
    X = _pts(3, D)
    op, f, lap = O.biharmonic_nested(net, X)
    r2 = np.sum(X**2, axis=1)
    np.testing.assert_allclose(op, 8 * D * (D + 2), rtol=1e-12)
    np.testing.assert_allclose(lap, 4 * (D + 2) * r2, rtol=1e-13)
    np.testing.assert_allclose(f, r2**2, rtol=1e-14)
    W1 = np.array([[1.0, 1.0], [1.0, -1.0], [1.0, 0.0], [0.0, 1.0]])
    net = O.Net([W1, np.eye(4), np.array([[1.0, 1.0, -2.0, -2.0]]) / 12.0],
                [np.zeros(4), np.zeros(4), np.zeros(1)], "square")
    np.testing.assert_allclose(O.biharmonic_nested(net, _pts(4, 2))[0], 8.0, rtol=1e-12)


def test_nested_biharmonic_sum_of_sines_and_linear_net():
    rng = np.random.default_rng(9)
    D = 4
    bvec, phi, a = rng.uniform(0.5, 2, D), rng.uniform(-1, 1, D), rng.uniform(-1, 1, D)
    net = O.Net([np.diag(bvec), a[None, :]], [phi, np.array([0.3])], "sin")
    X = _pts(5, D)
    s = np.sin(X * bvec + phi)
    op, _, lap = O.biharmonic_nested(net, X)
    np.testing.assert_allclose(op, (s * a * bvec**4).sum(1), rtol=1e-11)
    np.testing.assert_allclose(lap, -(s * a * bvec**2).sum(1), rtol=1e-12)
    Ws, bs = random_params([4, 7, 5, 1], 1)
    assert np.max(np.abs(O.biharmonic_nested(O.Net(Ws, bs, "identity"), X)[0])) < 1e-13


def test_nested_biharmonic_one_hidden_layer_tanh_closed_form():
    D, H = 5, 7
    Ws, bs = random_params([D, H, 1], 11, scale=2.0)
    X = _pts(4, D)
    W1, c = Ws[0], Ws[1][0]
    t4 = _tanh_derivs_autograd(X @ W1.T + bs[0], 4)
    np.testing.assert_allclose(O.biharmonic_nested(O.Net(Ws, bs), X)[0], (t4 * c * np.sum(W1**2, 1) ** 2).sum(1),
                               rtol=1e-11)


def test_nested_biharmonic_vs_tensor_route_interpolation_and_autograd():
    """Three independent derivations of the same number: the explicit 4th-derivative
    tensor (O2), the interpolation family (O1), and torch's nested autograd Laplacian."""
    for D, seed in ((3, 31), (5, 7), (1, 51)):
        Ws, bs = random_params([D, 10, 8, 6, 1], seed, scale=1.5)
        net = O.Net(Ws, bs, "tanh")
        X = _pts(3, D, seed=seed + 1)
        op, f, lap = O.biharmonic_nested(net, X)
        want, _, norm = O.biharmonic(net, X, O.O1)
        assert np.max(np.abs(op - want) / norm) < 1e-12
        if D <= 3:
            np.testing.assert_allclose(op, O.biharmonic(net, X, O.O2)[0], rtol=1e-11)
        np.testing.assert_allclose(lap, O.laplacian(net, X)[0], rtol=1e-12)
        np.testing.assert_allclose(f, O.forward(net, X), rtol=1e-14)
    D = 3
    Ws, bs = random_params([D, 10, 8, 1], 31, scale=1.5)
    tf = _torch_f(Ws, bs)
    x = torch.tensor(_pts(1, D, seed=32)[0], requires_grad=True)

    def lap(g, y):
        (gr,) = torch.autograd.grad(g(y), y, create_graph=True)
        return sum(torch.autograd.grad(gr[i], y, create_graph=True)[0][i] for i in range(D))

    want = lap(lambda y: lap(tf, y), x).item()
    got = O.biharmonic_nested(O.Net(Ws, bs), x.detach().numpy()[None])[0][0]
    assert abs(got - want) < 1e-10 * max(1.0, abs(want))


# --------------------------------------------------------------------------
# Weighted directional sums (Eq. 5 with weights; Eq. 13-15 general approach)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("K", [2, 4])
@pytest.mark.parametrize("per_point", [False, True])
def test_directional_sum_routes_agree(K, per_point):
    D, J, N = 3, 5, 4
    net = _mid_net(D, 61)
    rng = np.random.default_rng(62)
    X = _pts(N, D, seed=63)
    dirs = rng.standard_normal((N, J, D) if per_point else (J, D))
    w = rng.uniform(-1, 1, J)
    w[1] = w[0]  # a group of two equal weights for the collapsed route
    o1, f1, norm = O.directional_sum(net, X, K, dirs, w, O.O1)
    o2, f2, _ = O.directional_sum(net, X, K, dirs, w, O.O2)
    o3, _, _ = O.directional_sum(net, X, K, dirs, w, O.O3)
    assert np.max(np.abs(o1 - o3) / norm) < 1e-12
    assert np.max(np.abs(o1 - o2) / norm) < 1e-11
    np.testing.assert_allclose(f1, O.forward(net, X), rtol=1e-14)


def test_directional_sum_reduces_to_the_named_operators():
    D = 4
    net = _mid_net(D, 64)
    X = _pts(3, D, seed=65)
    np.testing.assert_allclose(O.directional_sum(net, X, 2, np.eye(D), np.ones(D))[0], O.laplacian(net, X)[0],
                               rtol=1e-13)
    dirs, coef = O.biharmonic_set(D)
    np.testing.assert_allclose(O.directional_sum(net, X, 4, dirs, coef)[0], O.biharmonic(net, X)[0], rtol=1e-12)
    sig = np.random.default_rng(66).standard_normal((D, 3))
    sx = np.broadcast_to(sig, (3, D, 3))
    np.testing.assert_allclose(O.weighted_laplacian_pointwise(net, X, sx)[0], O.weighted_laplacian(net, X, sig)[0],
                               rtol=1e-13)


def test_directional_sum_closed_forms():
    # quadratic net: <d^2 f, u^2> = u^T H u;  ||x||^4: <d^4 f, u^4> = 24 |u|^4
    D, H = 5, 6
    Ws, bs = random_params([D, H, 1], 3, scale=2.0)
    net = O.Net(Ws, bs, "square")
    Hess = 2 * (Ws[0].T * Ws[1][0]) @ Ws[0]
    rng = np.random.default_rng(67)
    X = _pts(4, D)
    dirs, w = rng.standard_normal((3, D)), np.array([0.5, -2.0, 1.25])
    np.testing.assert_allclose(O.directional_sum(net, X, 2, dirs, w)[0], np.einsum("j,ja,ab,jb->", w, dirs, Hess, dirs),
                               rtol=1e-12)
    sx = rng.standard_normal((4, D, 2))  # sigma(x_n): a different sigma per point
    np.testing.assert_allclose(O.weighted_laplacian_pointwise(net, X, sx)[0],
                               np.einsum("ab,nar,nbr->n", Hess, sx, sx), rtol=1e-12)
    net4 = _norm4_net(D)
    np.testing.assert_allclose(O.directional_sum(net4, X, 4, dirs, w)[0], 24 * np.sum(w * np.sum(dirs**2, 1) ** 2),
                               rtol=1e-12)


@pytest.mark.parametrize("i", [(3, 1), (2, 2)])
def test_interpolation_family_eq15_recovers_mixed_partials(i):
    """Eq. 15 with I = 2, v_1 = e_1, v_2 = e_2: the family j in N^2, |j| = 4, directions
    j_1 e_1 + j_2 e_2, weights gamma_{i,j} / 4!, gives d_1^{i_1} d_2^{i_2} f, checked against
    torch fp64 autograd on a tanh net (gamma pinned by Fig. 3 separately)."""
    D = 2
    Ws, bs = random_params([D, 9, 7, 1], 71, scale=1.5)
    net = O.Net(Ws, bs, "tanh")
    x = _pts(1, D, seed=72)[0]
    fam = [(j1, 4 - j1) for j1 in range(5)]
    dirs = np.array([[j1, j2] for j1, j2 in fam], dtype=float)
    w = np.array([float(O.gamma(i, j)) / 24.0 for j in fam])
    got = O.directional_sum(net, x[None], 4, dirs, w)[0][0]
    tf = _torch_f(Ws, bs)
    xt = torch.tensor(x, requires_grad=True)
    g = tf(xt)
    for ax in [0] * i[0] + [1] * i[1]:
        (gr,) = torch.autograd.grad(g, xt, create_graph=True)
        g = gr[ax]
    assert abs(got - g.item()) < 1e-10 * max(1.0, abs(g.item()))


def test_direction_blocks_are_exact_in_the_collapsed_route():
    """The GPU's direction blocks rest on Eq. 7 being linear in the collapsed
    top: propagating a direction set in blocks, each with its own primal and partial top,
    and adding the block results gives the collapsed result of the whole set. Checked on
    the oracle's collapsed route O3 (K = 2 and K = 4, uneven blocks), against O1."""
    rng = np.random.default_rng(11)
    Ws, bs = random_params([6, 20, 16, 1], 3)
    net = O.Net(Ws, bs)
    X = rng.uniform(-1, 1, size=(5, 6))
    for K, J in ((2, 23), (4, 17)):
        dirs = rng.standard_normal((J, 6))
        w = rng.uniform(-1, 1, size=J)
        whole, _, norm = O.directional_sum(net, X, K, dirs, w, O.O1)
        cuts = [0, 7, 8, 15, J]
        parts = sum(O.directional_sum(net, X, K, dirs[a:b], w[a:b], O.O3)[0] for a, b in zip(cuts, cuts[1:]))
        assert np.max(np.abs(parts - whole) / norm) < 1e-12


def test_spec_worked_examples():
    """The worked examples SPEC.md prints (tests/golden/spec_worked_examples.txt, cited per row)."""
    want = {r[0]: float(r[1]) for r in golden("spec_worked_examples.txt")}
    I = np.eye
    for x0, name in ((np.pi / 4, "appC_sin_2jet_x0_pi4"), (0.0, "appC_sin_2jet_x0_0")):
        net = O.Net([I(1), I(1)], [np.zeros(1), np.zeros(1)], "sin")  # f = sin(x), D = 1
        for route in ROUTES:
            got = O.directional_sum(net, np.array([[x0]]), 2, np.array([[1.0], [2.0]]), np.ones(2), route=route)[0]
            np.testing.assert_allclose(got, want[name], rtol=1e-14, atol=1e-15)
    half = lambda D: O.Net([I(D), np.full((1, D), 0.5)], [np.zeros(D), np.zeros(1)], "square")  # 1/2 ||x||^2
    X7 = _pts(3, 7)
    for route in ROUTES:
        np.testing.assert_allclose(O.laplacian(half(7), X7, route)[0], want["half_norm2_D7_laplacian"], rtol=1e-13)
        sig = np.zeros((4, 1))
        sig[0, 0] = 2.0
        np.testing.assert_allclose(O.weighted_laplacian(half(4), _pts(3, 4), sig, route)[0],
                                   want["weighted_diag2_half_norm2"], rtol=1e-13)
        norm4 = O.Net([I(2), np.ones((1, 2)), np.ones((1, 1))], [np.zeros(2), np.zeros(1), np.zeros(1)], "square")
        np.testing.assert_allclose(O.biharmonic(norm4, _pts(3, 2), route)[0], want["norm4_D2_biharmonic"], rtol=1e-12)
        x1p4 = O.Net([np.array([[1.0, 0, 0]]), np.ones((1, 1)), np.ones((1, 1))], [np.zeros(1)] * 3, "square")
        np.testing.assert_allclose(O.biharmonic(x1p4, _pts(3, 3), route)[0], want["x1pow4_D3_biharmonic"], rtol=1e-12)
