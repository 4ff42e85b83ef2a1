"""GPU parity of fp16x3 training ("fp16x3 training"): in the fp16x3 mode the
differentiable path of the fixed-direction K=2 operators runs every contraction -- forward
layers, adjoint layers (jet_layer_kernel<kBwd2>) and weight gradients (wgrad_kernel) -- on
two power-of-two-scaled fp16 planes per operand, with ONE scale per slot block (the weight
gradients contract over all slot rows). Compared with the fp64 reverse-mode oracle
(oracle/grad.py) at the bars of reading R10, the same as the fp32 mode's tests."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import (gaussian_directions, mlp_params, points, sigma as make_sigma, sigma_field, signed_weights,
                   widths_for)
from tests.test_gpu_grad import GTOL, _check_grads, _gs, _k2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctm():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2505_13644_b200 as ctm

    ctm.lib()
    return ctm


def _mlp(ctm, params, act="tanh"):
    m = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0, act=act,
                precision="fp16x3")
    m.grad_enable()
    return m


def _np64(params):
    return [W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params]


def test_fp16x3_training_covers_the_k2_operators(ctm):
    """Grad mode in the fp16x3 mode: the exact / weighted Laplacians, K=2 directional sums and
    the per-point directions (randomized with or without sigma, sigma(x)) run fp16x3."""
    params = mlp_params([5, 64, 48, 1], 0)
    X = torch.from_numpy(points(9, 5)).cuda()
    m = _mlp(ctm, params)
    m.laplacian(X)
    assert m.last_precision() == "fp16x3"
    m.weighted_laplacian(X, torch.from_numpy(make_sigma(5, 3, kind="rect")).cuda())
    assert m.last_precision() == "fp16x3"
    m.randomized_laplacian(X, S=4, seed=1)
    assert m.last_precision() == "fp16x3"
    m.randomized_laplacian(X, S=4, seed=1, sigma=torch.from_numpy(make_sigma(5, 5)).cuda())
    assert m.last_precision() == "fp16x3"
    m.close()


def test_fp16x3_per_point_direction_gradients(ctm):
    """Per-point directions in grad mode (layer 1 on the tensor cores, B_0 = [x0; u; 0] with
    one scale): randomized Rademacher / Gaussian (generated in-kernel), sigma(x), per-point
    K=2 directional sums -- against the fp64 reverse-mode oracle."""
    widths = [5, 48, 40, 1]
    params = mlp_params(widths, 0)
    Ws, bs = _np64(params)
    D, N = 5, 11
    X = points(N, D)
    Xc = torch.from_numpy(X).cuda()
    Xd = X.astype(np.float64)
    gop, gf = _gs(N)
    g_op, g_f = torch.from_numpy(gop).cuda(), torch.from_numpy(gf).cuda()
    m = _mlp(ctm, params)
    m.randomized_laplacian(Xc, S=6, seed=3)
    assert m.last_precision() == "fp16x3"
    V = O.rademacher(3, 0, N, 6, D)
    dW, db, mag = _k2(Ws, bs, Xd, V, np.full(6, 1 / 6), gop, gf)
    _check_grads("fp16x3_randomized", m.backward(g_op, g_f), dW, db, mag)
    Vg = gaussian_directions(N, 5, D, seed=4)
    m.randomized_laplacian(Xc, V=torch.from_numpy(Vg).cuda(), dist="gaussian")
    dW, db, mag = _k2(Ws, bs, Xd, Vg.astype(np.float64), np.full(5, 1 / 5), gop, gf)
    _check_grads("fp16x3_randomized_gaussian_V", m.backward(g_op, g_f), dW, db, mag)
    sx = sigma_field(X, 4)
    m.weighted_laplacian_pointwise(Xc, torch.from_numpy(sx).cuda())
    assert m.last_precision() == "fp16x3"
    dW, db, mag = _k2(Ws, bs, Xd, np.transpose(sx.astype(np.float64), (0, 2, 1)), np.ones(4), gop, gf)
    _check_grads("fp16x3_pointwise", m.backward(g_op, g_f), dW, db, mag)
    w = signed_weights(4)
    dirs = gaussian_directions(N, 4, D, seed=8)
    m.directional_sum(Xc, 2, torch.from_numpy(dirs).cuda(), torch.from_numpy(w).cuda())
    assert m.last_precision() == "fp16x3"
    dW, db, mag = _k2(Ws, bs, Xd, dirs.astype(np.float64), w.astype(np.float64), gop, gf)
    _check_grads("fp16x3_directional_per_point", m.backward(g_op, g_f), dW, db, mag)
    m.close()


@pytest.mark.parametrize("act", ["tanh", "sin"])
@pytest.mark.parametrize("widths,N", [([3, 16, 12, 1], 9), ([5, 64, 48, 1], 33), ([4, 40, 48, 36, 1], 7),
                                      ([3, 300, 130, 260, 1], 5), (widths_for(50), 6)])
def test_fp16x3_laplacian_gradients(ctm, widths, N, act):
    params = mlp_params(widths, 0)
    D = widths[0]
    X = points(N, D)
    gop, gf = _gs(N)
    m = _mlp(ctm, params, act=act)
    m.laplacian(torch.from_numpy(X).cuda())
    assert m.last_precision() == "fp16x3"
    grads = m.backward(torch.from_numpy(gop).cuda(), torch.from_numpy(gf).cuda())
    Ws, bs = _np64(params)
    dW, db, mag = _k2(Ws, bs, X.astype(np.float64), np.eye(D), np.ones(D), gop, gf, act=act)
    _check_grads(f"fp16x3_laplacian{widths}_{act}", grads, dW, db, mag)
    m.close()


def test_fp16x3_weighted_and_directional_gradients(ctm):
    widths = [5, 48, 40, 1]
    params = mlp_params(widths, 0)
    Ws, bs = _np64(params)
    D, N = 5, 11
    X = points(N, D)
    Xc = torch.from_numpy(X).cuda()
    Xd = X.astype(np.float64)
    gop, gf = _gs(N)
    g_op, g_f = torch.from_numpy(gop).cuda(), torch.from_numpy(gf).cuda()
    m = _mlp(ctm, params)
    for kind, R in (("rect", 3), ("dense", 5)):
        sig = make_sigma(D, R, kind=kind)
        m.weighted_laplacian(Xc, torch.from_numpy(sig).cuda())
        assert m.last_precision() == "fp16x3"
        dW, db, mag = _k2(Ws, bs, Xd, sig.astype(np.float64).T, np.ones(R), gop, gf)
        _check_grads(f"fp16x3_weighted_{kind}", m.backward(g_op, g_f), dW, db, mag)
    w = signed_weights(4)
    dirs = gaussian_directions(1, 4, D, seed=8)[0]
    m.directional_sum(Xc, 2, torch.from_numpy(dirs).cuda(), torch.from_numpy(w).cuda())
    assert m.last_precision() == "fp16x3"
    dW, db, mag = _k2(Ws, bs, Xd, dirs.astype(np.float64), w.astype(np.float64), gop, gf)
    _check_grads("fp16x3_directional", m.backward(g_op, g_f), dW, db, mag)
    # only gop (gf = None): the f-adjoint bound is zero
    m.laplacian(Xc)
    dW, db, mag = _k2(Ws, bs, Xd, np.eye(D), np.ones(D), gop, np.zeros(N, np.float32))
    _check_grads("fp16x3_gop_only", m.backward(g_op), dW, db, mag)
    m.close()


@pytest.mark.parametrize("scale", [1e-3, 10.0])
def test_fp16x3_gradients_far_from_unit_scale(ctm, scale):
    """Inputs scaled by 1e-3 (tiny first-order and top values) or 10 (saturated tanh units):
    the block scales follow the bounds, no plane overflows, the gradients meet the bars.
    (At x * 30 the fp32 mode itself misses the per-element bar, 5.5e-3 at a unit whose M_i is
    3.9e-6 of the tensor's largest -- cancellation upstream of the final contraction, reading
    R10 -- and fp16x3 gives the same error to four digits: scripts/diag_grad_scale.py.)"""
    widths = [5, 64, 48, 1]
    params = mlp_params(widths, 0)
    N = 13
    X = points(N, 5) * scale
    gop, gf = _gs(N)
    m = _mlp(ctm, params)
    m.laplacian(torch.from_numpy(X).cuda())
    grads = m.backward(torch.from_numpy(gop).cuda(), torch.from_numpy(gf).cuda())
    Ws, bs = _np64(params)
    dW, db, mag = _k2(Ws, bs, X.astype(np.float64), np.eye(5), np.ones(5), gop, gf)
    _check_grads(f"fp16x3_scale{scale}", grads, dW, db, mag)
    m.close()


def test_fp16x3_backward_is_deterministic(ctm):
    params = mlp_params([5, 64, 48, 1], 0)
    X = torch.from_numpy(points(33, 5)).cuda()
    gop, gf = (torch.from_numpy(t).cuda() for t in _gs(33))
    m = _mlp(ctm, params)
    m.laplacian(X)
    a = m.backward(gop, gf)
    m.laplacian(X)
    b = m.backward(gop, gf)
    for (aw, ab), (bw, bb) in zip(a, b):
        assert torch.equal(aw, bw) and torch.equal(ab, bb)
    m.close()


def test_fp16x3_full_size_gradient_is_the_sum_of_its_shards(ctm):
    """C1 at N = 16384 (the training bench's batch) in the fp16x3 mode: the gradient of the
    batch equals the accumulated gradients of four quarter batches (each quarter has its
    own block scales; fp32 order of the 852k-row reductions: GTOL)."""
    params = mlp_params(widths_for(50), 0)
    N = 16384
    X = torch.from_numpy(points(N, 50)).cuda()
    gop, gf = (torch.from_numpy(t).cuda() / N for t in _gs(N))
    m = _mlp(ctm, params)
    m.laplacian(X)
    assert m.last_precision() == "fp16x3"
    full = m.backward(gop, gf)
    acc = None
    for q in range(4):
        sl = slice(q * N // 4, (q + 1) * N // 4)
        m.laplacian(X[sl])
        acc = m.backward(gop[sl], gf[sl], grads=acc, accumulate=acc is not None)
    for (fw, fb), (aw, ab) in zip(full, acc):
        for a, b in ((fw, aw), (fb, ab)):
            scale = max(a.abs().max().item(), 1e-30)
            assert (a - b).abs().max().item() / scale < GTOL
    m.close()
