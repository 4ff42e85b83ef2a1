"""GPU parity of the differentiable path (NEXT-3): ctm_backward vs the fp64 reverse-mode
oracle (oracle/grad.py) on identical seeded inputs.

Metric (reading R10): per parameter tensor,
    max_i |g_gpu,i - g_oracle,i| / max_i |g_oracle,i|  <= GTOL
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
from oracle import grad as OG
from synth import gaussian_directions, mlp_params, points, sigma as make_sigma, sigma_field, signed_weights, widths_for

pytestmark = pytest.mark.gpu

GTOL = 1e-4
ERRS = {}


@pytest.fixture(scope="module")
def ctm():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2505_13644_b200 as ctm

    ctm.lib()
    return ctm


@pytest.fixture(scope="module", autouse=True)
def _dump():
    yield
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if ERRS and os.path.isdir(out):
        with open(os.path.join(out, "grad_errors.json"), "w") as fh:
            json.dump(ERRS, fh, indent=1, sort_keys=True)


def _mlp(ctm, params, act="tanh"):
    m = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0, act=act)
    m.grad_enable()
    return m


def _k2(*a, **k):
    """fp64 oracle gradients and their per-element magnitudes (oracle/grad.py)."""
    _, _, dW, db = OG.k2_grad(*a, **k)
    return dW, db, OG.k2_grad_magnitude(*a, **k)


ETOL = 1e-3  # per-element bar (R10): M covers only the final contraction, not cancellation upstream


def _check_grads(name, grads, dW, db, mag, tol=GTOL, etol=ETOL):
    """Two bars (reading R10): per tensor, max|g - r| <= tol * max|r|; and per ELEMENT,
    |g_i - r_i| <= etol * M_i (+ 1e-12 * max M for elements whose terms are all zero), M the
    sum of the absolute terms of the element's final contraction (k2_grad_magnitude), which
    also checks the small elements. M does not see cancellation inside the adjoints z_bar
    upstream of that contraction, so its bar is 1e-3: a 60-case soak found an element at
    2.6e-4 of M in fp32 arithmetic."""
    rec = {}
    MW, Mb = mag
    for l, ((gW, gb), rW, rb, mW, mb) in enumerate(zip(grads, dW, db, MW, Mb)):
        for tag, g, r, m in (("W", gW, rW, mW), ("b", gb, rb, mb)):
            g = g.double().cpu().numpy()
            assert np.all(np.isfinite(g))
            scale = np.max(np.abs(r))
            err = np.max(np.abs(g - r)) / scale if scale > 0 else np.max(np.abs(g))
            rec[f"{tag}{l}"] = float(err)
            m = np.asarray(m).reshape(r.shape)
            floor = 1e-12 * max(float(np.max(m)), 1e-30)
            rel = np.abs(g - r) / np.maximum(m, floor)
            rec[f"{tag}{l}_elem"] = float(np.max(rel))
    ERRS[name] = rec
    worst = max(v for k, v in rec.items() if not k.endswith("_elem"))
    worst_elem = max(v for k, v in rec.items() if k.endswith("_elem"))
    assert worst <= tol and worst_elem <= etol, f"{name}: {rec}"


def _gs(N, seed=7):
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal(N).astype(np.float32), rng.standard_normal(N).astype(np.float32)


@pytest.mark.parametrize("widths,N", [([3, 16, 12, 1], 9), ([5, 16, 16, 1], 16), ([4, 40, 48, 36, 1], 7),
                                      ([6, 24, 1], 5), (widths_for(50), 6)])
def test_laplacian_gradients(ctm, widths, N):
    params = mlp_params(widths, 0)
    D = widths[0]
    X = points(N, D)
    gop, gf = _gs(N)
    mlp = _mlp(ctm, params)
    op, f = mlp.laplacian(torch.from_numpy(X).cuda())
    grads = mlp.backward(torch.from_numpy(gop).cuda(), torch.from_numpy(gf).cuda())
    Ws = [W.astype(np.float64) for W, _ in params]
    bs = [b.astype(np.float64) for _, b in params]
    dW, db, mag = _k2(Ws, bs, X.astype(np.float64), np.eye(D), np.ones(D), gop, gf)
    _check_grads(f"laplacian{widths}", grads, dW, db, mag)


def test_weighted_randomized_pointwise_and_directional_gradients(ctm):
    widths = [5, 48, 40, 1]
    params = mlp_params(widths, 0)
    Ws = [W.astype(np.float64) for W, _ in params]
    bs = [b.astype(np.float64) for _, b in params]
    D, N = 5, 11
    X = points(N, D)
    Xc = torch.from_numpy(X).cuda()
    Xd = X.astype(np.float64)
    gop, gf = _gs(N)
    g_op, g_f = torch.from_numpy(gop).cuda(), torch.from_numpy(gf).cuda()
    mlp = _mlp(ctm, params)
    # weighted (sigma rect R = 3)
    sig = make_sigma(D, 3, kind="rect")
    mlp.weighted_laplacian(Xc, torch.from_numpy(sig).cuda())
    dW, db, mag = _k2(Ws, bs, Xd, sig.astype(np.float64).T, np.ones(3), gop, gf)
    _check_grads("weighted", mlp.backward(g_op, g_f), dW, db, mag)
    # randomized (Rademacher generated in-kernel, S = 6): op carries 1/S
    mlp.randomized_laplacian(Xc, S=6, seed=3)
    V = O.rademacher(3, 0, N, 6, D)
    dW, db, mag = _k2(Ws, bs, Xd, V, np.full(6, 1 / 6), gop, gf)
    _check_grads("randomized", mlp.backward(g_op, g_f), dW, db, mag)
    # sigma(x)
    sx = sigma_field(X, 4)
    mlp.weighted_laplacian_pointwise(Xc, torch.from_numpy(sx).cuda())
    dW, db, mag = _k2(Ws, bs, Xd, np.transpose(sx.astype(np.float64), (0, 2, 1)), np.ones(4), gop, gf)
    _check_grads("pointwise", mlp.backward(g_op, g_f), dW, db, mag)
    # directional sums K = 2 with signed weights, shared and per point
    w = signed_weights(4)
    for per_point in (False, True):
        dirs = gaussian_directions(N, 4, D, seed=8) if per_point else gaussian_directions(1, 4, D, seed=8)[0]
        mlp.directional_sum(Xc, 2, torch.from_numpy(dirs).cuda(), torch.from_numpy(w).cuda())
        dW, db, mag = _k2(Ws, bs, Xd, dirs.astype(np.float64), w.astype(np.float64), gop, gf)
        _check_grads(f"directional_pp{int(per_point)}", mlp.backward(g_op, g_f), dW, db, mag)


@pytest.mark.parametrize("act", ["sin", "exp"])
def test_sin_exp_activation_gradients(ctm, act):
    widths = [4, 32, 24, 1]
    params = mlp_params(widths, 0)
    X = points(8, 4)
    gop, gf = _gs(8)
    mlp = _mlp(ctm, params, act=act)
    mlp.laplacian(torch.from_numpy(X).cuda())
    grads = mlp.backward(torch.from_numpy(gop).cuda(), torch.from_numpy(gf).cuda())
    dW, db, mag = _k2([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params],
                              X.astype(np.float64), np.eye(4), np.ones(4), gop, gf, act=act)
    _check_grads(act, grads, dW, db, mag)


def test_backward_is_deterministic_accumulates_and_needs_a_tape(ctm):
    params = mlp_params([5, 64, 48, 1], 0)
    X = torch.from_numpy(points(33, 5)).cuda()
    gop = torch.from_numpy(_gs(33)[0]).cuda()
    mlp = _mlp(ctm, params)
    mlp.laplacian(X)
    a = mlp.backward(gop)
    b = mlp.backward(gop)
    for (aw, ab), (bw, bb) in zip(a, b):
        assert torch.equal(aw, bw) and torch.equal(ab, bb)
    c = mlp.backward(gop, grads=[(w.clone(), v.clone()) for w, v in a], accumulate=True)
    for (aw, ab), (cw, cb) in zip(a, c):
        torch.testing.assert_close(cw, 2 * aw, rtol=1e-6, atol=0)
    assert torch.all(a[-1][1] == 0)  # gf = None: d/db_L of sum gop op = 0
    mlp.biharmonic(X)  # not differentiable: clears the tape
    with pytest.raises(ctm.CTMError, match="EUNSUPPORTED"):
        mlp.backward(gop)


def test_set_weights_matches_a_fresh_load_bitwise(ctm):
    p0 = mlp_params([5, 64, 48, 1], 0)
    p1 = mlp_params([5, 64, 48, 1], 1)
    X = torch.from_numpy(points(19, 5)).cuda()
    a = _mlp(ctm, p0)
    a.set_weights([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in p1])
    b = _mlp(ctm, p1)
    for name in ("laplacian", "biharmonic", "biharmonic_nested"):
        oa, fa = getattr(a, name)(X)
        ob, fb = getattr(b, name)(X)
        assert torch.equal(oa, ob) and torch.equal(fa, fb), name
    gop = torch.from_numpy(_gs(19)[0]).cuda()
    a.laplacian(X)
    b.laplacian(X)
    for (wa, ba), (wb, bb) in zip(a.backward(gop), b.backward(gop)):
        assert torch.equal(wa, wb) and torch.equal(ba, bb)


def test_sharded_gradients_sum_to_the_full_batch(ctm):
    """Data parallelism on one GPU: the gradient of the full batch equals the sum of the
    two shards' gradients (accumulate=True), randomized directions keyed on point_offset."""
    params = mlp_params([6, 64, 64, 1], 0)
    N = 40
    X = torch.from_numpy(points(N, 6)).cuda()
    gop, gf = (torch.from_numpy(t).cuda() for t in _gs(N))
    mlp = _mlp(ctm, params)
    mlp.randomized_laplacian(X, S=7, seed=5)
    full = mlp.backward(gop, gf)
    mlp.randomized_laplacian(X[:17], S=7, seed=5, point_offset=0)
    acc = mlp.backward(gop[:17], gf[:17])
    mlp.randomized_laplacian(X[17:], S=7, seed=5, point_offset=17)
    acc = mlp.backward(gop[17:], gf[17:], grads=acc, accumulate=True)
    for (fw, fb), (aw, ab) in zip(full, acc):
        scale = max(fw.abs().max().item(), 1e-30)
        assert (fw - aw).abs().max().item() / scale < 1e-5
        scale = max(fb.abs().max().item(), 1e-30)
        assert (fb - ab).abs().max().item() / scale < 1e-5


def test_full_size_gradient_is_the_sum_of_its_shards(ctm):
    """C1 at N = 16384 (the training bench's batch): a property that holds at any size —
    the gradient of the batch equals the accumulated gradients of four quarter batches, up
    to the fp32 order of the 852k-row reductions (~sqrt(K) u = 6e-5 worst case; GTOL)."""
    params = mlp_params(widths_for(50), 0)
    N = 16384
    X = torch.from_numpy(points(N, 50)).cuda()
    gop, gf = (torch.from_numpy(t).cuda() / N for t in _gs(N))
    mlp = _mlp(ctm, params)
    mlp.laplacian(X)
    full = mlp.backward(gop, gf)
    acc = None
    for q in range(4):
        sl = slice(q * N // 4, (q + 1) * N // 4)
        mlp.laplacian(X[sl])
        acc = mlp.backward(gop[sl], gf[sl], grads=acc, accumulate=acc is not None)
    for (fw, fb), (aw, ab) in zip(full, acc):
        for a, b in ((fw, aw), (fb, ab)):
            scale = max(a.abs().max().item(), 1e-30)
            assert (a - b).abs().max().item() / scale < GTOL


@pytest.mark.parametrize("case", range(int(os.environ.get("CTM_FUZZ_GRAD", "16"))))
def test_fuzz_shapes_gradients(ctm, case):
    """Random nets, batch sizes and direction sets through the differentiable path: the
    exact, weighted and randomized Laplacians and a signed directional sum, each forward in
    grad mode then ctm_backward, against the fp64 reverse-mode oracle."""
    rng = np.random.default_rng(2000 + case)
    D = int(rng.integers(1, 33))
    hidden = [int(rng.integers(8, 300)) for _ in range(int(rng.integers(1, 4)))]
    widths = [D] + hidden + [1]
    N = int(rng.integers(1, 25))
    params = mlp_params(widths, case)
    X = points(N, D, seed=case)
    Xc = torch.from_numpy(X).cuda()
    Xd = X.astype(np.float64)
    Ws = [W.astype(np.float64) for W, _ in params]
    bs = [b.astype(np.float64) for _, b in params]
    gop, gf = _gs(N, seed=case)
    go, gfc = torch.from_numpy(gop).cuda(), torch.from_numpy(gf).cuda()
    mlp = _mlp(ctm, params)
    which = ["lap", "wlap", "rlap", "dsum"][case % 4]
    if which == "lap":
        mlp.laplacian(Xc)
        dirs, w = np.eye(D), np.ones(D)
    elif which == "wlap":
        R = int(rng.integers(1, 90))
        sig = make_sigma(D, R, kind="rect")
        mlp.weighted_laplacian(Xc, torch.from_numpy(sig).cuda())
        dirs, w = sig.astype(np.float64).T, np.ones(R)
    elif which == "rlap":
        S = int(rng.integers(1, 90))
        mlp.randomized_laplacian(Xc, S=S, seed=case)
        dirs, w = O.rademacher(case, 0, N, S, D), np.full(S, 1.0 / S)
    else:
        J = int(rng.integers(1, 60))
        d = gaussian_directions(N, J, D, seed=case)
        ws = signed_weights(J, seed=case)
        mlp.directional_sum(Xc, 2, torch.from_numpy(d).cuda(), torch.from_numpy(ws).cuda())
        dirs, w = d.astype(np.float64), ws.astype(np.float64)
    grads = mlp.backward(go, gfc)
    dW, db, mag = _k2(Ws, bs, Xd, dirs, w, gop, gf)
    _check_grads(f"fuzz{case}_{which}_{widths}_N{N}", grads, dW, db, mag)


def test_pinn_poisson_example_trains(ctm):
    """examples/pinn_poisson.py: 150 Adam steps through ctm_laplacian + ctm_backward (two
    backward calls per step, the second accumulating) reduce the PINN loss by > 10x."""
    import importlib.util

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("pinn_poisson", os.path.join(root, "examples", "pinn_poisson.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    hist, err = mod.train(D=3, steps=150, N=1024, Nb=256, width=64, log_every=0)
    assert all(np.isfinite(hist))
    assert np.mean(hist[-10:]) < 0.1 * np.mean(hist[:5]), (hist[:5], hist[-10:])
