"""The fp16x3 precision mode (ctm_set_precision(CTM_PRECISION_FP16X3)): two
power-of-two-scaled fp16 planes per operand (11 + 11 significant bits, the operand split of
3xTF32 that north_star names), products p1*p0 + p0*p1 over the whole K, then p0*p0.

* which calls it covers, and that every other call on an fp16x3 handle runs the fp32 mode;
* parity at the north_star metric for every covered operator (1e-4 of the normaliser), tanh
  and sin nets, BASELINE shapes and small nets;
* the GEMM alone against fp64 (ctm_gemm_probe), relative to sum_k |B_k W_k|;
* the scale machinery: values far above and below 1 (no fp16 overflow, no loss of the small
  ones), the bound records of a call do not leak into the next call.
The whole parity suite also runs in this mode with CTM_PRECISION=fp16x3 (scripts/gpu_fp16x3_suite.sh).
"""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gaussian_directions, mlp_params, points, sigma as make_sigma, sigma_field, signed_weights, widths_for

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def ctm():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2505_13644_b200 as ctm

    ctm.lib()
    return ctm


def _nets(widths, seed=0, scale=1.0):
    params = mlp_params(widths, seed)
    params = [(W * scale, b * scale) for W, b in params]
    onet = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params])
    return params, onet


def _mlp(ctm, params, act="tanh", precision="fp16x3"):
    return ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0, act=act,
                   precision=precision)


def _check(got, want, norm, tol=TOL):
    e = np.abs(got.double().cpu().numpy() - want) / norm
    assert np.all(np.isfinite(e)) and e.max() <= tol, e.max()
    return e.max()


def test_fp16x3_covers_the_k2_forward_operators_and_falls_back_otherwise(ctm):
    params, _ = _nets([5, 64, 48, 1])
    X = torch.from_numpy(points(9, 5)).cuda()
    m = _mlp(ctm, params)
    m.laplacian(X)
    assert m.last_precision() == "fp16x3"
    m.weighted_laplacian(X, torch.from_numpy(make_sigma(5, 3, kind="rect")).cuda())
    assert m.last_precision() == "fp16x3"
    m.randomized_laplacian(X, S=4, seed=1)
    assert m.last_precision() == "fp16x3"
    m.randomized_laplacian(X, S=4, seed=1, sigma=torch.from_numpy(make_sigma(5, 5)).cuda())
    assert m.last_precision() == "fp16x3"  # with a sigma matrix too
    m.biharmonic(X)
    assert m.last_precision() == "fp16x3"  # K=4, the interpolation family
    m.stochastic_biharmonic(X, S=3, seed=2)
    assert m.last_precision() == "fp16x3"  # per-point K=4 directions: layer 1 fp32, its output fp16x3
    m.biharmonic_nested(X)
    assert m.last_precision() == "fp16x3"  # the nested Laplacians: one scale per block
    m.laplacian_standard(X)
    assert m.last_precision() == "fp16x3"  # the standard-mode baselines too
    m.grad_enable()
    m.laplacian(X)
    assert m.last_precision() == "fp16x3"  # fp16x3 training: fixed direction sets
    m.randomized_laplacian(X, S=4, seed=1)
    assert m.last_precision() == "fp16x3"  # per-point directions in grad mode too
    m.randomized_laplacian(X, S=4, seed=1, sigma=torch.from_numpy(make_sigma(5, 5)).cuda())
    assert m.last_precision() == "fp16x3"
    m.grad_enable(False)
    m.laplacian(X)
    assert m.last_precision() == "fp16x3"
    e = _mlp(ctm, params, act="exp")
    e.laplacian(X)
    assert e.last_precision() == "fp32"
    f = _mlp(ctm, params, precision="bf16x3")
    f.laplacian(X)
    assert f.last_precision() == "bf16x3"
    for h in (m, e, f):
        h.close()


@pytest.mark.parametrize("act", ["tanh", "sin"])
@pytest.mark.parametrize("widths,N", [([5, 64, 48, 1], 37), ([50, 768, 256, 1], 65), ([3, 300, 130, 260, 1], 23)])
def test_fp16x3_parity_every_covered_operator(ctm, act, widths, N):
    params, onet = _nets(widths, seed=4)
    onet = O.Net(onet.Ws, onet.bs, act)
    D = widths[0]
    X = points(N, D, seed=4)
    Xc, Xd = torch.from_numpy(X).cuda(), X.astype(np.float64)
    m = _mlp(ctm, params, act=act)
    want, fw, norm = O.laplacian(onet, Xd)
    op, f = m.laplacian(Xc)
    assert m.last_precision() == "fp16x3"
    _check(op, want, norm)
    assert np.abs(f.double().cpu().numpy() - fw).max() <= 1e-5 * max(1.0, np.abs(fw).max())
    sig = make_sigma(D, min(D, 7), kind="rect")
    want, _, norm = O.weighted_laplacian(onet, Xd, sig.astype(np.float64))
    _check(m.weighted_laplacian(Xc, torch.from_numpy(sig).cuda())[0], want, norm)
    V = O.rademacher(3, 0, N, 6, D)
    want, _, norm = O.randomized_laplacian(onet, Xd, V)
    _check(m.randomized_laplacian(Xc, S=6, seed=3)[0], want, norm)
    Vg = np.random.default_rng(2).standard_normal((N, 5, D)).astype(np.float32)
    want, _, norm = O.randomized_laplacian(onet, Xd, Vg.astype(np.float64))
    _check(m.randomized_laplacian(Xc, V=torch.from_numpy(Vg).cuda(), dist="gaussian")[0], want, norm)
    # with a sigma matrix (Eq. 10 stochastic: u = sigma v), Rademacher v drawn in-kernel
    sg = make_sigma(D, min(D, 4), kind="rect")
    Vs = O.rademacher(3, 0, N, 6, sg.shape[1])
    want, _, norm = O.randomized_laplacian(onet, Xd, Vs, sg.astype(np.float64))
    _check(m.randomized_laplacian(Xc, S=6, seed=3, sigma=torch.from_numpy(sg).cuda())[0], want, norm)
    assert m.last_precision() == "fp16x3"
    sx = sigma_field(X, 4)
    want, _, norm = O.weighted_laplacian_pointwise(onet, Xd, sx.astype(np.float64))
    _check(m.weighted_laplacian_pointwise(Xc, torch.from_numpy(sx).cuda())[0], want, norm)
    w = signed_weights(5)
    for per_point in (False, True):
        dirs = gaussian_directions(N, 5, D, seed=8) if per_point else gaussian_directions(1, 5, D, seed=8)[0]
        got = m.directional_sum(Xc, 2, torch.from_numpy(dirs).cuda(), torch.from_numpy(w).cuda())[0]
        assert m.last_precision() == "fp16x3"
        want, _, norm = O.directional_sum(onet, Xd, 2, dirs.astype(np.float64), w.astype(np.float64))
        _check(got, want, norm)
    if D <= 7:  # K=4: the biharmonic family and a shared K=4 directional sum; nested Laplacians
        want, _, norm = O.biharmonic(onet, Xd)
        _check(m.biharmonic(Xc)[0], want, norm)
        assert m.last_precision() == "fp16x3"
        _check(m.biharmonic_nested(Xc)[0], want, norm)
        assert m.last_precision() == "fp16x3"
    w4 = signed_weights(4)
    for per_point in (False, True):  # K=4 sums, shared and per-point directions
        dirs = gaussian_directions(N, 4, D, seed=9) if per_point else gaussian_directions(1, 4, D, seed=9)[0]
        got = m.directional_sum(Xc, 4, torch.from_numpy(dirs).cuda(), torch.from_numpy(w4).cuda())[0]
        assert m.last_precision() == "fp16x3"
        want, _, norm = O.directional_sum(onet, Xd, 4, dirs.astype(np.float64), w4.astype(np.float64))
        _check(got, want, norm)
    # the stochastic biharmonic (Eq. 12 stochastic, scale 1/(3S)) with explicit Gaussian V,
    # collapsed and standard
    Vb = gaussian_directions(N, 6, D, seed=10)
    want, _, norm = O.stochastic_biharmonic(onet, Xd, Vb.astype(np.float64))
    for std in (False, True):
        got = m.stochastic_biharmonic(Xc, V=torch.from_numpy(Vb).cuda(), standard=std)[0]
        assert m.last_precision() == "fp16x3"
        _check(got, want, norm)
    # the standard-mode baselines: exact and randomized Laplacian, biharmonic
    want, _, norm = O.laplacian(onet, Xd)
    _check(m.laplacian_standard(Xc)[0], want, norm)
    assert m.last_precision() == "fp16x3"
    V = O.rademacher(3, 0, N, 6, D)
    want, _, norm = O.randomized_laplacian(onet, Xd, V)
    _check(m.randomized_laplacian(Xc, S=6, seed=3, standard=True)[0], want, norm)
    assert m.last_precision() == "fp16x3"
    if D <= 7:
        want, _, norm = O.biharmonic(onet, Xd)
        _check(m.biharmonic_standard(Xc)[0], want, norm)
        assert m.last_precision() == "fp16x3"
    m.close()


@pytest.mark.parametrize("op,S", [("laplacian", 0), ("weighted", 0), ("randomized", 8), ("randomized", 32),
                                  ("randomized", 128), ("biharmonic", 0), ("biharmonic_nested", 0),
                                  ("stochastic_biharmonic", 16)])
def test_fp16x3_full_size_sampled(ctm, op, S):
    """BASELINE C1 / C2 / C3 / C4 at N = 16384 in the bench's launch configuration (the bench's
    default mode), 256 sampled points at every position inside a tile; op at the north_star
    metric and f(x) to 1e-5 max(1, |f|)."""
    D = 5 if "biharmonic" in op else 50
    params, onet = _nets(widths_for(D), 0)
    N = 16384
    X = points(N, D)
    Xc = torch.from_numpy(X).cuda()
    m = _mlp(ctm, params)
    idx = np.unique(np.minimum(np.arange(0, N, N // 256)[:256] + np.arange(256) % 16, N - 1))
    Xs = X[idx].astype(np.float64)
    if op == "laplacian":
        got, f = m.laplacian(Xc)
        want, fwant, norm = O.laplacian(onet, Xs)
    elif op == "weighted":
        sig = make_sigma(D, D, kind="dense")
        got, f = m.weighted_laplacian(Xc, torch.from_numpy(sig).cuda())
        want, fwant, norm = O.weighted_laplacian(onet, Xs, sig.astype(np.float64))
    elif op == "biharmonic":
        got, f = m.biharmonic(Xc)
        want, fwant, norm = O.biharmonic(onet, Xs)
    elif op == "biharmonic_nested":
        got, f = m.biharmonic_nested(Xc)
        want, fwant, norm = O.biharmonic(onet, Xs)
    elif op == "stochastic_biharmonic":  # explicit Gaussian directions (the oracle needs them)
        Vb = gaussian_directions(N, S, D, seed=5)
        got, f = m.stochastic_biharmonic(Xc, V=torch.from_numpy(Vb).cuda())
        want, fwant, norm = O.stochastic_biharmonic(onet, Xs, Vb[idx].astype(np.float64))
    else:
        got, f = m.randomized_laplacian(Xc, S=S, seed=2)
        V = np.concatenate([O.rademacher(2, int(n), 1, S, 50) for n in idx])
        want, fwant, norm = O.randomized_laplacian(onet, Xs, V)
    assert m.last_precision() == "fp16x3"
    _check(got.cpu()[idx], want, norm)
    fe = np.abs(f.double().cpu().numpy()[idx] - fwant) / np.maximum(1.0, np.abs(fwant))
    assert fe.max() <= 1e-5, fe.max()
    m.close()


def test_fp16x3_c1_every_point(ctm):
    """The bench's default line exactly: C1 (D = 50, 768-768-512-512), N = 16384, the fp16x3
    mode, the same seeded weights and points as bench.py -- EVERY point against the fp64
    oracle (route O1, ~70 s on the box's cores): op at the north_star metric, f(x) to
    1e-5 max(1, |f|)."""
    params, onet = _nets(widths_for(50), 0)
    N = 16384
    X = points(N, 50, 1)  # bench.py: points(n_glob, D, 1)
    m = _mlp(ctm, params)
    got, f = m.laplacian(torch.from_numpy(X).cuda())
    assert m.last_precision() == "fp16x3"
    want, fwant, norm = O.laplacian(onet, X.astype(np.float64))
    e = _check(got.cpu(), want, norm)
    fe = np.abs(f.double().cpu().numpy() - fwant) / np.maximum(1.0, np.abs(fwant))
    assert fe.max() <= 1e-5, fe.max()
    print(f"C1 fp16x3, all {N} points: max err {e:.2e}, f max err {fe.max():.2e}")
    m.close()


@pytest.mark.parametrize("scale", [1e-3, 30.0])
def test_fp16x3_scales_follow_the_data(ctm, scale):
    """Inputs far from 1 (x scaled by 1e-3 or 30 -- tiny first-order values, or saturated tanh
    with top coefficients in the hundreds): the per-slot-type scales keep every plane inside
    fp16's range, and the result still meets the metric."""
    widths = [6, 128, 96, 1]
    params, onet = _nets(widths, seed=6, scale=3.0)
    X = (points(40, 6, seed=6) * scale).astype(np.float32)
    m = _mlp(ctm, params)
    got = m.laplacian(torch.from_numpy(X).cuda())[0]
    want, _, norm = O.laplacian(onet, X.astype(np.float64))
    _check(got, want, norm)
    m.close()


def test_fp16x3_records_do_not_leak_between_calls(ctm):
    """A call with huge values, then one with tiny values on the same handle: the second must
    not inherit the first call's bounds (records are reset per call), and equals a fresh handle
    bit for bit."""
    params, _ = _nets([8, 96, 64, 1], seed=2)
    big = torch.from_numpy((points(30, 8, seed=2) * 40).astype(np.float32)).cuda()
    small = torch.from_numpy((points(30, 8, seed=3) * 1e-3).astype(np.float32)).cuda()
    a = _mlp(ctm, params)
    a.laplacian(big)
    got = a.laplacian(small)[0].clone()
    b = _mlp(ctm, params)
    want = b.laplacian(small)[0]
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    a.close()
    b.close()


def _rows(rng, n, k, decades):
    B = rng.uniform(-1.0, 1.0, size=(n, k)) * 10.0 ** rng.uniform(-decades / 2, decades / 2, size=(n, 1))
    return B.astype(np.float32)


@pytest.mark.parametrize("layer", [2, 3, 4])
def test_fp16x3_gemm_probe_c1_layers(ctm, layer):
    """The contraction alone vs fp64, relative to sum_k |B_k W_k|, rows spanning 4 decades (the
    probe scales the whole block by one power of two): <= 1e-6, the fp32-mode bar; and above
    the fp32 mode's error on the same rows (the 22-bit split is measurably coarser)."""
    params = mlp_params(widths_for(50), 0)
    W = params[layer - 1][0]
    B = _rows(np.random.default_rng(layer), 1001, W.shape[1], 4.0)
    Bt = torch.from_numpy(B).cuda()
    Bd, Wd = B.astype(np.float64), W.astype(np.float64)
    scale = np.abs(Bd) @ np.abs(Wd).T
    errs = {}
    for prec in ("fp16x3", "fp32"):
        m = _mlp(ctm, params, precision=prec)
        Z = m.gemm_probe(layer, Bt).double().cpu().numpy()
        errs[prec] = (np.abs(Z - Bd @ Wd.T) / scale).max()
        m.close()
    assert errs["fp16x3"] <= 1e-6, errs
    assert errs["fp16x3"] > errs["fp32"], errs


@pytest.mark.parametrize("op", ["laplacian", "randomized"])
def test_fp16x3_split_batches_are_bitwise_equal(ctm, op):
    """The block scales are chosen per call from the call's data, but scaling by a power of two
    is exact and the residual plane is lifted out of fp16's subnormal range, so the result of a
    point does not depend on the rest of its batch: a batch equals its two halves bit for bit
    (the 1-vs-G invariant of SURVEY §8(e))."""
    params, _ = _nets([20, 256, 128, 1], seed=5)
    X = torch.from_numpy(points(100, 20, seed=5)).cuda()
    X[:37] *= 8.0  # the halves have different maxima, so different scales
    m = _mlp(ctm, params)
    if op == "laplacian":
        full = m.laplacian(X)[0].clone()
        parts = torch.cat([m.laplacian(X[:37])[0].clone(), m.laplacian(X[37:])[0].clone()])
    else:
        full = m.randomized_laplacian(X, S=12, seed=9)[0].clone()
        parts = torch.cat([m.randomized_laplacian(X[:37], S=12, seed=9, point_offset=0)[0].clone(),
                           m.randomized_laplacian(X[37:], S=12, seed=9, point_offset=37)[0].clone()])
    torch.cuda.synchronize()
    assert m.last_precision() == "fp16x3"
    assert torch.equal(full, parts)
    m.close()
