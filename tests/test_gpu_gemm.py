"""GEMM-only accuracy of the layer contraction (SURVEY §7 phase 3, §8(c) "Parity unpinned").

ctm_gemm_probe runs Z = B W_l^T through the operator path's own kernel (jet_layer_kernel,
the handle's precision mode) with the Taylor rule bypassed, so the bf16 plane split and the
tensor-core accumulation are measured alone against the plain definition (an fp64 matmul of
the same fp32 values), per element, relative to sum_k |B_k W_k|:

* fp32 mode (three planes, bf16x6 in two phases): <= 1e-6 on mixed-sign data
  (activations and weights as the network has them), and within the a-priori bound
  (K/16 + 1) 2^-23 on same-sign data, where the round-toward-zero accumulation of the
  K/16 leading MMAs meets its worst case (every partial sum as large as sum |B W|);
* fast mode (two planes, 3xBF16): <= 3e-5 (the 2^-17 operand split, three products).
"""
import numpy as np
import pytest
import torch

from synth import mlp_params, widths_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctm():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2505_13644_b200 as ctm

    ctm.lib()
    return ctm


def _mlp(ctm, params, precision):
    m = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0)
    m.set_precision(precision)
    return m


def _rows(rng, n, k, kind):
    """Slot rows like the network's blocks: tanh-range primals, first-order coefficients and
    collapsed tops whose magnitudes span 1e-4 .. 1e2 (per-row scale), ragged row count."""
    B = rng.uniform(-1.0, 1.0, size=(n, k))
    if kind == "mixed":
        B *= 10.0 ** rng.uniform(-4.0, 2.0, size=(n, 1))
    elif kind == "same_sign":
        B = np.abs(B) * 10.0 ** rng.uniform(-2.0, 1.0, size=(n, 1))
    return B.astype(np.float32)


def _err(Z, B, W):
    Bd, Wd = B.astype(np.float64), W.astype(np.float64)
    want = Bd @ Wd.T
    scale = np.abs(Bd) @ np.abs(Wd).T
    return np.abs(Z.double().cpu().numpy() - want) / np.maximum(scale, 1e-300)


@pytest.mark.parametrize("layer", [2, 3, 4])
def test_gemm_probe_fp32_mode_c1_layers(ctm, layer):
    """Every C1 hidden layer (768x768, 768x512, 512x512), 1001 rows (a ragged last tile)."""
    params = mlp_params(widths_for(50), 0)
    mlp = _mlp(ctm, params, "fp32")
    W = params[layer - 1][0]
    rng = np.random.default_rng(layer)
    B = _rows(rng, 1001, W.shape[1], "mixed")
    e = _err(mlp.gemm_probe(layer, torch.from_numpy(B).cuda()), B, W)
    assert e.max() <= 1e-6, e.max()


def test_gemm_probe_fp32_mode_same_sign_within_the_accumulation_bound(ctm):
    params = mlp_params(widths_for(50), 0)
    W = np.abs(params[1][0])
    params = [(p[0], p[1]) for p in params]
    params[1] = (W, params[1][1])
    mlp = _mlp(ctm, params, "fp32")
    B = _rows(np.random.default_rng(7), 400, W.shape[1], "same_sign")
    e = _err(mlp.gemm_probe(2, torch.from_numpy(B).cuda()), B, W)
    bound = (W.shape[1] / 16 + 1) * 2.0 ** -23
    assert e.max() <= bound, (e.max(), bound)


@pytest.mark.parametrize("widths", [[7, 40, 24, 1], [3, 300, 130, 260, 1]])
def test_gemm_probe_fp32_mode_padded_widths(ctm, widths):
    """Widths that are not multiples of the 256-feature pair tile or the 64-K block."""
    params = mlp_params(widths, 3)
    mlp = _mlp(ctm, params, "fp32")
    rng = np.random.default_rng(3)
    for layer in range(2, len(widths) - 1):
        W = params[layer - 1][0]
        B = _rows(rng, 37, W.shape[1], "mixed")
        e = _err(mlp.gemm_probe(layer, torch.from_numpy(B).cuda()), B, W)
        assert e.max() <= 1e-6, (layer, e.max())


def test_gemm_probe_fast_mode(ctm):
    params = mlp_params(widths_for(50), 0)
    mlp = _mlp(ctm, params, "bf16x3")
    W = params[1][0]
    B = _rows(np.random.default_rng(5), 513, W.shape[1], "mixed")
    e = _err(mlp.gemm_probe(2, torch.from_numpy(B).cuda()), B, W)
    assert e.max() <= 3e-5, e.max()
    assert e.max() > 1e-7  # the fast mode is measurably coarser than the fp32 mode


def test_gemm_probe_is_deterministic_and_row_independent(ctm):
    """The same row gives the same bits wherever it sits in the block (no N-dependent
    tiling or split-K): rows 0..99 alone vs inside a 1000-row block."""
    params = mlp_params(widths_for(50), 0)
    mlp = _mlp(ctm, params, "fp32")
    W = params[2][0]
    B = _rows(np.random.default_rng(9), 1000, W.shape[1], "mixed")
    Bt = torch.from_numpy(B).cuda()
    Z1 = mlp.gemm_probe(3, Bt)
    Z2 = mlp.gemm_probe(3, Bt[:100].contiguous())
    Z3 = mlp.gemm_probe(3, Bt)
    assert torch.equal(Z1, Z3)
    assert torch.equal(Z1[:100], Z2)
