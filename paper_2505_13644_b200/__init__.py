"""paper_2505_13644_b200 — collapsed Taylor mode PDE operators on B200 (arXiv 2505.13644).

A thin ctypes binding of ``libctm.so`` (C ABI: ``include/ctm.h``). Argument
marshalling only: every step of the hot path runs in the library's sm_100a
kernels. PyTorch provides device memory and streams. There is no CPU fallback:
if the CUDA library is missing or a call fails, this module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libctm.so")

CTM_RADEMACHER, CTM_GAUSSIAN = 0, 1
_STATUS = {0: "CTM_OK", 1: "CTM_EINVAL", 2: "CTM_ESHAPE", 3: "CTM_ENOMEM", 4: "CTM_ECUDA", 5: "CTM_EUNSUPPORTED"}

# The C ABI (include/ctm.h): name -> (restype, argtypes)
_VP, _I32, _I64, _U64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
ABI = {
    "ctm_load_mlp": (ctypes.c_int, [_I32, _VP, _VP, _VP, _I32, ctypes.POINTER(_VP)]),
    "ctm_free_mlp": (ctypes.c_int, [_VP]),
    "ctm_laplacian": (ctypes.c_int, [_VP, _VP, _I64, _VP, _VP, _VP]),
    "ctm_laplacian_standard": (ctypes.c_int, [_VP, _VP, _I64, _VP, _VP, _VP]),
    "ctm_weighted_laplacian": (ctypes.c_int, [_VP, _VP, _I64, _VP, _I32, _VP, _VP, _VP]),
    "ctm_randomized_laplacian": (
        ctypes.c_int,
        [_VP, _VP, _I64, _I32, _VP, ctypes.c_int, _U64, _I64, _VP, _I32, _VP, _VP, _VP],
    ),
    "ctm_biharmonic": (ctypes.c_int, [_VP, _VP, _I64, _VP, _VP, _VP]),
    "ctm_biharmonic_nested": (ctypes.c_int, [_VP, _VP, _I64, _VP, _VP, _VP]),
    "ctm_biharmonic_standard": (ctypes.c_int, [_VP, _VP, _I64, _VP, _VP, _VP]),
    "ctm_randomized_laplacian_standard": (
        ctypes.c_int,
        [_VP, _VP, _I64, _I32, _VP, ctypes.c_int, _U64, _I64, _VP, _I32, _VP, _VP, _VP],
    ),
    "ctm_stochastic_biharmonic_standard": (ctypes.c_int, [_VP, _VP, _I64, _I32, _VP, ctypes.c_int, _U64, _I64, _VP,
                                                          _VP, _VP]),
    "ctm_weighted_laplacian_pointwise": (ctypes.c_int, [_VP, _VP, _I64, _VP, _I32, _VP, _VP, _VP]),
    "ctm_directional_sum": (ctypes.c_int, [_VP, _VP, _I64, _I32, _I32, _VP, _I32, _VP, _VP, _VP, _VP]),
    "ctm_stochastic_biharmonic": (ctypes.c_int, [_VP, _VP, _I64, _I32, _VP, ctypes.c_int, _U64, _I64, _VP, _VP,
                                                 _VP]),
    "ctm_set_activation": (ctypes.c_int, [_VP, ctypes.c_int]),
    "ctm_set_precision": (ctypes.c_int, [_VP, ctypes.c_int]),
    "ctm_grad_enable": (ctypes.c_int, [_VP, _I32]),
    "ctm_set_weights": (ctypes.c_int, [_VP, _VP, _VP, _VP]),
    "ctm_backward": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _I32, _VP]),
    "ctm_status_str": (ctypes.c_char_p, [ctypes.c_int]),
    "ctm_last_error": (ctypes.c_char_p, []),
    "ctm_last_precision": (ctypes.c_int, [_VP, ctypes.POINTER(_I32)]),
    "ctm_last_plan": (ctypes.c_int, [_VP, ctypes.POINTER(_I32), ctypes.POINTER(_I32), ctypes.POINTER(_I32),
                                     ctypes.POINTER(_I32)]),
    "ctm_last_blocks": (ctypes.c_int, [_VP, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "ctm_set_direction_block": (ctypes.c_int, [_VP, _I32]),
    "ctm_plan_blocks": (ctypes.c_int, [_I32, _I32, _I32] + [ctypes.POINTER(_I32)] * 5),
    "ctm_gemm_probe": (ctypes.c_int, [_VP, _I32, _VP, _I64, _VP, _VP]),
    "ctm_profile_enable": (ctypes.c_int, [_VP, _I32]),
    "ctm_profile_read": (ctypes.c_int, [_VP, _VP, _VP, _VP]),
}
KINDS = ("prep", "seed", "layer", "final", "bwd", "wgrad", "baux")

_lib = None


class CTMError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    """Load libctm.so (built in-tree by ``paper_2505_13644_b200.build``). Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CTMError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2505_13644_b200.build` "
                "(there is no fallback path)"
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in ABI.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != 0:
        detail = lib().ctm_last_error().decode()
        raise CTMError(f"{what} -> {_STATUS.get(status, status)}: {detail}")


def _stream_ptr(stream: Optional[torch.cuda.Stream], device) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def _streamed(method):
    """Run an operator method with ``stream`` as torch's current stream, so every
    temporary (dtype/layout conversions, outputs) is allocated and written on the stream
    the library's kernels run on: the caching allocator cannot hand a block back to
    other work while the library still reads it (ctm.h: inputs stay valid until the
    stream passes the call)."""
    import functools

    @functools.wraps(method)
    def run(self, *args, stream=None, **kw):
        if stream is None or stream == torch.cuda.current_stream(self.device):
            return method(self, *args, **kw)
        with torch.cuda.stream(stream):
            return method(self, *args, **kw)

    return run


def _dev_f32(t: torch.Tensor, device, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t)
    t = t.to(device=device, dtype=torch.float32).contiguous()
    if t.data_ptr() % 16:
        t = t.clone()
    return t


def plan_blocks(order: int, R: int, forced_rb: int = 0) -> dict:
    """The library's direction-block planner (host only, no GPU): ``ctm_plan_blocks``."""
    out = [_I32() for _ in range(5)]
    _check(lib().ctm_plan_blocks(int(order), int(R), int(forced_rb), *[ctypes.byref(o) for o in out]),
           "ctm_plan_blocks")
    keys = ("blocks", "per_block", "slots_per_block", "points_per_tile", "mma_n")
    return {k: o.value for k, o in zip(keys, out)}


ACTIVATIONS = {"tanh": 0, "identity": 1, "square": 2, "sin": 3, "exp": 4}  # ctm_activation
PRECISIONS = {"fp32": 0, "bf16x3": 1, "fp16x3": 2}  # ctm_precision


class MLP:
    """An MLP f: R^D -> R loaded into libctm (weights copied to the device).

    params: sequence of (W_l [w_l, w_{l-1}], b_l [w_l]) as in ``torch.nn.Linear``;
    the activation (tanh by default; or sin, exp, identity, square) after every layer
    but the last.
    """

    def __init__(self, params: Sequence, device: int | str | torch.device | None = None, act: str = "tanh",
                 precision: str | None = None):
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        Ws = [_dev_f32(W, self.device, "W") for W, _ in params]
        bs = [_dev_f32(b, self.device, "b").reshape(-1) for _, b in params]
        widths = [Ws[0].shape[1]] + [W.shape[0] for W in Ws]
        self.widths = widths
        self.D = widths[0]
        w_arr = (_I32 * len(widths))(*widths)
        W_arr = (_VP * len(Ws))(*[W.data_ptr() for W in Ws])
        b_arr = (_VP * len(bs))(*[b.data_ptr() for b in bs])
        h = _VP()
        _check(
            lib().ctm_load_mlp(len(Ws), w_arr, W_arr, b_arr, self.device.index, ctypes.byref(h)), "ctm_load_mlp"
        )
        self._h = h
        if act not in ACTIVATIONS:
            raise CTMError(f"unknown activation {act!r}")
        _check(lib().ctm_set_activation(self._h, ACTIVATIONS[act]), "ctm_set_activation")
        self.act = act
        self._grad = False
        self._tape_n = None
        # the environment may choose the default arithmetic of new handles (CTM_PRECISION)
        self.set_precision(precision or os.environ.get("CTM_PRECISION", "fp32"))

    def set_precision(self, precision: str = "fp32"):
        """Arithmetic of the layer contractions (ctm_set_precision): "fp32" (default, three
        bf16 planes, six products), "fp16x3" (two scaled fp16 planes, three products: the
        3xTF32 operand split at bf16 speed, K=2 forward operators; others run fp32) or
        "bf16x3" (two bf16 planes, three products, ~17 bits)."""
        if precision not in PRECISIONS:
            raise CTMError(f"unknown precision {precision!r} (fp32, fp16x3 or bf16x3)")
        _check(lib().ctm_set_precision(self._h, PRECISIONS[precision]), "ctm_set_precision")
        self.precision = precision
        self._tape_n = None

    # ------------------------------------------------------------------ helpers
    def _io(self, X, out, f_out, want_f):
        X = _dev_f32(X, self.device, "X")
        if X.dim() != 2 or X.shape[1] != self.D:
            raise CTMError(f"X must be [N, {self.D}]")
        N = X.shape[0]
        if out is None:
            out = torch.empty(N, device=self.device, dtype=torch.float32)
        if f_out is None and want_f:
            f_out = torch.empty(N, device=self.device, dtype=torch.float32)
        return X, N, out, f_out

    @staticmethod
    def _p(t):
        return None if t is None else t.data_ptr()

    def _taped(self, N):
        """A K=2 operator call in grad mode recorded a tape of N points."""
        self._tape_n = N if self._grad else None

    # ------------------------------------------------------------------ operators
    @_streamed
    def laplacian(self, X, out=None, f_out=None, want_f=True, stream=None):
        """Exact Laplacian (Eq. 8). Returns (op [N], f [N] or None)."""
        X, N, out, f_out = self._io(X, out, f_out, want_f)
        _check(lib().ctm_laplacian(self._h, X.data_ptr(), N, out.data_ptr(), self._p(f_out),
                                   _stream_ptr(stream, self.device)), "ctm_laplacian")
        self._taped(N)
        return out, f_out

    @_streamed
    def laplacian_standard(self, X, out=None, f_out=None, want_f=True, stream=None):
        """Exact Laplacian by STANDARD Taylor mode (1 + 2D vectors per layer): the
        paper's baseline, same value as ``laplacian``."""
        X, N, out, f_out = self._io(X, out, f_out, want_f)
        _check(lib().ctm_laplacian_standard(self._h, X.data_ptr(), N, out.data_ptr(), self._p(f_out),
                                            _stream_ptr(stream, self.device)), "ctm_laplacian_standard")
        return out, f_out

    @_streamed
    def weighted_laplacian(self, X, sigma, out=None, f_out=None, want_f=True, stream=None):
        """<d^2 f, sigma sigma^T> (Eq. 10), sigma [D, R]."""
        X, N, out, f_out = self._io(X, out, f_out, want_f)
        sigma = _dev_f32(sigma, self.device, "sigma")
        if sigma.dim() != 2 or sigma.shape[0] != self.D:
            raise CTMError(f"sigma must be [D={self.D}, R]")
        _check(lib().ctm_weighted_laplacian(self._h, X.data_ptr(), N, sigma.data_ptr(), sigma.shape[1],
                                            out.data_ptr(), self._p(f_out), _stream_ptr(stream, self.device)),
               "ctm_weighted_laplacian")
        self._taped(N)
        return out, f_out

    @_streamed
    def randomized_laplacian(self, X, S=None, V=None, seed=0, point_offset=0, sigma=None, dist="rademacher",
                             out=None, f_out=None, want_f=True, stream=None, standard=False):
        """(1/S) sum_s <d^2 f, (sigma v_s)^2> (Eq. 8/10 stochastic). V [N, S, Rv] or generated.
        standard=True: the same estimator by standard (uncollapsed) Taylor mode (baseline)."""
        X, N, out, f_out = self._io(X, out, f_out, want_f)
        if V is not None:
            V = _dev_f32(V, self.device, "V")
            if V.dim() != 3 or V.shape[0] != N:
                raise CTMError(f"V must be [N={N}, S, Rv]")
            S, Rv = V.shape[1], V.shape[2]
        if sigma is not None:
            sigma = _dev_f32(sigma, self.device, "sigma")
            if sigma.dim() != 2 or sigma.shape[0] != self.D:
                raise CTMError(f"sigma must be [D={self.D}, Rv]")
            if V is not None and sigma.shape[1] != Rv:
                raise CTMError(f"sigma must be [D, Rv={Rv}] to match V [N, S, Rv]")
            Rv = sigma.shape[1]
        elif V is None:
            Rv = self.D
        elif Rv != self.D:
            raise CTMError(f"V must be [N, S, D={self.D}] without sigma")
        if S is None:
            raise CTMError("S is required when V is not given")
        d = {"rademacher": CTM_RADEMACHER, "gaussian": CTM_GAUSSIAN}[dist]
        fn = lib().ctm_randomized_laplacian_standard if standard else lib().ctm_randomized_laplacian
        _check(fn(self._h, X.data_ptr(), N, int(S), self._p(V), d, int(seed) & (2**64 - 1), int(point_offset),
                  self._p(sigma), int(Rv), out.data_ptr(), self._p(f_out), _stream_ptr(stream, self.device)),
               "ctm_randomized_laplacian" + ("_standard" if standard else ""))
        self._taped(N if not standard else None)
        return out, f_out

    @_streamed
    def biharmonic(self, X, out=None, f_out=None, want_f=True, stream=None):
        """Exact biharmonic (Eq. 12) via the interpolation family, one collapsed slot."""
        X, N, out, f_out = self._io(X, out, f_out, want_f)
        _check(lib().ctm_biharmonic(self._h, X.data_ptr(), N, out.data_ptr(), self._p(f_out),
                                    _stream_ptr(stream, self.device)), "ctm_biharmonic")
        return out, f_out

    @_streamed
    def biharmonic_standard(self, X, out=None, f_out=None, want_f=True, stream=None):
        """The same biharmonic by standard (uncollapsed) Taylor mode: 1 + 4J vectors (baseline)."""
        X, N, out, f_out = self._io(X, out, f_out, want_f)
        _check(lib().ctm_biharmonic_standard(self._h, X.data_ptr(), N, out.data_ptr(), self._p(f_out),
                                             _stream_ptr(stream, self.device)), "ctm_biharmonic_standard")
        return out, f_out

    @_streamed
    def weighted_laplacian_pointwise(self, X, sigma_x, out=None, f_out=None, want_f=True, stream=None):
        """<d^2 f(x_n), sigma(x_n) sigma(x_n)^T> with sigma_x [N, D, R] (Eq. 10, sigma depending on x)."""
        X, N, out, f_out = self._io(X, out, f_out, want_f)
        sigma_x = _dev_f32(sigma_x, self.device, "sigma_x")
        if sigma_x.dim() != 3 or sigma_x.shape[0] != N or sigma_x.shape[1] != self.D:
            raise CTMError(f"sigma_x must be [N={N}, D={self.D}, R]")
        _check(lib().ctm_weighted_laplacian_pointwise(self._h, X.data_ptr(), N, sigma_x.data_ptr(),
                                                      int(sigma_x.shape[2]), out.data_ptr(), self._p(f_out),
                                                      _stream_ptr(stream, self.device)),
               "ctm_weighted_laplacian_pointwise")
        self._taped(N)
        return out, f_out

    @_streamed
    def directional_sum(self, X, K, dirs, weights, out=None, f_out=None, want_f=True, stream=None):
        """sum_j w_j <d^K f, u_j^K>, K in {2, 4}; dirs [J, D] shared or [N, J, D] per point (Eq. 5, Eq. 13-15)."""
        X, N, out, f_out = self._io(X, out, f_out, want_f)
        dirs = _dev_f32(dirs, self.device, "dirs")
        weights = _dev_f32(weights, self.device, "weights")
        per_point = dirs.dim() == 3
        J = int(weights.numel())
        if dirs.dim() not in (2, 3) or dirs.shape[-2] != J or dirs.shape[-1] != self.D or (
                per_point and dirs.shape[0] != N):
            raise CTMError(f"dirs must be [J, D={self.D}] or [N={N}, J, D] with J = len(weights)")
        _check(lib().ctm_directional_sum(self._h, X.data_ptr(), N, int(K), J, dirs.data_ptr(), int(per_point),
                                         weights.data_ptr(), out.data_ptr(), self._p(f_out),
                                         _stream_ptr(stream, self.device)), "ctm_directional_sum")
        self._taped(N if int(K) == 2 else None)
        return out, f_out

    @_streamed
    def biharmonic_nested(self, X, out=None, f_out=None, want_f=True, stream=None):
        """Exact biharmonic (Eq. 12) by nested collapsed Laplacians, 2 + 2D + D(D+1)/2 slots."""
        X, N, out, f_out = self._io(X, out, f_out, want_f)
        _check(lib().ctm_biharmonic_nested(self._h, X.data_ptr(), N, out.data_ptr(), self._p(f_out),
                                           _stream_ptr(stream, self.device)), "ctm_biharmonic_nested")
        return out, f_out

    @_streamed
    def stochastic_biharmonic(self, X, S=None, V=None, seed=0, point_offset=0, out=None, f_out=None, want_f=True,
                              stream=None, standard=False):
        """1/(3S) sum_s <d^4 f, v_s^4>, v_s ~ N(0, I) (Eq. 12 stochastic; V [N, S, D] or generated).
        standard=True: the same estimator by standard (uncollapsed) Taylor mode (baseline)."""
        X, N, out, f_out = self._io(X, out, f_out, want_f)
        if V is not None:
            V = _dev_f32(V, self.device, "V")
            S = V.shape[1]
        if S is None:
            raise CTMError("S is required when V is not given")
        fn = lib().ctm_stochastic_biharmonic_standard if standard else lib().ctm_stochastic_biharmonic
        _check(fn(self._h, X.data_ptr(), N, int(S), self._p(V), CTM_GAUSSIAN, int(seed) & (2**64 - 1),
                  int(point_offset), out.data_ptr(), self._p(f_out), _stream_ptr(stream, self.device)),
               "ctm_stochastic_biharmonic" + ("_standard" if standard else ""))
        return out, f_out

    @_streamed
    def set_weights(self, params: Sequence, stream=None):
        """Replace the weights (same widths) asynchronously on ``stream`` (e.g. after an
        optimizer step). Keeps device copies alive until the next call."""
        Ws = [_dev_f32(W, self.device, "W") for W, _ in params]
        bs = [_dev_f32(b, self.device, "b").reshape(-1) for _, b in params]
        if [Ws[0].shape[1]] + [W.shape[0] for W in Ws] != list(self.widths):
            raise CTMError("set_weights: widths differ from the loaded MLP")
        W_arr = (_VP * len(Ws))(*[W.data_ptr() for W in Ws])
        b_arr = (_VP * len(bs))(*[b.data_ptr() for b in bs])
        _check(lib().ctm_set_weights(self._h, W_arr, b_arr, _stream_ptr(stream, self.device)), "ctm_set_weights")
        self._keep = (Ws, bs)

    # ------------------------------------------------------------------ differentiable path
    def grad_enable(self, enable: bool = True):
        """Record a tape on later K=2 operator calls so that ``backward`` can run (NEXT-3)."""
        _check(lib().ctm_grad_enable(self._h, int(bool(enable))), "ctm_grad_enable")
        self._grad = bool(enable)
        self._tape_n = None

    @_streamed
    def backward(self, gop, gf=None, grads=None, accumulate=False, stream=None):
        """Gradients of sum_n gop[n] op[n] + gf[n] f[n] for the last recorded call.

        Returns [(dW_l, db_l)] in nn.Linear layout (fp32, on the device); pass ``grads``
        (same structure) to write into existing tensors, with ``accumulate`` to add."""
        gop = _dev_f32(gop, self.device, "gop").reshape(-1)
        gf = None if gf is None else _dev_f32(gf, self.device, "gf").reshape(-1)
        if self._tape_n is not None and (gop.numel() != self._tape_n or (gf is not None and gf.numel() != self._tape_n)):
            raise CTMError(f"gop/gf must have the {self._tape_n} elements of the recorded call")
        if grads is None:
            grads = [(torch.empty(self.widths[l + 1], self.widths[l], device=self.device),
                      torch.empty(self.widths[l + 1], device=self.device)) for l in range(len(self.widths) - 1)]
        L = len(grads)
        dW = (_VP * L)(*[g[0].data_ptr() for g in grads])
        db = (_VP * L)(*[g[1].data_ptr() for g in grads])
        _check(lib().ctm_backward(self._h, gop.data_ptr(), self._p(gf), dW, db, int(bool(accumulate)),
                                  _stream_ptr(stream, self.device)), "ctm_backward")
        return grads

    @_streamed
    def gemm_probe(self, layer: int, B, Z=None, stream=None):
        """Z = B W_layer^T (no bias) through the layer kernel with the Taylor rule bypassed
        (ctm_gemm_probe; the GEMM-only accuracy test). layer is 1-based (2 .. L-1)."""
        B = _dev_f32(B, self.device, "B")
        if B.dim() != 2 or B.shape[1] != self.widths[layer - 1]:
            raise CTMError(f"B must be [rows, {self.widths[layer - 1]}]")
        if Z is None:
            Z = torch.empty(B.shape[0], self.widths[layer], device=self.device, dtype=torch.float32)
        _check(lib().ctm_gemm_probe(self._h, int(layer), B.data_ptr(), B.shape[0], Z.data_ptr(),
                                    _stream_ptr(stream, self.device)), "ctm_gemm_probe")
        return Z

    def last_precision(self) -> str:
        """The arithmetic the last operator call ran in (ctm_last_precision)."""
        v = _I32()
        _check(lib().ctm_last_precision(self._h, ctypes.byref(v)), "ctm_last_precision")
        return {c: k for k, c in PRECISIONS.items()}[v.value]

    def last_plan(self) -> dict:
        a, b, c, d = _I32(), _I32(), _I32(), _I32()
        _check(lib().ctm_last_plan(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d)),
               "ctm_last_plan")
        nb, rb = _I32(), _I32()
        _check(lib().ctm_last_blocks(self._h, ctypes.byref(nb), ctypes.byref(rb)), "ctm_last_blocks")
        return {"launches": a.value, "slots_per_point": b.value, "points_per_tile": c.value, "mma_n": d.value,
                "blocks": nb.value, "per_block": rb.value}

    def set_direction_block(self, rb: int = 0):
        """Fix the directions per block of later calls (0: the library's planner); ctm.h."""
        _check(lib().ctm_set_direction_block(self._h, int(rb)), "ctm_set_direction_block")

    def profile(self, enable: bool = True):
        """Bracket every launch with CUDA events on its stream (see ctm_profile_read)."""
        _check(lib().ctm_profile_enable(self._h, int(enable)), "ctm_profile_enable")

    def profile_read(self) -> dict:
        """{kind: {"ms", "launches", "work"}} summed since the last read; clears."""
        import numpy as np

        ms = np.zeros(len(KINDS))
        n = np.zeros(len(KINDS), dtype=np.int64)
        w = np.zeros(len(KINDS))
        _check(lib().ctm_profile_read(self._h, ms.ctypes.data, n.ctypes.data, w.ctypes.data), "ctm_profile_read")
        return {k: {"ms": float(ms[i]), "launches": int(n[i]), "work": float(w[i])} for i, k in enumerate(KINDS)}

    def close(self):
        if getattr(self, "_h", None):
            lib().ctm_free_mlp(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
