"""fp64 CPU oracle for collapsed Taylor mode (arXiv 2505.13644) — ctypes binding.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module. The product package (``paper_2505_13644_b200``) never imports it, and
the C source (``oracle/ctmo.c``) shares no code with the CUDA path.

Every function here is marshalling only; the arithmetic is in ``ctmo.c``, which
cites the passage of the paper each routine follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ctmo.c")
_LIB = os.path.join(_HERE, "libctmo.so")

TANH, IDENTITY, SQUARE, SIN, EXP = 0, 1, 2, 3, 4
O1, O2, O3 = 1, 2, 3
ACTS = {"tanh": TANH, "identity": IDENTITY, "square": SQUARE, "sin": SIN, "exp": EXP}


def build(force: bool = False) -> str:
    """Compile ``ctmo.c`` into ``libctmo.so`` (gcc, fp64, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "ctmo.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


class _Net(ctypes.Structure):
    _fields_ = [
        ("L", ctypes.c_int32),
        ("widths", ctypes.POINTER(ctypes.c_int32)),
        ("params", ctypes.POINTER(ctypes.c_double)),
        ("act", ctypes.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d, i64, i32, vp = ctypes.c_double, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        P = ctypes.POINTER
        for name in ("ctmo_laplacian", "ctmo_biharmonic"):
            getattr(_lib, name).argtypes = [P(_Net), vp, i64, i32, vp, vp, vp]
            getattr(_lib, name).restype = ctypes.c_int
        _lib.ctmo_weighted_laplacian.argtypes = [P(_Net), vp, i64, vp, i32, i32, vp, vp, vp]
        _lib.ctmo_randomized_laplacian.argtypes = [P(_Net), vp, i64, vp, i32, vp, i32, i32, vp, vp, vp]
        _lib.ctmo_forward.argtypes = [P(_Net), vp, i64, vp]
        _lib.ctmo_stochastic_biharmonic.argtypes = [P(_Net), vp, i64, vp, i32, i32, vp, vp, vp]
        _lib.ctmo_directional_sum.argtypes = [P(_Net), vp, i64, i32, i32, vp, i32, vp, i32, vp, vp, vp]
        _lib.ctmo_biharmonic_nested.argtypes = [P(_Net), vp, i64, vp, vp, vp]
        _lib.ctmo_act_derivs.argtypes = [i32, d, vp]
        _lib.ctmo_act_derivs.restype = None
        _lib.ctmo_gamma.argtypes = [i32, i32, i32, i32, P(ctypes.c_int64), P(ctypes.c_int64)]
        _lib.ctmo_biharmonic_set.argtypes = [i32, vp, vp]
        _lib.ctmo_biharmonic_set.restype = ctypes.c_int64
        _lib.ctmo_partition.argtypes = [i32, i32, vp, P(ctypes.c_int64)]
        _lib.ctmo_partition.restype = ctypes.c_int32
        _lib.ctmo_rademacher.argtypes = [ctypes.c_uint64, i64, i64, i32, i32, vp]
        _lib.ctmo_rademacher.restype = None
        _lib.ctmo_splitmix64.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        _lib.ctmo_splitmix64.restype = ctypes.c_uint64
        _lib.ctmo_num_threads.restype = ctypes.c_int32
        _lib.ctmo_set_num_threads.argtypes = [i32]
        _lib.ctmo_set_num_threads.restype = None
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Net:
    """MLP weights as fp64 arrays: Ws[l] is [w_{l+1}, w_l] (nn.Linear layout)."""

    Ws: list
    bs: list
    act: str = "tanh"

    def __post_init__(self):
        self.Ws = [_f64(W) for W in self.Ws]
        self.bs = [_f64(b).reshape(-1) for b in self.bs]
        self.widths = np.array([self.Ws[0].shape[1]] + [W.shape[0] for W in self.Ws], dtype=np.int32)
        self.params = np.concatenate([np.concatenate([W.reshape(-1), b]) for W, b in zip(self.Ws, self.bs)])
        self._c = _Net(
            len(self.Ws),
            self.widths.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            self.params.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            ACTS[self.act],
        )

    @property
    def D(self) -> int:
        return int(self.widths[0])

    def cref(self):
        return ctypes.byref(self._c)


def _call(fn, net: Net, X, *extra, route=O1):
    X = _f64(X)
    N = X.shape[0]
    op = np.empty(N)
    f = np.empty(N)
    norm = np.empty(N)
    rc = fn(net.cref(), _ptr(X), N, *extra, route, _ptr(op), _ptr(f), _ptr(norm))
    if rc != 0:
        raise ValueError(f"oracle call failed (rc={rc})")
    return op, f, norm


def laplacian(net: Net, X, route=O1):
    """Exact Laplacian (Eq. 8). Returns (op, f, norm)."""
    return _call(lib().ctmo_laplacian, net, X, route=route)


def weighted_laplacian(net: Net, X, sigma, route=O1):
    """<d^2 f, sigma sigma^T> (Eq. 10), sigma [D, R]."""
    sigma = _f64(sigma)
    return _call(lib().ctmo_weighted_laplacian, net, X, _ptr(sigma), sigma.shape[1], route=route)


def randomized_laplacian(net: Net, X, V, sigma=None, route=O1):
    """(1/S) sum_s <d^2 f, (sigma v_s)^2> with V [N, S, Rv] (Eq. 8/10 stochastic)."""
    V = _f64(V)
    S, Rv = V.shape[1], V.shape[2]
    sig = None if sigma is None else _f64(sigma)
    return _call(
        lib().ctmo_randomized_laplacian, net, X, _ptr(V), S, None if sig is None else _ptr(sig), Rv, route=route
    )


def biharmonic(net: Net, X, route=O1):
    """Exact biharmonic (Eq. 12) via the interpolation family (O1/O3) or T4 (O2)."""
    return _call(lib().ctmo_biharmonic, net, X, route=route)


def stochastic_biharmonic(net: Net, X, V, route=O1):
    """1/(3S) sum_s <d^4 f, v_s^4> with V [N, S, D] (Eq. 12 stochastic, unbiased scale, Q1)."""
    V = _f64(V)
    return _call(lib().ctmo_stochastic_biharmonic, net, X, _ptr(V), V.shape[1], route=route)


def directional_sum(net: Net, X, K: int, dirs, w, route=O1):
    """sum_j w_j <d^K f, u_j^K> (K = 2 or 4); dirs [J, D] shared or [N, J, D] per point."""
    dirs, w = _f64(dirs), _f64(w).reshape(-1)
    per_point = dirs.ndim == 3
    return _call(lib().ctmo_directional_sum, net, X, int(K), int(w.size), _ptr(dirs), int(per_point), _ptr(w),
                 route=route)


def weighted_laplacian_pointwise(net: Net, X, sigma_x, route=O1):
    """<d^2 f(x_n), sigma(x_n) sigma(x_n)^T> with sigma_x [N, D, R] (Eq. 10, sigma depending on x)."""
    sigma_x = _f64(sigma_x)
    U = np.ascontiguousarray(np.transpose(sigma_x, (0, 2, 1)))  # [N, R, D]: the columns s_r(x_n)
    return directional_sum(net, X, 2, U, np.ones(U.shape[1]), route)


def biharmonic_nested(net: Net, X):
    """Laplacian^2 f by nested collapsed Laplacians. Returns (op, f, lap)."""
    X = _f64(X)
    N = X.shape[0]
    op, f, lap = np.empty(N), np.empty(N), np.empty(N)
    if lib().ctmo_biharmonic_nested(net.cref(), _ptr(X), N, _ptr(op), _ptr(f), _ptr(lap)) != 0:
        raise ValueError("oracle call failed")
    return op, f, lap


def forward(net: Net, X) -> np.ndarray:
    X = _f64(X)
    f = np.empty(X.shape[0])
    if lib().ctmo_forward(net.cref(), _ptr(X), X.shape[0], _ptr(f)) != 0:
        raise ValueError("oracle forward failed")
    return f


def act_derivs(act: str, z: float) -> np.ndarray:
    d = np.empty(5)
    lib().ctmo_act_derivs(ACTS[act], float(z), _ptr(d))
    return d


def gamma(i, j) -> Fraction:
    n, d = ctypes.c_int64(), ctypes.c_int64()
    if lib().ctmo_gamma(i[0], i[1], j[0], j[1], ctypes.byref(n), ctypes.byref(d)) != 0:
        raise ValueError("bad multi-index")
    return Fraction(n.value, d.value)


def biharmonic_set(D: int):
    J = lib().ctmo_biharmonic_set(D, None, None)
    dirs = np.empty((J, D))
    coef = np.empty(J)
    lib().ctmo_biharmonic_set(D, _ptr(dirs), _ptr(coef))
    return dirs, coef


def partitions(k: int):
    """[(parts tuple, nu)] for the integer partitions of k (Eq. 3)."""
    out = []
    parts = np.zeros(16, dtype=np.int32)
    nu = ctypes.c_int64()
    p = 0
    while True:
        n = lib().ctmo_partition(k, p, _ptr(parts), ctypes.byref(nu))
        if n == 0:
            return out
        out.append((tuple(int(x) for x in parts[:n]), nu.value))
        p += 1


def rademacher(seed: int, point_offset: int, N: int, S: int, Rv: int) -> np.ndarray:
    V = np.empty((N, S, Rv))
    lib().ctmo_rademacher(seed, point_offset, N, S, Rv, _ptr(V))
    return V


def splitmix64(seed: int, idx: int) -> int:
    return int(lib().ctmo_splitmix64(seed, idx))


def num_threads() -> int:
    return int(lib().ctmo_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP threads of the oracle's loops over points (no arithmetic change)."""
    lib().ctmo_set_num_threads(int(n))
