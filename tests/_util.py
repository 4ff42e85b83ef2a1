"""Shared helpers for the tests (fixtures parsing, small random nets)."""
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def golden(name):
    """Parse a tests/golden/*.txt fixture: '|'-separated rows, '#' comments."""
    rows = []
    with open(os.path.join(ROOT, "tests", "golden", name)) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append([c.strip() for c in line.split("|")])
    return rows


def random_params(widths, seed, scale=1.0):
    """fp64 (W, b) list, U(+-scale/sqrt(fan_in))."""
    rng = np.random.default_rng(seed)
    Ws, bs = [], []
    for fi, fo in zip(widths[:-1], widths[1:]):
        bound = scale / np.sqrt(fi)
        Ws.append(rng.uniform(-bound, bound, size=(fo, fi)))
        bs.append(rng.uniform(-bound, bound, size=(fo,)))
    return Ws, bs


def rel_err(a, b, norm):
    return np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.asarray(norm))


def _abs_derivs(act, z):
    """s and |s'|, |s''|, |s'''|, |s''''| of the activation at z (textbook derivatives)."""
    if act == "tanh":
        t = np.tanh(z)
        s = 1.0 - t * t
        return t, np.abs(s), np.abs(2 * t * s), np.abs(s * (6 * t * t - 2)), np.abs(8 * t * s * (2 - 3 * t * t))
    if act == "sin":
        sn, cs = np.abs(np.sin(z)), np.abs(np.cos(z))
        return np.sin(z), cs, sn, cs, sn
    raise ValueError(act)


def magnitude_k4(Ws, bs, X, dirs, coef, act="tanh"):
    """Running magnitude M of the fourth-order Taylor computation (K = 4), as magnitude_k2
    for K = 2: the vanilla per-jet rules (Eq. 3 with K = 4, the rows of P:1370-1424)
        x1' = s1 x1,  x2' = s2 x1^2 + s1 x2,  x3' = s3 x1^3 + 3 s2 x1 x2 + s1 x3,
        x4' = s4 x1^4 + 6 s3 x1^2 x2 + 4 s2 x1 x3 + 3 s2 x2^2 + s1 x4     (sk = k-th derivative)
    with every quantity replaced by a bound of its absolute value, and
    M = sum_j |c_j| |w_out| A4_j. Ws/bs fp64; X [N, D]; dirs [J, D] or [N, J, D]; coef
    scalar or [J]. Test infrastructure only."""
    X = np.asarray(X, np.float64)
    dirs = np.asarray(dirs, np.float64)
    if dirs.ndim == 2:
        dirs = np.broadcast_to(dirs, (X.shape[0],) + dirs.shape)
    c = np.abs(np.broadcast_to(np.asarray(coef, np.float64), dirs.shape[1:2]))
    out = np.empty(X.shape[0])
    for n, x in enumerate(X):
        h0 = x
        A1 = np.abs(dirs[n])
        A2 = np.zeros_like(A1)
        A3 = np.zeros_like(A1)
        A4 = np.zeros_like(A1)
        for W, b in zip(Ws[:-1], bs[:-1]):
            aW = np.abs(W)
            z0 = W @ h0 + b
            Z1, Z2, Z3, Z4 = A1 @ aW.T, A2 @ aW.T, A3 @ aW.T, A4 @ aW.T
            h0, d1, d2, d3, d4 = _abs_derivs(act, z0)
            A1, A2, A3, A4 = (d1 * Z1, d2 * Z1**2 + d1 * Z2, d3 * Z1**3 + 3 * d2 * Z1 * Z2 + d1 * Z3,
                              d4 * Z1**4 + 6 * d3 * Z1**2 * Z2 + 4 * d2 * Z1 * Z3 + 3 * d2 * Z2**2 + d1 * Z4)
        out[n] = float(c @ (A4 @ np.abs(Ws[-1][0])))
    return out


def magnitude_k2(Ws, bs, X, dirs, coef, act="tanh"):
    """Running magnitude M of the second-order Taylor computation (K = 2, tanh).

    The same coefficient rules as the oracle's vanilla route (Eq. 3 with K = 2:
    x1' = s' x1,  x2' = s'' x1^2 + s' x2; Eq. 4 for the linear layers), with every
    quantity replaced by an upper bound of its absolute value:
        |z1| <= |W| A1,  |z2| <= |W| A2,  A1' = |s'| |z1|,  A2' = |s''| |z1|^2 + |s'| |z2|
    and M = sum_r |c_r| |w_out| A2_r. M bounds the sum of the absolute values of all
    products the computation forms (Higham's running error magnitude), so a
    faithful fp32-class evaluation has |error| <= (small constant) * u * M even where
    a direction's second derivative cancels internally — which the north_star
    normaliser sum_r |c_r f_{2,r}| cannot see (reading R9).

    Ws/bs: fp64 layers (nn.Linear layout); X [N, D]; dirs [R, D] shared or [N, R, D]
    per point; coef scalar or [R]. Test infrastructure only.
    """
    X = np.asarray(X, np.float64)
    dirs = np.asarray(dirs, np.float64)
    if dirs.ndim == 2:
        dirs = np.broadcast_to(dirs, (X.shape[0],) + dirs.shape)
    c = np.abs(np.broadcast_to(np.asarray(coef, np.float64), dirs.shape[1:2]))
    out = np.empty(X.shape[0])
    for n, x in enumerate(X):
        h0 = x
        A1 = np.abs(dirs[n])          # [R, D]
        A2 = np.zeros_like(A1)
        for W, b in zip(Ws[:-1], bs[:-1]):
            aW = np.abs(W)
            z0 = W @ h0 + b
            Z1, Z2 = A1 @ aW.T, A2 @ aW.T
            t, d1, d2, _, _ = _abs_derivs(act, z0)
            h0, A1, A2 = t, d1 * Z1, d2 * Z1 ** 2 + d1 * Z2
        out[n] = float(c @ (A2 @ np.abs(Ws[-1][0])))
    return out


def _derivs32(act, z):
    if act == "tanh":
        t = np.tanh(z)
        s = np.float32(1) - t * t
        return t, s, -2 * t * s, s * (6 * t * t - 2), 8 * t * s * (2 - 3 * t * t)
    if act == "sin":
        sn, cs = np.sin(z), np.cos(z)
        return sn, cs, -sn, -cs, sn
    raise ValueError(act)


def vanilla32(params, act, X, dirs, coef, K):
    """sum_j coef_j <d^K f(x), u_j^K> by PLAIN fp32 arithmetic: the vanilla Taylor rules (Eq. 3
    with K = 2 or 4, one jet per direction, the rows of P:1370-1424) in numpy float32 end to
    end (BLAS sgemm for the linear layers). The reference for "what plain fp32 gets" at a
    point (reading R9). params: the fp32 (W, b) list; X [n, D]; dirs [J, D] or
    [n, J, D]; coef scalar or [J]. Test infrastructure only."""
    X = np.asarray(X, np.float32)
    dirs = np.asarray(dirs, np.float32)
    if dirs.ndim == 2:
        dirs = np.broadcast_to(dirs, (X.shape[0],) + dirs.shape)
    coef = np.broadcast_to(np.asarray(coef, np.float32), dirs.shape[1:2])
    out = np.empty(X.shape[0])
    for n in range(X.shape[0]):
        h0 = X[n]
        x = [dirs[n].copy()] + [np.zeros_like(dirs[n]) for _ in range(K - 1)]
        for W, b in params[:-1]:
            z0 = W @ h0 + b
            z = [xi @ W.T for xi in x]
            h0, s1, s2, s3, s4 = _derivs32(act, z0)
            if K == 2:
                x = [s1 * z[0], s2 * z[0] * z[0] + s1 * z[1]]
            else:
                z1, z2, z3, z4 = z
                x = [s1 * z1, s2 * z1 * z1 + s1 * z2, s3 * z1 * z1 * z1 + 3 * s2 * z1 * z2 + s1 * z3,
                     s4 * z1**4 + 6 * s3 * z1 * z1 * z2 + 4 * s2 * z1 * z3 + 3 * s2 * z2 * z2 + s1 * z4]
        out[n] = float(np.float32(coef @ (x[-1] @ params[-1][0][0])))
    return out


def ref32(params, X, dirs, coef, K, act="tanh"):
    """A closure idx -> plain-fp32 values at points idx (vanilla32), for check()'s R9 rule."""
    def f(idx):
        d = np.asarray(dirs)
        return vanilla32(params, act, np.asarray(X)[idx], d[idx] if d.ndim == 3 else d, coef, K)
    return f
