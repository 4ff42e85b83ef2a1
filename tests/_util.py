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


def magnitude_k2(Ws, bs, X, dirs, coef):
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
            t = np.tanh(z0)
            d1 = 1.0 - t * t
            d2 = -2.0 * t * d1
            h0, A1, A2 = t, np.abs(d1) * Z1, np.abs(d2) * Z1 ** 2 + np.abs(d1) * Z2
        out[n] = float(c @ (A2 @ np.abs(Ws[-1][0])))
    return out
