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
