"""Numerics emulation: operand-split schemes x tensor-core accumulation models.

Emulates the collapsed Laplacian of the C1 net (50-768-768-512-512-1) in numpy for
several ways of forming fp32-accurate products on bf16/tf32 tensor cores, with the
fp32 accumulator rounded toward zero after every MMA instruction (the model that
reproduces the measured GPU error). Prints the normalised error vs
the fp64 oracle (max, q99, median). Analysis tool (imports oracle/), not product.

    python scripts/emulate_schemes.py [npts]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from synth import mlp_params, points, widths_for  # noqa: E402


def bf16_rn(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return r.astype(np.uint32).view(np.float32)


def tf32_rna(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x1000) & 0xFFFFE000).astype(np.uint32).view(np.float32)


def tf32_trunc(x):
    return (np.asarray(x, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def rz32(x):
    f = x.astype(np.float32)
    over = np.abs(f.astype(np.float64)) > np.abs(x)
    f[over] = np.nextafter(f[over], np.float32(0))
    return f


def fp16_rn(x):
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)


def split(x, planes, kind):
    out = []
    r = np.asarray(x, np.float32)
    for _ in range(planes):
        h = bf16_rn(r) if kind == "bf16" else fp16_rn(r) if kind == "fp16" else tf32_rna(r)
        out.append(h)
        r = (r - h).astype(np.float32)
    if kind == "tf32":
        out = [out[0]] + [tf32_trunc(p) for p in out[1:]]
    return out


# scheme: (kind, planes, [(i, j, acc)]) - product A_i * B_j goes to accumulator acc,
# listed in issue order within a K step.
SCHEMES = {
    "bf16x3 (hi/lo, 3 products, 1 acc) [r1]": ("bf16", 2, [(1, 0, 0), (0, 1, 0), (0, 0, 0)]),
    "bf16x3, 2 accs": ("bf16", 2, [(1, 0, 1), (0, 1, 1), (0, 0, 0)]),
    "tf32x3 (1 acc)": ("tf32", 2, [(1, 0, 0), (0, 1, 0), (0, 0, 0)]),
    "tf32x3, 2 accs": ("tf32", 2, [(1, 0, 1), (0, 1, 1), (0, 0, 0)]),
    "bf16x6 (3 planes, 1 acc)": ("bf16", 3, [(2, 0, 0), (1, 1, 0), (0, 2, 0), (1, 0, 0), (0, 1, 0), (0, 0, 0)]),
    "bf16x6, 2 accs": ("bf16", 3, [(2, 0, 1), (1, 1, 1), (0, 2, 1), (1, 0, 1), (0, 1, 1), (0, 0, 0)]),
    "bf16x5 (no mid*mid), 2 accs": ("bf16", 3, [(2, 0, 1), (0, 2, 1), (1, 0, 1), (0, 1, 1), (0, 0, 0)]),
    # one accumulator, two phases over the whole K: the five correction products first, then hi*hi
    "bf16x6 two-phase (1 acc)": ("bf16", 3, [(2, 0, 0), (1, 1, 0), (0, 2, 0), (1, 0, 0), (0, 1, 0), "phase", (0, 0, 0)]),
    # fp16 hi/lo planes with power-of-two scales: A per output row (from max |W[m, :]|), B per
    # slot type of the block (primal / first order / top, from the block's max |value| of
    # that type: FP16_BOUND = "max" uses the actual max, "bound" a one-layer bound)
    "fp16x3 two-phase, scaled (1 acc)": ("fp16", 2, [(1, 0, 0), (0, 1, 0), "phase", (0, 0, 0)]),
    "fp16x3 two-phase, unscaled (1 acc)": ("fp16u", 2, [(1, 0, 0), (0, 1, 0), "phase", (0, 0, 0)]),
    # candidates for less operand traffic: the corrections and the main product per K step
    # (one group of slots per K block), or the two phases per K CHUNK (phase 2 re-reading the
    # chunk's resident p0 tiles): the 4th entry is the chunk length in K
    "fp16x3 interleaved, scaled (1 acc)": ("fp16", 2, [(1, 0, 0), (0, 1, 0), (0, 0, 0)]),
    "fp16x3 two-phase per 256-K chunk (1 acc)": ("fp16", 2, [(1, 0, 0), (0, 1, 0), "phase", (0, 0, 0)], 256),
    "fp16x3 two-phase per 128-K chunk (1 acc)": ("fp16", 2, [(1, 0, 0), (0, 1, 0), "phase", (0, 0, 0)], 128),
}


def pow2_scale(maxabs, target=14):
    """exponent e with maxabs * 2^e in [2^(target-1), 2^target] (0 for an all-zero set)"""
    m = np.asarray(maxabs, np.float64)
    e = np.where(m > 0, target - np.ceil(np.log2(np.where(m > 0, m, 1.0))), 0.0)
    return e


def gemm(blk, W, scheme, btype=None):
    kind, planes, prods = scheme[:3]
    chunk = scheme[3] if len(scheme) > 3 else blk.shape[1]
    kstep = 8 if kind == "tf32" else 16
    sa = sb = None
    if kind == "fp16":
        sa = pow2_scale(np.abs(W).max(1))                       # per output row
        sb = np.zeros(blk.shape[0])
        for t in np.unique(btype):                              # per slot type of the block
            sel = btype == t
            sb[sel] = pow2_scale(np.abs(blk[sel]).max())
        B = split(blk * np.exp2(sb)[:, None], planes, "fp16")
        A = split(W * np.exp2(sa)[:, None], planes, "fp16")
    elif kind == "fp16u":
        B = split(blk, planes, "fp16")
        A = split(W, planes, "fp16")
    else:
        B = split(blk, planes, kind)
        A = split(W, planes, kind)
    accs = [np.zeros((blk.shape[0], W.shape[0]), np.float32) for _ in range(2)]
    phases = [prods]
    if "phase" in prods:
        i = prods.index("phase")
        phases = [prods[:i], prods[i + 1:]]
    for c0 in range(0, blk.shape[1], chunk):
        for ph in phases:
            for k0 in range(c0, min(c0 + chunk, blk.shape[1]), kstep):
                sl = slice(k0, k0 + kstep)
                for i, j, a in ph:
                    s = B[j][:, sl].astype(np.float64) @ A[i][:, sl].astype(np.float64).T
                    accs[a] = rz32(accs[a].astype(np.float64) + s)
    Z = accs[0].astype(np.float64) + accs[1].astype(np.float64)
    if sa is not None:
        Z = (Z * np.exp2(-sb)[:, None] * np.exp2(-sa)[None, :]).astype(np.float32).astype(np.float64)
    return Z


def run(params, X, want, norm, scheme):
    W1, b1 = params[0]
    P = X.shape[1] + 2
    n = X.shape[0]
    z0 = (X.astype(np.float64) @ W1.T.astype(np.float64) + b1).astype(np.float32)
    t = np.tanh(z0); d1 = 1 - t * t; d2 = -2 * t * d1
    U = W1.T.astype(np.float32)
    blk = np.empty((n, P, W1.shape[0]), np.float32)
    blk[:, 0] = t
    blk[:, 1:-1] = d1[:, None, :] * U[None]
    blk[:, -1] = d2 * (U.astype(np.float64) ** 2).sum(0)
    for l in (1, 2, 3):
        W, b = params[l]
        if scheme is None:
            Z = blk.reshape(n * P, -1).astype(np.float64) @ W.astype(np.float64).T
        else:
            btype = np.tile(np.r_[0, np.ones(P - 2), 2], n)
            Z = gemm(blk.reshape(n * P, -1), W, scheme, btype)
        Z = Z.reshape(n, P, -1)
        z0 = Z[:, 0] + b; t = np.tanh(z0); d1 = 1 - t * t; d2 = -2 * t * d1
        z1 = Z[:, 1:-1]
        top = d1 * Z[:, -1] + d2 * (z1 ** 2).sum(1)
        blk = np.empty((n, P, W.shape[0]), np.float32)
        blk[:, 0] = t; blk[:, 1:-1] = d1[:, None] * z1; blk[:, -1] = top
    w5 = params[4][0][0].astype(np.float64)
    out = blk[:, -1].astype(np.float64) @ w5
    e = np.abs(out - want) / norm
    return e


def main():
    npts = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    params = mlp_params(widths_for(50), 0)
    net = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params])
    X = points(npts, 50, seed=11)
    want, _, norm = O.laplacian(net, X.astype(np.float64), O.O1)
    e = run(params, X, want, norm, None)
    print(f"{'fp64 products':40s} max {e.max():.2e}")
    only = sys.argv[2:] 
    for name, sch in SCHEMES.items():
        if only and not any(o in name for o in only):
            continue
        e = run(params, X, want, norm, sch)
        print(f"{name:40s} max {e.max():.2e}  q90 {np.quantile(e, 0.9):.2e}  median {np.median(e):.2e}", flush=True)


if __name__ == "__main__":
    main()
