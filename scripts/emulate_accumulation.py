"""Numerics emulation: why the GPU C1 error is ~2.5e-5.

Emulates the collapsed Laplacian of the C1 net (50-768-768-512-512-1) in numpy with
3xTF32 products and three models of the tensor-core fp32 accumulation per MMA
instruction (K=8): exact (fp64), round-to-nearest, round-toward-zero; prints the
max normalised error vs the fp64 oracle. Analysis tool (imports oracle/), not
part of the product. See DESIGN.md §5.
"""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import oracle as O
from synth import mlp_params, points, widths_for
params = mlp_params(widths_for(50), 0)
net = O.Net([W.astype(np.float64) for W,_ in params],[b.astype(np.float64) for _,b in params])
X = points(203, 50)
idx = np.arange(0,203,7)
X = X[idx]
want,_,norm = O.laplacian(net, X.astype(np.float64), O.O1)

def tf32_rna(x):
    x = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((x + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return r.view(np.float32)
def tf32_trunc(x):
    x = np.asarray(x, np.float32).view(np.uint32)
    return (x & np.uint32(0xFFFFE000)).view(np.float32)
def rz32(x):  # round toward zero to fp32 from float64
    f = x.astype(np.float32)
    over = np.abs(f.astype(np.float64)) > np.abs(x)
    f[over] = np.nextafter(f[over], np.float32(0))
    return f

def gemm(Bh, Bl, Wh, Wl, mode):
    # Z[slot, feat] = sum_k B[slot,k] W[feat,k], 3xTF32 products, accumulate per 8-K MMA
    K = Bh.shape[1]
    acc = np.zeros((Bh.shape[0], Wh.shape[0]), np.float32)
    bl = tf32_trunc(Bl); wl = tf32_trunc(Wl)
    for k0 in range(0, K, 8):
        sl = slice(k0, k0+8)
        for (a, b) in ((bl, Wh), (Bh, wl), (Bh, Wh)):
            s = a[:, sl].astype(np.float64) @ b[:, sl].astype(np.float64).T
            t = acc.astype(np.float64) + s
            acc = t.astype(np.float32) if mode == 'rn' else rz32(t)
    return acc

def run(mode):
    W1,b1 = params[0]
    outs=[]
    for x in X:
        z0 = (W1 @ x + b1).astype(np.float32)
        t = np.tanh(z0); d1 = 1-t*t; d2 = -2*t*d1
        U = W1.T  # [D, 768]
        blk = np.concatenate([t[None], d1[None]*U, (d2*(U**2).sum(0))[None]]).astype(np.float32)
        for l in (1,2,3):
            W,b = params[l]
            if mode == 'fp64':
                Z = blk.astype(np.float64) @ W.astype(np.float64).T
            else:
                Bh = tf32_rna(blk); Bl = (blk - Bh).astype(np.float32)
                Wh = tf32_rna(W); Wl = (W - Wh).astype(np.float32)
                Z = gemm(Bh, Bl, Wh, Wl, mode).astype(np.float64)
            z0 = Z[0] + b; t = np.tanh(z0); d1 = 1-t*t; d2 = -2*t*d1
            z1 = Z[1:-1]; top = d1*Z[-1] + d2*(z1**2).sum(0)
            blk = np.concatenate([t[None], d1[None]*z1, top[None]]).astype(np.float32)
        w5,b5 = params[4]
        outs.append(float(w5[0].astype(np.float64) @ blk[-1].astype(np.float64)))
    e = np.abs(np.array(outs)-want)/norm
    print(mode, e.max(), np.median(e))
for m in ('fp64','rn','rz'): run(m)
