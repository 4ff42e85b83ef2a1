import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2505_13644_b200 as ctm
from synth import mlp_params, points
from tests.test_gpu_grad import _gs, _k2
widths = [5, 64, 48, 1]; params = mlp_params(widths, 0); N = 13
for scale in (30.0, 10.0, 1.0):
  X = points(N, 5) * scale
  gop, gf = _gs(N)
  Ws = [W.astype(np.float64) for W, _ in params]; bs = [b.astype(np.float64) for _, b in params]
  dW, db, (MW, Mb) = _k2(Ws, bs, X.astype(np.float64), np.eye(5), np.ones(5), gop, gf)
  for prec in ("fp32", "fp16x3"):
    m = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0, precision=prec)
    m.grad_enable(); m.laplacian(torch.from_numpy(X).cuda())
    g = m.backward(torch.from_numpy(gop).cuda(), torch.from_numpy(gf).cuda())
    gW = g[0][0].double().cpu().numpy(); M = np.asarray(MW[0]).reshape(gW.shape)
    rel = np.abs(gW - dW[0]) / np.maximum(M, 1e-300)
    i = np.unravel_index(np.argmax(rel), rel.shape)
    print(scale, prec, m.last_precision(), "W0 elem max", rel.max(), "at", i, "M_i/maxM", M[i] / M.max(), "g", gW[i], "ref", dW[0][i], "tensor", np.abs(gW-dW[0]).max()/np.abs(dW[0]).max())
    m.close()
