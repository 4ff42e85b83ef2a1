"""BASELINE configs[0]: the exact Laplacian of the tanh MLP 5->16->16->1 at N = 8 points,
by the fp64 CPU oracle's three routes (O1 vanilla Taylor, O2 explicit Hessian, O3 collapsed;
SURVEY §8(c)) -- wall seconds, their mutual agreement and, when a GPU is present, the GPU
parity at the same inputs. Test infrastructure (calls oracle/). Prints one JSON object."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from synth import mlp_params, points  # noqa: E402


def main():
    widths = [5, 16, 16, 1]
    params = mlp_params(widths, 0)
    net = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params])
    X = points(8, 5).astype(np.float64)
    res = {"config": "C0: exact Laplacian, tanh MLP 5->16->16->1, N=8", "threads": O.num_threads(), "routes": {}}
    vals = {}
    for name, route in (("O1_vanilla", O.O1), ("O2_hessian", O.O2), ("O3_collapsed", O.O3)):
        reps, t0 = 0, time.perf_counter()
        while True:
            op, f, norm = O.laplacian(net, X, route)
            reps += 1
            if time.perf_counter() - t0 > 0.5:
                break
        dt = (time.perf_counter() - t0) / reps
        vals[name] = op
        res["routes"][name] = {"seconds_per_call": dt, "reps": reps}
    _, _, norm = O.laplacian(net, X, O.O1)
    res["agreement"] = {k: float(np.max(np.abs(v - vals["O1_vanilla"]) / norm)) for k, v in vals.items()}
    try:
        import torch

        if torch.cuda.is_available():
            import paper_2505_13644_b200 as ctm

            mlp = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0)
            op, f = mlp.laplacian(torch.from_numpy(X.astype(np.float32)).cuda())
            torch.cuda.synchronize()
            res["gpu_parity_max_norm_err"] = float(np.max(np.abs(op.double().cpu().numpy() - vals["O1_vanilla"]) / norm))
            mlp.close()
    except Exception as e:  # noqa: BLE001
        res["gpu"] = f"not run: {e}"
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
