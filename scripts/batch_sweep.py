"""C1 batch sweep (BASELINE configs[1]: N = 128 ... 16384) on one GPU.

For every N: the exact Laplacian of the D=50 MLP through the C ABI, timed on the device
with CUDA events over K back-to-back calls (after W warm-up calls), both as eager launches
and as a CUDA-graph replay of one captured call (small N is launch-bound).
Inputs are resident in HBM; no L2 flush between calls (the small-N working sets are
L2-resident by nature, which is the regime this sweep describes). Prints one JSON object.

usage: python scripts/batch_sweep.py [--op laplacian] [--K 50] [--W 5]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_13644_b200 as ctm  # noqa: E402
from synth import mlp_params, points, widths_for  # noqa: E402

MFLOP = {"laplacian": 129.6e6, "biharmonic_nested": None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="laplacian", choices=["laplacian", "biharmonic", "biharmonic_nested"])
    ap.add_argument("--K", type=int, default=50)
    ap.add_argument("--W", type=int, default=5)
    args = ap.parse_args()
    D = 5 if "biharmonic" in args.op else 50
    widths = widths_for(D)
    params = mlp_params(widths, 0)
    mlp = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0)
    fn = getattr(mlp, args.op)
    rows = []
    for N in [128, 256, 512, 1024, 2048, 4096, 8192, 16384]:
        X = torch.from_numpy(points(N, D)).cuda()
        out = torch.empty(N, device="cuda")
        f = torch.empty(N, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(args.W):
                fn(X, out=out, f_out=f)
        torch.cuda.synchronize()
        plan = mlp.last_plan()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(s):
            ev[0].record(s)
            for _ in range(args.K):
                fn(X, out=out, f_out=f)
            ev[1].record(s)
        torch.cuda.synchronize()
        eager_ms = ev[0].elapsed_time(ev[1]) / args.K
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn(X, out=out, f_out=f)
        for _ in range(args.W):
            g.replay()
        torch.cuda.synchronize()
        ev[2].record()
        for _ in range(args.K):
            g.replay()
        ev[3].record()
        torch.cuda.synchronize()
        graph_ms = ev[2].elapsed_time(ev[3]) / args.K
        best = min(eager_ms, graph_ms)
        slots = plan["slots_per_point"] * plan["blocks"]
        tiles = -(-N * plan["blocks"] // plan["points_per_tile"])
        rows.append({"N": N, "eager_ms": eager_ms, "graph_ms": graph_ms,
                     "points_per_s_eager": N / eager_ms * 1e3, "points_per_s_graph": N / graph_ms * 1e3,
                     "useful_tflops": (MFLOP.get(args.op) or 0) * N / best * 1e3 / 1e12,
                     "launches": plan["launches"], "slots_per_point": slots, "n_tiles_per_layer_pair_grid": tiles})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    print(json.dumps({"op": args.op, "widths": widths, "K": args.K, "W": args.W,
                      "device": torch.cuda.get_device_name(0), "rows": rows}))
    mlp.close()


if __name__ == "__main__":
    main()
