#!/usr/bin/env python
"""bench.py — collapsed-Taylor Laplacian throughput on B200 (BASELINE.json metric).

One step = one full pass of the hot path (seed + layer 1,
the three fused tcgen05 layers, readout) over one batch of synthetic points:
config C1 = exact Laplacian of the tanh MLP 50-768-768-512-512-1 on
N = 16384 points per GPU (weak scaling: every rank processes its own batch;
points shard with no collective in the step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0. Timing: W untimed warm-up steps; then K steps,
each bracketed by CUDA events on the launch stream, with an L2 flush (256 MiB
write) between steps outside the events; barrier + synchronize around the timed
loop; the max over ranks. `roofline` comes from per-kernel events recorded by
the library on the same stream during the timed steps (ctm_profile_*).
`--impl reference` times the fp64 CPU oracle (oracle/, test infrastructure) on
bounded samples of the same workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "collapsed-Taylor Laplacian points/s, D=50 MLP, 1/2/4/8 B200; % TC peak"
# The paper's own per-datum times for the same workload on its hardware (context):
# P:1205 collapsed Taylor 0.33 ms/datum, standard Taylor 0.60 ms/datum (exact Laplacian, D=50 MLP,
# RTX 6000, PyTorch). No other operator has a published absolute number.
PAPER_PTS_PER_S = {"laplacian": 1.0 / 0.33e-3, "standard": 1.0 / 0.60e-3}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=16384, help="points per GPU")
    ap.add_argument("--op", choices=["laplacian", "weighted", "randomized", "biharmonic", "standard",
                                   "stochastic_biharmonic", "biharmonic_nested", "biharmonic_standard", "randomized_standard",
                                   "stochastic_biharmonic_standard", "laplacian_train"],
                    default="laplacian")
    ap.add_argument("--S", type=int, default=8, help="samples for --op randomized")
    ap.add_argument("--direction-block", type=int, default=0,
                    help="directions per block (ctm_set_direction_block); 0 = the library's planner")
    ap.add_argument("--precision", choices=["fp32", "bf16x3"], default="fp32",
                    help="layer-contraction arithmetic (ctm_set_precision, DESIGN.md §5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: total CPU seconds spread over the warm-up + timed steps")
    return ap.parse_args()


def workload(args):
    from synth import widths_for

    D = 5 if args.op in ("biharmonic", "stochastic_biharmonic", "biharmonic_nested", "biharmonic_standard",
                         "stochastic_biharmonic_standard") else 50
    names = {
        "laplacian": "C1 exact Laplacian",
        "laplacian_train": ("C1 PINN training step: exact Laplacian forward (grad mode) + loss cotangent + "
                            "ctm_backward + gradient all-reduce (N>1) + SGD update via ctm_set_weights"),
        "standard": "C1 exact Laplacian by STANDARD Taylor mode (1+2D vectors; the paper's baseline)",
        "weighted": "C2 weighted Laplacian (dense full-rank sigma, R=50)",
        "randomized": f"C3 randomized Laplacian (Rademacher, S={args.S}, generated in-kernel)",
        "biharmonic": "C4 exact biharmonic (interpolation family, J=35)",
        "biharmonic_nested": "C4 exact biharmonic by nested collapsed Laplacians (P:4073; 27 vectors)",
        "biharmonic_standard": "C4 exact biharmonic by STANDARD 4th-order Taylor mode (1+4J = 141 vectors; the paper's baseline)",
        "stochastic_biharmonic": f"stochastic biharmonic (Gaussian, S={args.S}, generated in-kernel)",
        "randomized_standard": f"C3 randomized Laplacian by STANDARD Taylor mode (S={args.S}; 1+2S vectors, baseline)",
        "stochastic_biharmonic_standard": f"stochastic biharmonic by STANDARD Taylor mode (S={args.S}; 1+4S vectors, baseline)",
    }
    w = widths_for(D)
    return D, w, f"{names[args.op]}, tanh MLP {'-'.join(map(str, w[:-1]))}-1, N={args.n} points per GPU"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms (B200_PROFILING recipe)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in self.rows if num(r[0])]
        mx = [num(r[1]) for r in self.rows if num(r[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- CPU oracle
def oracle_rate(D, widths, op, S, budget_s, seed_pts=1):
    """Time the fp64 oracle (vanilla Taylor route O1, as it stands) on a bounded
    sample of the workload; returns (points/s, points, seconds, threads)."""
    import oracle as O
    from synth import mlp_params, points, sigma as make_sigma

    params = mlp_params(widths, 0)
    net = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params])
    sig = make_sigma(D, D, kind="dense").astype(np.float64)

    def run(X):
        if op in ("laplacian", "standard"):
            O.laplacian(net, X, O.O1)
        elif op == "laplacian_train":
            from oracle import grad as OG
            OG.k2_grad(net.Ws, net.bs, X, np.eye(D), np.ones(D), np.ones(X.shape[0]) / X.shape[0])
        elif op == "weighted":
            O.weighted_laplacian(net, X, sig, O.O1)
        elif op in ("randomized", "randomized_standard"):
            O.randomized_laplacian(net, X, O.rademacher(2, 0, X.shape[0], S, D), route=O.O1)
        elif op in ("stochastic_biharmonic", "stochastic_biharmonic_standard"):
            V = np.random.default_rng(2).standard_normal((X.shape[0], S, D))
            O.stochastic_biharmonic(net, X, V, O.O1)
        elif op == "biharmonic_nested":
            O.biharmonic_nested(net, X)
        else:
            O.biharmonic(net, X, O.O1)

    nthr = O.num_threads()
    Xall = points(4096, D, seed_pts).astype(np.float64)
    m = max(nthr, 8)
    t0 = time.perf_counter()
    run(Xall[:m])
    dt = time.perf_counter() - t0
    rate = m / dt
    M = int(min(4096, max(m, rate * budget_s)))
    t0 = time.perf_counter()
    run(Xall[:M])
    dt = time.perf_counter() - t0
    return M / dt, M, dt, nthr


def reference_arm(args, rank):
    if rank != 0:
        return
    # rank 0 runs alone (the other ranks exit without work): give the oracle every host
    # core, as at N = 1 (torchrun exports OMP_NUM_THREADS=1 to each rank)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import oracle as O

        O.set_num_threads(os.cpu_count() or 1)
    D, widths, wl = workload(args)
    per_step = []
    total_pts = 0
    nthr = None
    budget = max(1.0, args.ref_budget_s / max(1, args.steps + args.warmup))
    for i in range(args.warmup + args.steps):
        rate, M, dt, nthr = oracle_rate(D, widths, args.op, args.S, budget)
        if i >= args.warmup:
            per_step.append(dt)
            total_pts += M
    value = total_pts / sum(per_step)
    sample = f"{total_pts // args.steps} points per step of the {wl.split(',')[0]} workload (fp64 oracle, vanilla Taylor route O1)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(per_step) / len(per_step),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl, "parallelism": "host cores (OpenMP)"},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": nthr, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2505_13644_b200 as ctm
    from synth import mlp_params, points, sigma as make_sigma

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    D, widths, wl = workload(args)
    N = args.n
    params = mlp_params(widths, 0)
    mlp = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=local)
    mlp.set_direction_block(args.direction_block)
    mlp.set_precision(args.precision)
    prods = 6 if args.precision == "fp32" else 3  # bf16 tensor products per useful product
    # each rank: its own contiguous slice of the global point set (global index rank*N ...)
    X_host = points(N * world, D, 1)[rank * N:(rank + 1) * N]
    X = torch.from_numpy(X_host).to(dev)
    sig = torch.from_numpy(make_sigma(D, D, kind="dense")).to(dev)
    op_out = torch.empty(N, device=dev)
    f_out = torch.empty(N, device=dev)
    train = args.op == "laplacian_train"
    if train:
        from paper_2505_13644_b200.dist import allreduce_grads

        mlp.grad_enable()
        pdev = [(torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)) for W, b in params]
        grads = [(torch.empty_like(W), torch.empty_like(b)) for W, b in pdev]
        flat_p = [t for pair in pdev for t in pair]
        flat_g = [t for pair in grads for t in pair]
        # Poisson-type residual: Laplacian f(x) - g(x), g = sum_d sin(pi x_d) (synthetic source)
        target = torch.sin(torch.pi * X).sum(1)
        res = torch.empty(N, device=dev)
        n_glob = N * world
        launches = {}

    def train_step(Xd, op_out=op_out, f_out=f_out):
        mlp.laplacian(Xd, out=op_out, f_out=f_out)
        launches["fwd"] = mlp.last_plan()["launches"]
        torch.sub(op_out, target, out=res)
        res.mul_(2.0 / n_glob)  # d/d op_n of mean_n (op_n - g_n)^2
        mlp.backward(res, grads=grads)
        launches["bwd"] = mlp.last_plan()["launches"]
        if world > 1:
            allreduce_grads(grads)
        torch._foreach_add_(flat_p, flat_g, alpha=-1e-4)
        mlp.set_weights(pdev)
        launches["upd"] = mlp.last_plan()["launches"]

    def step(Xd, op_out=op_out, f_out=f_out):
        if train:
            train_step(Xd, op_out, f_out)
        elif args.op == "laplacian":
            mlp.laplacian(Xd, out=op_out, f_out=f_out)
        elif args.op == "standard":
            mlp.laplacian_standard(Xd, out=op_out, f_out=f_out)
        elif args.op == "weighted":
            mlp.weighted_laplacian(Xd, sig, out=op_out, f_out=f_out)
        elif args.op == "randomized":
            mlp.randomized_laplacian(Xd, S=args.S, seed=2, point_offset=rank * N, out=op_out, f_out=f_out)
        elif args.op == "stochastic_biharmonic":
            mlp.stochastic_biharmonic(Xd, S=args.S, seed=2, point_offset=rank * N, out=op_out, f_out=f_out)
        elif args.op == "biharmonic_nested":
            mlp.biharmonic_nested(Xd, out=op_out, f_out=f_out)
        elif args.op == "biharmonic_standard":
            mlp.biharmonic_standard(Xd, out=op_out, f_out=f_out)
        elif args.op == "randomized_standard":
            mlp.randomized_laplacian(Xd, S=args.S, seed=2, point_offset=rank * N, out=op_out, f_out=f_out,
                                     standard=True)
        elif args.op == "stochastic_biharmonic_standard":
            mlp.stochastic_biharmonic(Xd, S=args.S, seed=2, point_offset=rank * N, out=op_out, f_out=f_out,
                                      standard=True)
        else:
            mlp.biharmonic(Xd, out=op_out, f_out=f_out)

    flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(3, args.warmup)):
        step(X)
    torch.cuda.synchronize()
    if train:
        mlp.laplacian(X, out=op_out, f_out=f_out)  # plan of the forward
    plan = mlp.last_plan()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    # ---------------- device-resident timed loop
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    mlp.profile(True)
    for a, b in evs:
        flush_buf.zero_()
        a.record()
        step(X)
        b.record()
    torch.cuda.synchronize()
    barrier()
    prof = mlp.profile_read()
    mlp.profile(False)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = max_over_ranks(sum(step_ms))
    best_ms = max_over_ranks(min(step_ms))      # the paper's protocol: best of the repetitions
    median_ms = max_over_ranks(float(np.median(step_ms)))

    # ---------------- end to end, pipelined: every step uploads its inputs from pinned host
    # memory on a copy stream, runs the operator on the compute stream and downloads its
    # results to pinned host memory on a third stream; two buffer sets let step i+1's upload
    # and step i-1's download overlap step i's kernels (each step's bytes still cross PCIe
    # inside the timed region). No L2 flush: the step's working set is > 10 GB >> L2.
    Xh = torch.from_numpy(X_host.copy()).pin_memory()
    ohs = [torch.empty(N, dtype=torch.float32).pin_memory() for _ in range(2)]
    fhs = [torch.empty(N, dtype=torch.float32).pin_memory() for _ in range(2)]
    Xds = [torch.empty_like(X) for _ in range(2)]
    outs = [(torch.empty(N, device=dev), torch.empty(N, device=dev)) for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    comp = torch.cuda.current_stream(dev)

    def e2e_run(nsteps, t0=None, t1=None):
        done, downloaded = [], []
        if t0 is not None:
            t0.record(s_in)
        for i in range(nsteps):
            b = i % 2
            with torch.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(done[i - 2])          # step i-2 no longer reads Xds[b]
                Xds[b].copy_(Xh, non_blocking=True)
                up = torch.cuda.Event()
                up.record(s_in)
            comp.wait_event(up)
            if i >= 2:
                comp.wait_event(downloaded[i - 2])        # outs[b] of step i-2 is on the host
            step(Xds[b], outs[b][0], outs[b][1])
            e = torch.cuda.Event()
            e.record(comp)
            done.append(e)
            with torch.cuda.stream(s_out):
                s_out.wait_event(e)
                ohs[b].copy_(outs[b][0], non_blocking=True)
                fhs[b].copy_(outs[b][1], non_blocking=True)
                d = torch.cuda.Event()
                d.record(s_out)
                downloaded.append(d)
        if t1 is not None:
            s_out.wait_event(done[-1])
            t1.record(s_out)
        torch.cuda.synchronize()
        return (nsteps - 1) % 2

    e2e_run(2)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    last = e2e_run(args.steps, t0, t1)
    barrier()
    e2e_ms = max_over_ranks(t0.elapsed_time(t1))
    oh = ohs[last]

    clk = clocks.stop()

    # sanity: the e2e result equals the device-resident one bit for bit (the training step
    # updates the weights every step, so its results move on)
    if not train:
        assert torch.equal(oh, op_out.cpu()), "e2e result differs from the device-resident run"

    value = N * world * args.steps / (total_ms / 1e3)
    e2e_value = N * world * args.steps / (e2e_ms / 1e3)

    # roofline of the dominant kernel (the fused tcgen05 layer kernel)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh_:
            peaks = json.load(fh_)
        peak_src = "measured"
    except OSError:
        peak_src = "fallback"
    bf16_sust = peaks.get("bf16_tflops_sustained", 1400.0)
    tensor_peak = bf16_sust                # the layer MMAs are kind::f16 with bf16 operands
    useful_peak = tensor_peak / prods      # bf16 tensor products per useful fp32-accurate product
    dom = max(("layer", "bwd", "wgrad"), key=lambda k: prof[k]["ms"]) if train else "layer"
    lay = prof[dom]
    achieved = lay["work"] / (lay["ms"] / 1e3) / 1e12 if lay["ms"] > 0 else None
    kernel_name = {
        "layer": "jet_layer_kernel (layers 2-4: tcgen05 3xBF16 GEMM + tanh Taylor epilogue)",
        "bwd": "jet_layer_kernel<kBwd2> (adjoint layers: tcgen05 3xBF16 W^T GEMM + transposed Taylor rule)",
        "wgrad": "weight-gradient GEMMs Z_bar^T B (cuBLAS, 3 bf16 GEMMs per layer, fp32 accumulate)",
    }[dom]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "layer_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh_:
            tj = json.load(fh_)
        key = f"{args.op}_S{args.S}" if args.op == "randomized" else args.op
        traffic = tj.get(key, {}).get("dram_bytes_per_launch")
    roofline = {
        "bound": "tensor", "achieved": achieved, "peak": useful_peak, "unit": "TFLOP/s",
        "frac": (achieved / useful_peak) if achieved else None, "traffic": traffic,
        "kernel": kernel_name,
        "peak_basis": (f"{peak_src} bf16 sustained {bf16_sust} TF/s / {prods} (bf16 tensor "
                       "products per useful product)"),
        "tensor_pipe_frac": (prods * achieved / tensor_peak) if achieved else None,
        # context: the same against the burst bf16 rate (cuBLAS timed alone at full clocks);
        # the sustained peak above was measured with the clocks the power cap allows, so a
        # step that keeps 1965 MHz can exceed 1.0 against it
        "frac_vs_burst": (prods * achieved / peaks["bf16_tflops"]) if achieved and "bf16_tflops" in peaks else None,
        "layer_ms_share": lay["ms"] / sum(step_ms) if sum(step_ms) > 0 else None,
        "kernel_ms_per_step": {k: v["ms"] / args.steps for k, v in prof.items()},
        "launches_per_step": {k: v["launches"] / args.steps for k, v in prof.items()},
    }
    # the HBM-bound stage: layer 1 written by the seed kernel (fixed direction sets; bytes
    # written = the layer-1 block, bf16 pairs) against the measured HBM bandwidth
    sd = prof["seed"]
    hbm = peaks.get("hbm_gbs", 6546.0)
    if sd["ms"] > 0 and sd["work"] > 0:
        gbs = sd["work"] / (sd["ms"] / 1e3) / 1e9
        roofline["seed_hbm"] = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                                "note": "algorithmic bytes written by the seed kernel per its event time; the peak "
                                        "is the measured copy (read+write) bandwidth"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, M, dt, nthr = oracle_rate(D, widths, args.op, args.S, budget_s=12.0)
        cpu = {"value": rate, "unit": "points/s", "cores": nthr, "kind": "oracle",
               "sample": f"{M} points of the same workload ({dt:.1f} s, fp64 vanilla-Taylor route O1, OpenMP)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "best_ms_per_step": best_ms, "median_ms_per_step": median_ms,
            "scaling": "weak",
            "vs_baseline": (value / PAPER_PTS_PER_S[args.op]) if args.op in PAPER_PTS_PER_S else None,
            "vs_baseline_ref": ("paper P:1205, marginal ms/datum on an RTX 6000, PyTorch (another machine: context)"
                                if args.op in PAPER_PTS_PER_S else "no published number for this operator"),
            "dtype": ("f32 (bf16x6: three bf16 planes per operand, six tensor products, fp32 accumulate)"
                      if args.precision == "fp32" else "f32 storage, bf16x3 products (~17-bit operands, fp32 accumulate)"),
            "data": "synthetic",
            "config": {"workload": wl, "op": args.op, "N_per_gpu": N, "D": D, "widths": widths,
                       "slots_per_point": plan["slots_per_point"], "points_per_tile": plan["points_per_tile"],
                       "mma_n": plan["mma_n"], "direction_blocks": plan["blocks"],
                       "directions_per_block": plan["per_block"],
                       "parallelism": (f"dp{world} (points sharded; gradient all-reduce, one 5 MB NCCL bucket)"
                                       if train else f"dp{world} (points sharded, no collective in step)"),
                       "l2": "flushed between timed steps (256 MiB write, outside the step events); "
                             "step working set > 10 GB >> L2"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": N * D * 4,
                    "d2h_bytes_per_step": 2 * N * 4},
            "clocks": clk,
            "gpu_launches": (sum(launches.values()) if train else plan["launches"]) * args.steps,
        }
        print(json.dumps(line), flush=True)
    mlp.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
