#!/usr/bin/env python
"""bench.py — collapsed-Taylor Laplacian throughput on B200 (BASELINE.json metric).

One step = one full pass of the hot path (seed + layer 1,
the three fused tcgen05 layers, readout) over one batch of synthetic points:
config C1 = exact Laplacian of the tanh MLP 50-768-768-512-512-1 on
N = 16384 points per GPU, in the fp16x3 mode: north_star's 3xTF32 operand split
(11 + 11 significant bits) on fp16 tensor cores, three products per useful product
(DESIGN.md §5); --precision fp32 times the library's default 24-bit mode (bf16x6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scaling weak|strong] [--precision fp32|fp16x3|bf16x3] [--op ...]
    torchrun --nproc-per-node N bench.py --gpus N ...

Scaling: "weak" (default) = every rank evaluates its own N points
(global indices rank*N ...), no collective in the step; "strong" = --n-total points split
by dist.shard over the ranks (global point_offset), timed without and with the NCCL
all_gather of op and f, and rank 0 checks the gathered result bitwise against its own
1-GPU evaluation of all --n-total points.

Prints ONE JSON line on rank 0. Timing: W untimed warm-up steps; then K steps,
each bracketed by CUDA events on the launch stream, with an L2 flush (256 MiB
write) between steps outside the events; barrier + synchronize around the timed
loop; the max over ranks. `roofline` comes from per-kernel events recorded by
the library on the same stream during the timed steps (ctm_profile_*); its peak is
the burst bf16 rate unless the timed region lasts >= 2 s (then the sustained one).
Clocks are sampled through NVML every 20 ms inside the timed region.
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
    ap.add_argument("--n", type=int, default=16384, help="points per GPU (weak scaling)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--n-total", type=int, default=16384, help="strong scaling: points over all ranks")
    ap.add_argument("--op", choices=["laplacian", "weighted", "randomized", "biharmonic", "standard",
                                   "stochastic_biharmonic", "biharmonic_nested", "biharmonic_standard", "randomized_standard",
                                   "stochastic_biharmonic_standard", "laplacian_train"],
                    default="laplacian")
    ap.add_argument("--S", type=int, default=8, help="samples for --op randomized")
    ap.add_argument("--direction-block", type=int, default=0,
                    help="directions per block (ctm_set_direction_block); 0 = the library's planner")
    ap.add_argument("--precision", choices=["fp32", "fp16x3", "bf16x3"], default="fp16x3",
                    help="layer-contraction arithmetic (ctm_set_precision, DESIGN.md §5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-precisions", action="store_true",
                    help="skip timing the operator in the other precision modes (the line's other_precisions)")
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
    npts = (f"N={args.n_total} points split over the GPUs" if args.scaling == "strong"
            else f"N={args.n} points per GPU")
    return D, w, f"{names[args.op]}, tanh MLP {'-'.join(map(str, w[:-1]))}-1, {npts}"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons through NVML every 20 ms on a thread (B200_PROFILING
    recipe's clocks line); `mark(tag)` records the wall time of the timed region's edges so
    the summary uses only samples inside [start, end]. Falls back to nvidia-smi -lms 20."""

    PERIOD = 0.02

    def __init__(self, index: int):
        self.index = index
        self.rows = []          # (t, sm_mhz, max_mhz, reasons set)
        self.marks = {}
        self._stop = threading.Event()
        self.t = None

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksThrottleReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def loop():
                while not self._stop.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        self.rows.append((time.perf_counter(), sm, mx, {k for k, v in bits.items() if r & v}))
                    except Exception:
                        pass
                    self._stop.wait(self.PERIOD)

            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
        except Exception:
            self.t = None

    def mark(self, tag):
        self.marks[tag] = time.perf_counter()

    def stop(self):
        self._stop.set()
        if self.t:
            self.t.join(timeout=2)
        t0, t1 = self.marks.get("start", 0.0), self.marks.get("end", float("inf"))
        rows = [r for r in self.rows if t0 <= r[0] <= t1] or self.rows
        sm = [r[1] for r in rows]
        reasons = sorted(set().union(*[r[3] for r in rows])) if rows else []
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(r[2] for r in rows) if rows else None,
                "sm_mhz_min": min(sm) if sm else None, "reasons": reasons, "samples": len(rows),
                "period_ms": 1e3 * self.PERIOD, "source": "nvml"}


# ----------------------------------------------------------------------------- CPU oracle
def oracle_rate(D, widths, op, S, budget_s, seed_pts=1, route=None):
    """Time the fp64 oracle (as it stands; vanilla Taylor route O1 unless `route`) on a
    bounded sample of the workload; returns (points/s, points, seconds, threads)."""
    import oracle as O
    from synth import mlp_params, points, sigma as make_sigma

    route = O.O1 if route is None else route
    params = mlp_params(widths, 0)
    net = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params])
    sig = make_sigma(D, D, kind="dense").astype(np.float64)

    def run(X):
        if op in ("laplacian", "standard"):
            O.laplacian(net, X, route)
        elif op == "laplacian_train":
            from oracle import grad as OG
            OG.k2_grad(net.Ws, net.bs, X, np.eye(D), np.ones(D), np.ones(X.shape[0]) / X.shape[0])
        elif op == "weighted":
            O.weighted_laplacian(net, X, sig, route)
        elif op in ("randomized", "randomized_standard"):
            O.randomized_laplacian(net, X, O.rademacher(2, 0, X.shape[0], S, D), route=route)
        elif op in ("stochastic_biharmonic", "stochastic_biharmonic_standard"):
            V = np.random.default_rng(2).standard_normal((X.shape[0], S, D))
            O.stochastic_biharmonic(net, X, V, route)
        elif op == "biharmonic_nested":
            O.biharmonic_nested(net, X)
        else:
            O.biharmonic(net, X, route)

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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(D, widths, op, S, flop_pt=None):
    """the oracle on the box's host cores: vanilla fp64 O1 (the headline
    cpu_baseline value) and collapsed fp64 O3 (the same schedule as the GPU) on all cores,
    O1 on one thread, with the CPU model; about 20 s of CPU work in all."""
    import oracle as O

    rate, M, dt, nthr = oracle_rate(D, widths, op, S, budget_s=8.0)
    out = {"value": rate, "unit": "points/s", "cores": nthr, "kind": "oracle",
           "sample": f"{M} points of the same workload ({dt:.1f} s, fp64 vanilla-Taylor route O1, OpenMP)",
           "cpu_model": cpu_model(), "logical_cpus": os.cpu_count()}
    if op not in ("laplacian_train", "biharmonic_nested"):
        r3, M3, dt3, _ = oracle_rate(D, widths, op, S, budget_s=5.0, route=O.O3)
        out["o3_collapsed"] = {"value": r3, "sample": f"{M3} points, {dt3:.1f} s, fp64 collapsed route O3, {nthr} threads"}
    O.set_num_threads(1)
    try:
        r1, M1, dt1, _ = oracle_rate(D, widths, op, S, budget_s=4.0)
    finally:
        O.set_num_threads(nthr)
    out["single_thread"] = {"value": r1, "sample": f"{M1} points, {dt1:.1f} s, O1, 1 thread"}
    if flop_pt:  # achieved fp64 GFLOP/s at the method's useful flop count per point
        out["useful_mflop_per_point"] = flop_pt / 1e6
        out["useful_gflops"] = rate * flop_pt / 1e9
        if "o3_collapsed" in out:
            out["o3_collapsed"]["useful_gflops"] = out["o3_collapsed"]["value"] * flop_pt / 1e9
        out["single_thread"]["useful_gflops"] = r1 * flop_pt / 1e9
    return out


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
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl, "parallelism": "host cores (OpenMP)"},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": nthr, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def write_ceiling_gbs(dev):
    """The device's measured write-only bandwidth: cudaMemsetAsync of 4 GiB (the CUDA
    runtime's own fill, through ctypes), best of 6, CUDA events on the current stream. The
    roofline peak of the HBM-write-bound seed kernel. (torch's zero_() fill kernel reaches
    less, so it would flatter the seed.)"""
    import ctypes
    import glob

    import torch

    libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                  "libcudart.so*"))
    cudart = ctypes.CDLL(libs[0] if libs else "libcudart.so")
    cudart.cudaMemsetAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p]
    nbytes = 4 << 30
    buf = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev)
    best = float("inf")
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        rc = cudart.cudaMemsetAsync(ctypes.c_void_p(buf.data_ptr()), 0, ctypes.c_size_t(nbytes),
                                    ctypes.c_void_p(st.cuda_stream))
        b.record(st)
        torch.cuda.synchronize()
        if rc != 0:
            raise RuntimeError(f"cudaMemsetAsync failed ({rc})")
        best = min(best, a.elapsed_time(b))
    del buf
    return nbytes / (best / 1e3) / 1e9


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return

    if world > 1:  # NCCL's init lines (communicator size per rank) on stderr, for the scaling record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import torch
    import torch.distributed as dist

    import paper_2505_13644_b200 as ctm
    from paper_2505_13644_b200.dist import gather, shard
    from synth import mlp_params, points, sigma as make_sigma

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    D, widths, wl = workload(args)
    strong = args.scaling == "strong"
    if strong:
        offset, N = shard(args.n_total, rank, world)
        n_glob = args.n_total
    else:
        N = args.n
        offset = rank * N
        n_glob = N * world
    params = mlp_params(widths, 0)
    mlp = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=local)
    mlp.set_direction_block(args.direction_block)
    mlp.set_precision(args.precision)
    prods = 6 if args.precision == "fp32" else 3  # tensor products per useful product (after the
    # warm-up: the arithmetic the calls actually ran in, an fp16x3 handle runs uncovered calls in fp32)
    # each rank: its own contiguous slice of the global point set (global index offset ...)
    X_host = points(n_glob, D, 1)[offset:offset + N]
    X = torch.from_numpy(X_host).to(dev)
    sig = torch.from_numpy(make_sigma(D, D, kind="dense")).to(dev)
    op_out = torch.empty(N, device=dev)
    f_out = torch.empty(N, device=dev)
    train = args.op == "laplacian_train"
    launches = {}
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

    def step(Xd, op_out=op_out, f_out=f_out, m=mlp, po=offset):
        if train:
            train_step(Xd, op_out, f_out)
        elif args.op == "laplacian":
            m.laplacian(Xd, out=op_out, f_out=f_out)
        elif args.op == "standard":
            m.laplacian_standard(Xd, out=op_out, f_out=f_out)
        elif args.op == "weighted":
            m.weighted_laplacian(Xd, sig, out=op_out, f_out=f_out)
        elif args.op == "randomized":
            m.randomized_laplacian(Xd, S=args.S, seed=2, point_offset=po, out=op_out, f_out=f_out)
        elif args.op == "stochastic_biharmonic":
            m.stochastic_biharmonic(Xd, S=args.S, seed=2, point_offset=po, out=op_out, f_out=f_out)
        elif args.op == "biharmonic_nested":
            m.biharmonic_nested(Xd, out=op_out, f_out=f_out)
        elif args.op == "biharmonic_standard":
            m.biharmonic_standard(Xd, out=op_out, f_out=f_out)
        elif args.op == "randomized_standard":
            m.randomized_laplacian(Xd, S=args.S, seed=2, point_offset=po, out=op_out, f_out=f_out, standard=True)
        elif args.op == "stochastic_biharmonic_standard":
            m.stochastic_biharmonic(Xd, S=args.S, seed=2, point_offset=po, out=op_out, f_out=f_out, standard=True)
        else:
            m.biharmonic(Xd, out=op_out, f_out=f_out)

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
    ran = mlp.last_precision()  # the arithmetic the calls ran in (training: the forward's, which the backward follows)
    prods = 6 if ran == "fp32" else 3

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.1)
    # ---------------- device-resident timed loop
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    mlp.profile(True)
    clocks.mark("start")
    for a, b in evs:
        flush_buf.zero_()
        a.record()
        step(X)
        b.record()
    torch.cuda.synchronize()
    clocks.mark("end")
    barrier()
    prof = mlp.profile_read()
    mlp.profile(False)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = max_over_ranks(sum(step_ms))
    best_ms = max_over_ranks(min(step_ms))      # the paper's protocol: best of the repetitions
    median_ms = max_over_ranks(float(np.median(step_ms)))
    clk = clocks.stop()

    # ---------------- strong scaling: the same steps with the all_gather of op and f inside
    gather_rec = None
    if strong and not train:
        gevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)]
        gathered = None
        barrier()
        torch.cuda.synchronize()
        for a, b in gevs:
            flush_buf.zero_()
            a.record()
            step(X)
            gathered = (gather(op_out, n_glob), gather(f_out, n_glob)) if world > 1 else (op_out, f_out)
            b.record()
        torch.cuda.synchronize()
        barrier()
        g_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in gevs))
        gather_rec = {"value": n_glob * args.steps / (g_ms / 1e3), "ms_per_step": g_ms / args.steps,
                      "collective": "all_gather_into_tensor of op and f (NCCL)" if world > 1 else "none (1 rank)"}
        if rank == 0:
            # the G-rank result against one GPU evaluating all n_total points
            Xall = torch.from_numpy(points(n_glob, D, 1)).to(dev)
            o1, f1 = torch.empty(n_glob, device=dev), torch.empty(n_glob, device=dev)
            step(Xall, o1, f1, mlp, 0)
            torch.cuda.synchronize()
            gather_rec["bitwise_equal_1gpu"] = bool(torch.equal(gathered[0], o1) and torch.equal(gathered[1], f1))

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

    # sanity: the e2e result equals the device-resident one bit for bit (the training step
    # updates the weights every step, so its results move on)
    if not train:
        assert torch.equal(oh, op_out.cpu()), "e2e result differs from the device-resident run"

    value = n_glob * args.steps / (total_ms / 1e3)
    e2e_value = n_glob * args.steps / (e2e_ms / 1e3)

    # ---------------- the same steps in the other precision modes (same protocol: warm-up, L2
    # flush between timed steps, CUDA events, max over ranks), for the line's `other_precisions`
    others = {}
    if not train and not args.no_other_precisions:
        for prec in [q for q in ("fp32", "fp16x3", "bf16x3") if q not in (args.precision, ran)]:
            mlp.set_precision(prec)
            for _ in range(3):
                step(X)
            torch.cuda.synchronize()
            q_ran = mlp.last_precision()
            if q_ran != prec:  # the mode does not cover this operator (it ran another arithmetic)
                continue
            qevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    for _ in range(args.steps)]
            barrier()
            torch.cuda.synchronize()
            for a, b in qevs:
                flush_buf.zero_()
                a.record()
                step(X)
                b.record()
            torch.cuda.synchronize()
            barrier()
            q_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in qevs))
            others[prec] = {"value": n_glob * args.steps / (q_ms / 1e3), "ms_per_step": q_ms / args.steps,
                            "unit": "points/s"}
        mlp.set_precision(args.precision)


    # ---------------- roofline of the dominant kernel
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh_:
            peaks = json.load(fh_)
        peak_src = "measured"
    except OSError:
        peak_src = "fallback"
    bf16_burst = peaks.get("bf16_tflops", 1590.0)
    bf16_sust = peaks.get("bf16_tflops_sustained", 1400.0)
    timed_s = total_ms / 1e3
    # the burst rate (cuBLAS timed alone) for a timed region of a fraction of a second; the
    # sustained rate (seconds-long loop under the power cap) once the region lasts >= 2 s
    sustained = timed_s >= 2.0
    tensor_peak = bf16_sust if sustained else bf16_burst
    useful_peak = tensor_peak / prods      # bf16 tensor products per useful fp32-accurate product
    dom = max(("layer", "bwd", "wgrad"), key=lambda k: prof[k]["ms"]) if train else "layer"
    lay = prof[dom]
    achieved = lay["work"] / (lay["ms"] / 1e3) / 1e12 if lay["ms"] > 0 else None
    mode = {"fp32": "bf16x6 (three planes, fp32 mode)", "fp16x3": "fp16x3 (two scaled fp16 planes, 3xTF32-class)",
            "bf16x3": "3xBF16 (two planes, fast mode)"}[ran]
    kernel_name = {
        "layer": f"jet_layer_kernel (hidden layers: tcgen05 {mode} GEMM + tanh Taylor epilogue)",
        "bwd": f"jet_layer_kernel<kBwd2> (adjoint layers: tcgen05 {mode} W^T GEMM + transposed Taylor rule)",
        "wgrad": f"wgrad_kernel (weight gradients Z_bar^T B: tcgen05 {mode}, MN-major operands)",
    }[dom]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "layer_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh_:
            tj = json.load(fh_)
        key = (f"{args.op}_S{args.S}" if args.op == "randomized" else args.op) + f"_{args.precision}"
        traffic = tj.get(key, {}).get({"layer": "", "bwd": "bwd_"}.get(dom, "wgrad_") + "dram_bytes_per_launch")
    roofline = {
        "bound": "tensor", "achieved": achieved, "peak": useful_peak, "unit": "TFLOP/s",
        "frac": (achieved / useful_peak) if achieved else None, "traffic": traffic,
        "kernel": kernel_name,
        "peak_basis": (f"{peak_src} bf16 {'sustained' if sustained else 'burst'} {tensor_peak} TF/s / {prods} (bf16 "
                       f"tensor products per useful product); timed region {timed_s:.2f} s "
                       f"({'>=' if sustained else '<'} 2 s)"),
        "work_basis": "useful FLOP = 2 * N * P * w_in * w_out per hidden layer, P the slots of a point with all its "
                      "directions in one block (C1: 52 slots, 129.6 MFLOP/point over layers 2-4)",
        "tensor_pipe_frac": (prods * achieved / tensor_peak) if achieved else None,
        "frac_vs_burst": (prods * achieved / bf16_burst) if achieved else None,
        "frac_vs_sustained": (prods * achieved / bf16_sust) if achieved else None,
        "layer_ms_share": lay["ms"] / sum(step_ms) if sum(step_ms) > 0 else None,
        "kernel_ms_per_step": {k: v["ms"] / args.steps for k, v in prof.items()},
        "launches_per_step": {k: v["launches"] / args.steps for k, v in prof.items()},
    }
    if train:
        tot = sum(v["ms"] for v in prof.values())
        roofline["kernel_share"] = {k: v["ms"] / tot for k, v in prof.items() if v["ms"] > 0}
        wg = prof["wgrad"]
        if wg["ms"] > 0:
            wa = wg["work"] / (wg["ms"] / 1e3) / 1e12
            roofline["wgrad"] = {"achieved": wa, "peak": useful_peak, "frac": wa / useful_peak, "unit": "TFLOP/s",
                                 "ms_share": wg["ms"] / tot}
    # the HBM-write-bound stage: layer 1 written by the seed kernel (fixed direction sets);
    # bytes written per its event time against this device's write-only ceiling measured here
    sd = prof["seed"]
    if sd["ms"] > 0 and sd["work"] > 0:
        wceil = write_ceiling_gbs(dev)
        gbs = sd["work"] / (sd["ms"] / 1e3) / 1e9
        roofline["seed_hbm"] = {"bound": "hbm", "achieved": gbs, "peak": wceil, "unit": "GB/s", "frac": gbs / wceil,
                                "copy_peak": peaks.get("hbm_gbs"), "frac_vs_copy_peak": gbs / peaks.get("hbm_gbs", 6546.0),
                                "note": "bytes the seed kernel writes (the layer-1 block, bf16 planes) per its event "
                                        "time; peak = cudaMemsetAsync of 4 GiB timed on this device in this run"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        flop_pt = prof["layer"]["work"] / (args.steps * N) if prof["layer"]["work"] > 0 else None
        cpu = cpu_baseline(D, widths, args.op, args.S, flop_pt)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "best_ms_per_step": best_ms, "median_ms_per_step": median_ms,
            "scaling": args.scaling,
            "vs_baseline": (value / PAPER_PTS_PER_S[args.op]) if args.op in PAPER_PTS_PER_S else None,
            "vs_baseline_ref": ("paper P:1205, marginal ms/datum on an RTX 6000, PyTorch (another machine: context)"
                                if args.op in PAPER_PTS_PER_S else "no published number for this operator"),
            "dtype": {"fp32": "f32 (bf16x6: three bf16 planes per operand, six tensor products, fp32 accumulate)",
                      "fp16x3": "f32 (fp16x3: two power-of-two-scaled fp16 planes per operand = 22-bit operands as "
                                "in 3xTF32, three tensor products, fp32 accumulate)",
                      "bf16x3": "f32 storage, bf16x3 products (~17-bit operands, fp32 accumulate)"}[ran],
            "data": "synthetic",
            "config": {"workload": wl, "op": args.op, "precision": args.precision, "precision_ran": ran,
                       "N_per_gpu": N, "N_total": n_glob, "D": D, "widths": widths,
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
        if gather_rec is not None:
            line["with_gather"] = gather_rec
        if others:
            line["other_precisions"] = {
                **others,
                "note": "the same operator and workload timed in the other ctm_set_precision modes after the main "
                        "timed region (same protocol; not part of value): fp32 = bf16x6 (24-bit operands), fp16x3 "
                        "= two scaled fp16 planes (22-bit operands, the 3xTF32 split), bf16x3 = ~17-bit operands"}
        print(json.dumps(line), flush=True)
    mlp.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
