"""Host-side logic on CPU: the C ABI library loads and exports every declared
symbol; sharding/gather over a world_size-2 gloo group; bench/entry plumbing."""
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests._util import ROOT

HEADER = os.path.join(ROOT, "include", "ctm.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ctm_[a-z_]+)\s*\(", src)))


def test_header_declares_the_survey_boundary():
    names = declared_functions()
    for n in ("ctm_load_mlp", "ctm_free_mlp", "ctm_laplacian", "ctm_weighted_laplacian",
              "ctm_randomized_laplacian", "ctm_biharmonic", "ctm_status_str", "ctm_last_error"):
        assert n in names


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2505_13644_b200 import build

    build.build()
    import ctypes

    lib = ctypes.CDLL(build.LIB)
    for n in declared_functions():
        assert hasattr(lib, n), n
    # host-only calls (no device work)
    lib.ctm_status_str.restype = ctypes.c_char_p
    assert lib.ctm_status_str(5) == b"CTM_EUNSUPPORTED"
    lib.ctm_free_mlp.argtypes = [ctypes.c_void_p]
    assert lib.ctm_free_mlp(None) == 0
    lib.ctm_laplacian.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int64] + [ctypes.c_void_p] * 3
    assert lib.ctm_laplacian(None, None, 0, None, None, None) == 1  # CTM_EINVAL: NULL handle


def test_binding_abi_table_matches_header():
    import paper_2505_13644_b200 as ctm

    assert sorted(ctm.ABI) == declared_functions()


def test_shard_partitions_exactly():
    from paper_2505_13644_b200.dist import shard

    for n in (0, 1, 7, 16384, 16385):
        for world in (1, 2, 3, 8):
            spans = [shard(n, r, world) for r in range(world)]
            assert sum(c for _, c in spans) == n
            assert spans[0][0] == 0
            for (o1, c1), (o2, _) in zip(spans, spans[1:]):
                assert o1 + c1 == o2
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_13644_b200.dist import gather, shard

    off, cnt = shard(n, rank, world)
    local = torch.arange(off, off + cnt, dtype=torch.float32) * 2.0
    full = gather(local, n)
    q.put((rank, full.numpy().tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [10, 11])
def test_gather_world2_gloo(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(2):
        assert res[r] == [2.0 * i for i in range(n)]


def test_randomized_directions_shard_invariant_in_oracle():
    """The counter-based generator makes a rank's draws independent of the split."""
    import oracle as O
    from paper_2505_13644_b200.dist import shard

    full = O.rademacher(3, 0, 20, 4, 6)
    parts = [O.rademacher(3, *shard(20, r, 3), 4, 6) for r in range(3)]
    np.testing.assert_array_equal(full, np.concatenate(parts))


def test_bench_reference_arm_runs_on_cpu(tmp_path):
    import json
    import subprocess
    import sys

    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--op", "biharmonic", "--ref-budget-s", "2"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle"


def _worker_grad(rank, world, port, q):
    """Data-parallel training on a world-2 gloo group: each rank differentiates its shard
    (the fp64 oracle stands in for ctm_backward on CPU), allreduce_grads sums them."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np

    from oracle import grad as OG
    from paper_2505_13644_b200.dist import allreduce_grads, shard
    from tests._util import random_params

    Ws, bs = random_params([3, 8, 6, 1], 4)
    n = 11
    X = np.random.default_rng(0).uniform(-1, 1, (n, 3))
    gop = np.random.default_rng(1).standard_normal(n)
    gf = np.random.default_rng(2).standard_normal(n)
    off, cnt = shard(n, rank, world)
    sl = slice(off, off + cnt)
    _, _, dW, db = OG.k2_grad(Ws, bs, X[sl], np.eye(3), np.ones(3), gop[sl], gf[sl])
    grads = [(torch.from_numpy(w.copy()), torch.from_numpy(b.copy())) for w, b in zip(dW, db)]
    allreduce_grads(grads)
    _, _, fW, fb = OG.k2_grad(Ws, bs, X, np.eye(3), np.ones(3), gop, gf)
    err = max(max(np.max(np.abs(g.numpy() - w)) for (g, _), w in zip(grads, fW)),
              max(np.max(np.abs(g.numpy() - b)) for (_, g), b in zip(grads, fb)))
    q.put((rank, float(err)))
    dist.destroy_process_group()


def test_data_parallel_gradient_allreduce_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_grad, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res[0] < 1e-12 and res[1] < 1e-12, res


# ------------------------------------------------------------------ direction-block planner
def _slots(order, rb):
    return {4: 3 * rb + 2, 3: 1 + 2 * rb, 5: 1 + 4 * rb}.get(order, rb + 2)


@pytest.mark.parametrize("order", [2, 3, 4, 5])
def test_direction_block_planner_invariants(order):
    """ctm_plan_blocks (host only): the blocks cover the R directions with padding only in
    the last block, a block fits one MMA tile, and the tile holds ppt blocks."""
    import paper_2505_13644_b200 as ctm

    for R in list(range(1, 70)) + [84, 85, 100, 127, 128, 129, 254, 255, 300, 1000, 2048]:
        pl = ctm.plan_blocks(order, R)
        nb, rb, P, ppt, n = (pl[k] for k in ("blocks", "per_block", "slots_per_block", "points_per_tile", "mma_n"))
        assert nb * rb >= R > (nb - 1) * rb, (R, pl)
        assert P == _slots(order, rb) and P <= 256
        assert n % 16 == 0 and ppt * P <= n <= 256 and (ppt + 1) * P > 256 or ppt == 128, (R, pl)
        assert ctm.plan_blocks(order, R) == pl  # a function of (order, R) only: never of N


def test_direction_block_planner_choices():
    import paper_2505_13644_b200 as ctm

    # C1 (R = D = 50, P = 52, four points in N = 208) stays one block
    assert ctm.plan_blocks(2, 50)["blocks"] == 1
    # C3 S = 128 (P = 130 alone in an N = 144 tile) is split into wide-tile blocks
    pl = ctm.plan_blocks(2, 128)
    assert pl["blocks"] > 1 and pl["mma_n"] >= 240
    # C4 biharmonic (J = 35) stays one block of 107 slots
    assert ctm.plan_blocks(4, 35)["slots_per_block"] == 107
    # beyond one tile: S = 255 and J = 85 need blocks
    assert ctm.plan_blocks(2, 255)["blocks"] >= 2 and ctm.plan_blocks(4, 85)["blocks"] >= 2
    # forced block sizes are honoured (clipped to R); one that does not fit a tile is refused
    assert ctm.plan_blocks(2, 50, 7) == {"blocks": 8, "per_block": 7, "slots_per_block": 9,
                                         "points_per_tile": 28, "mma_n": 256}
    assert ctm.plan_blocks(2, 5, 9)["per_block"] == 5
    with pytest.raises(ctm.CTMError, match="EUNSUPPORTED"):
        ctm.plan_blocks(2, 300, 300)
    with pytest.raises(ctm.CTMError, match="EINVAL"):
        ctm.plan_blocks(6, 10)


def test_product_package_never_touches_the_oracle():
    """The product path (the package and its kernels) shares no code with oracle/ and
    never imports it; only tests, smoke() and bench's CPU arms may."""
    import ast
    import pathlib

    pkg = pathlib.Path(__file__).resolve().parents[1] / "paper_2505_13644_b200"
    files = list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")) + list(pkg.rglob("*.h"))
    assert files
    for f in files:
        src = f.read_text()
        if f.suffix == ".py":
            for node in ast.walk(ast.parse(src)):
                if isinstance(node, ast.Import):
                    assert all(not a.name.split(".")[0] == "oracle" for a in node.names), f
                elif isinstance(node, ast.ImportFrom):
                    assert (node.module or "").split(".")[0] != "oracle", f
        else:
            assert "ctmo" not in src and "oracle/" not in src, f


def test_product_path_fails_loudly_without_the_library(monkeypatch, tmp_path):
    """No CPU fallback: with libctm.so missing, loading raises instead of computing."""
    import paper_2505_13644_b200 as ctm

    monkeypatch.setattr(ctm, "_lib", None)
    monkeypatch.setattr(ctm, "LIB_PATH", str(tmp_path / "libctm.so"))
    with pytest.raises(ctm.CTMError, match="no fallback"):
        ctm.lib()


def test_product_path_raises_without_a_gpu():
    """On a machine without a CUDA device the operators raise (nothing runs on the CPU)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2505_13644_b200 as ctm

    with pytest.raises(Exception):
        ctm.MLP([(torch.zeros(4, 3), torch.zeros(4)), (torch.zeros(1, 4), torch.zeros(1))], device=0)


def _worker_strong(rank, world, port, n_total, q):
    """bench.py --scaling strong on a world-2 gloo group with the fp64 oracle standing in for
    the GPU operator: each rank evaluates its dist.shard slice of the global point set with the
    global point_offset (randomized directions keyed on the global index), the results are
    all_gathered, and rank 0 compares them bitwise with one process evaluating all points."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2505_13644_b200.dist import gather, shard
    from synth import mlp_params, points

    params = mlp_params([4, 12, 10, 1], 0)
    net = O.Net([W.astype(np.float64) for W, _ in params], [b.astype(np.float64) for _, b in params])
    Xall = points(n_total, 4, 1).astype(np.float64)
    off, cnt = shard(n_total, rank, world)
    V = O.rademacher(2, off, cnt, 3, 4)          # generated from the GLOBAL point index
    op, f, _ = O.randomized_laplacian(net, Xall[off:off + cnt], V)
    g_op = gather(torch.from_numpy(op), n_total)
    g_f = gather(torch.from_numpy(f), n_total)
    if rank == 0:
        op1, f1, _ = O.randomized_laplacian(net, Xall, O.rademacher(2, 0, n_total, 3, 4))
        q.put(bool(torch.equal(g_op, torch.from_numpy(op1)) and torch.equal(g_f, torch.from_numpy(f1))))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [9, 16])
def test_strong_scaling_bookkeeping_world2_gloo(n_total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_strong, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in ps:
        p.start()
    ok = q.get(timeout=180)
    for p in ps:
        p.join(timeout=60)
    assert ok


def test_bench_strong_scaling_cli_and_workload_string():
    """The strong-scaling workload names the total batch (both arms print the same config)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    sys_argv = ["bench.py", "--scaling", "strong", "--n-total", "4096"]
    import sys

    old = sys.argv
    sys.argv = sys_argv
    try:
        args = bench.parse()
    finally:
        sys.argv = old
    D, widths, wl = bench.workload(args)
    assert args.scaling == "strong" and "N=4096 points split over the GPUs" in wl
