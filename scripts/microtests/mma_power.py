"""Sustained tensor throughput under the power cap by operand type and data: cuBLAS matmuls
(8192^3) back to back for ~3 s each, device time per matmul and the NVML SM clock. Answers
whether a cheaper-to-toggle operand format would raise the power-capped rate of the layer
kernel (power wall). Prints one JSON."""
import json
import subprocess
import threading
import time

import torch

n = 8192
dev = "cuda"


def clock_sampler(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True).stdout.strip().split(",")
        try:
            out.append((float(r[0]), float(r[1])))
        except Exception:
            pass
        time.sleep(0.1)


def run(tag, a, b, fn, secs=3.0):
    for _ in range(3):
        fn(a, b)
    torch.cuda.synchronize()
    stop, samples = threading.Event(), []
    th = threading.Thread(target=clock_sampler, args=(stop, samples))
    th.start()
    t0 = time.time()
    cnt = 0
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    while time.time() - t0 < secs:
        for _ in range(10):
            fn(a, b)
        cnt += 10
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = s.elapsed_time(e) / cnt
    tail = samples[len(samples) // 2:] or samples
    return {tag: {"tflops": 2 * n ** 3 / ms / 1e9, "ms": ms, "sm_mhz": sorted(x[0] for x in tail)[len(tail) // 2],
                  "power_w": sorted(x[1] for x in tail)[len(tail) // 2]}}


res = {}
g = torch.Generator(device=dev).manual_seed(0)
ra = torch.randn(n, n, device=dev, generator=g)
rb = torch.randn(n, n, device=dev, generator=g)
mm = lambda a, b: torch.matmul(a, b)
res.update(run("bf16_random", ra.bfloat16(), rb.bfloat16(), mm))
res.update(run("fp16_random", ra.half(), rb.half(), mm))
# bf16 values whose low 4 mantissa bits are zero (fewer toggling bits)
lowz = lambda t: (t.bfloat16().view(torch.int16) & ~0xF).view(torch.bfloat16)
res.update(run("bf16_low4zero", lowz(ra), lowz(rb), mm))
# residual-plane-like bf16 data: tiny values with random mantissas
res.update(run("bf16_residual_scale", (ra * 2 ** -9).bfloat16(), rb.bfloat16(), mm))
res.update(run("bf16_zeros_half", torch.where(ra > 0, ra, 0).bfloat16(), rb.bfloat16(), mm))
torch.backends.cuda.matmul.allow_tf32 = True
res.update(run("tf32_random", ra, rb, mm))
try:
    sa = torch.tensor(1.0, device=dev)
    fa, fb = ra.to(torch.float8_e4m3fn), rb.t().contiguous().to(torch.float8_e4m3fn).t()
    res.update(run("fp8_e4m3_random", fa, fb, lambda a, b: torch._scaled_mm(a, b, sa, sa, out_dtype=torch.bfloat16)))
except Exception as ex:  # noqa: BLE001
    res["fp8_e4m3_random"] = {"error": str(ex)[:200]}
print(json.dumps(res))
