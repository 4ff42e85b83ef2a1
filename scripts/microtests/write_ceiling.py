"""Write ceiling of this B200 under the conditions the seed runs in: cudaMemsetAsync (value 0
and 7, 4 GiB and 2.68 GB) timed cold, and again right after 3 s of C1 bench steps (power-
capped clocks), with the NVML SM clock sampled around each measurement. Prints one JSON."""
import ctypes
import glob
import json
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
rt = ctypes.CDLL(libs[0] if libs else "libcudart.so")
rt.cudaMemsetAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p]
buf = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")


def clock():
    out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    return int(out.split()[0]) if out else None


def ms(val, nbytes, reps=6):
    st = torch.cuda.current_stream()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(st)
        rt.cudaMemsetAsync(buf.data_ptr(), val, nbytes, st.cuda_stream)
        b.record(st)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return round(nbytes / best / 1e6, 1)  # GB/s


def sweep(tag):
    c0 = clock()
    r = {f"v{v}_{n >> 20}MiB": ms(v, n) for v in (0, 7) for n in (4 << 30, 2560 << 20)}
    r["sm_mhz_before"], r["sm_mhz_after"] = c0, clock()
    return {tag: r}


res = sweep("cold")
import paper_2505_13644_b200 as ctm  # noqa: E402
from synth import mlp_params, points, widths_for  # noqa: E402

params = mlp_params(widths_for(50), 0)
mlp = ctm.MLP([(torch.from_numpy(W), torch.from_numpy(b)) for W, b in params], device=0)
X = torch.from_numpy(points(16384, 50)).cuda()
t = time.time()
while time.time() - t < 3.0:
    mlp.laplacian(X)
    torch.cuda.synchronize()
res.update(sweep("after_load"))
print(json.dumps(res))
