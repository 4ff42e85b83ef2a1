"""Write-bandwidth ceiling on this B200: cudaMemsetAsync vs torch fill_ over the C1 seed
block size (2.56 GB), CUDA events, best of 10."""
import ctypes
import glob
import os

import torch

n = 1280 * 1024 * 1024
a = torch.empty(n, dtype=torch.uint16, device="cuda")
cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
    glob.glob("/usr/local/cuda/lib64/libcudart.so*")
rt = ctypes.CDLL(cands[0])
rt.cudaMemsetAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p]


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


stream = torch.cuda.current_stream().cuda_stream
ms = t(lambda: rt.cudaMemsetAsync(a.data_ptr(), 7, 2 * n, stream))
print(f"cudaMemsetAsync {2 * n / ms / 1e9:.2f} TB/s {ms:.3f} ms")
ms = t(lambda: a.fill_(7))
print(f"torch fill_     {2 * n / ms / 1e9:.2f} TB/s {ms:.3f} ms")
