"""Pure HBM write vs read vs copy bandwidth on this B200 (torch kernels, CUDA events)."""
import torch
n = 1280 * 1024 * 1024  # 2.56 GB of bf16 pairs ~ the C1 seed block
a = torch.empty(n, dtype=torch.uint16, device="cuda")
b = torch.empty(n, dtype=torch.uint16, device="cuda")
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
    return best
ms = t(lambda: a.fill_(7)); print(f"fill (write only) {2*n/ms/1e9:.2f} TB/s  {ms:.3f} ms")
ms = t(lambda: b.copy_(a)); print(f"copy (r+w)        {4*n/ms/1e9:.2f} TB/s  {ms:.3f} ms")
ms = t(lambda: a.sum(dtype=torch.float32)); print(f"sum (read only)   {2*n/ms/1e9:.2f} TB/s  {ms:.3f} ms")
