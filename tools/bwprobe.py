"""HBM read-only / write-only / copy bandwidth on this GPU (torch kernels, CUDA events)."""
import torch

n = 1 << 30  # 4 GiB of float32
a = torch.empty(n, dtype=torch.float32, device="cuda")
b = torch.empty(n, dtype=torch.float32, device="cuda")
a.fill_(1.0)
torch.cuda.synchronize()


def t(fn, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


ms = t(lambda: b.fill_(2.0))
print(f"write-only  {4 * n / ms / 1e6:8.1f} GB/s")
ms = t(lambda: b.copy_(a))
print(f"copy (r+w)  {8 * n / ms / 1e6:8.1f} GB/s")
s = torch.empty((), device="cuda")
ms = t(lambda: s.copy_(a.sum()))
print(f"read-only   {4 * n / ms / 1e6:8.1f} GB/s")
