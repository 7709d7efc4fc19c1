"""Write-only vs copy HBM bandwidth on this GPU (torch fill_ / copy_), the
ceilings for k_emit (a 1 GB dense store) and k_fused_tma (65 % reads)."""
import torch

n = 1 << 28
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
for name, fn, nbytes in (("fill (write only)", lambda: a.fill_(1.0), 4 * n),
                         ("copy (read + write)", lambda: b.copy_(a), 8 * n),
                         ("sum (read only)", lambda: a.sum(), 4 * n)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"{name:22s} {ms * 1e3:8.1f} us  {nbytes / ms / 1e6:8.1f} GB/s")
