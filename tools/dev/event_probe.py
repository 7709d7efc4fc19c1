"""Probe: are CUDA event timestamps ordered with pinned H2D copies on the same stream?"""
import torch
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
h = torch.zeros(1024, pin_memory=True)
d = torch.zeros(1024, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
for trial in range(3):
    torch.cuda.synchronize()
    ev[0].record(s)
    torch.cuda._sleep(400_000)          # ~200 us kernel
    d.copy_(h, non_blocking=True)       # pinned H2D on the same stream
    ev[1].record(s)
    torch.cuda._sleep(400_000)
    ev[2].record(s)
    d.copy_(h, non_blocking=True)
    torch.cuda._sleep(400_000)
    ev[3].record(s)
    x = torch.empty(1 << 24, device="cuda"); x.zero_()
    ev[4].record(s)
    torch.cuda._sleep(400_000)
    ev[5].record(s)
    torch.cuda.synchronize()
    print([round(ev[i].elapsed_time(ev[i + 1]), 4) for i in range(5)])
