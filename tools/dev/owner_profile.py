"""Per-kernel durations of isolated owner steps (CUPTI via torch.profiler),
to find which kernels make some steps slower than others."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2504_05638_b200 as tagc  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fused"
specs = bench.workload_specs()
shards = tagc.make_shards(specs, 1, 1)
total = shards[-1].end
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = tagc.Context(bench.cfg_obj(), device=0, stream=stream.cuda_stream)
gen = torch.Generator(device="cuda")
gen.manual_seed(1000)
mag = torch.randn(total, device="cuda", generator=gen).exp_()
sign = torch.randint(0, 2, (total,), device="cuda", generator=gen, dtype=torch.int8)
grad = torch.where(sign.bool(), -mag, mag)
acc = torch.zeros(total, device="cuda")
out = torch.empty(total, device="cuda")
params = torch.randn(total, device="cuda")
v = torch.zeros(total, device="cuda")


def fn(k):
    if mode == "fused":
        ctx.tagc_reduce_shards_step(shards, grad, acc, params, "adamw_nm", 1e-3, k, adam_v=v, weight_decay=0.01)
    elif mode == "unfused":
        ctx.tagc_reduce_shards(shards, grad, acc, out, stats=False)
        ctx.apply_optimizer("adamw_nm", 1e-3, params, out, 1, k, v, weight_decay=0.01)
    else:
        ctx.tagc_reduce_shards(shards, grad, acc, out, stats=False)


for k in range(1, 4):
    fn(k)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(4, 14):
        fn(k)
        torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
def nm(e):
    return e.name.replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "").split("::")[-1][:22]


t0 = evs[0].time_range.start
prev = t0
for e in evs:
    d = e.time_range.end - e.time_range.start
    gap = e.time_range.start - prev
    if d > 15 or gap > 15:
        print(f"{e.time_range.start - t0:9.1f} dur {d:7.1f} gap {gap:7.1f} {nm(e)}")
    prev = max(prev, e.time_range.end)
