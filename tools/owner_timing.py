"""Per-call device time of the owner step (unfused vs fused), mirroring
bench.py's owner_step block, with a kernel timeline of the fused calls."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2504_05638_b200 as tagc  # noqa: E402

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
wd = float(sys.argv[1]) if len(sys.argv) > 1 else 0.01


def unfused(k):
    ctx.tagc_reduce_shards(shards, grad, acc, out, stats=False)
    ctx.apply_optimizer("adamw_nm", 1e-3, params, out, 1, k, v, weight_decay=wd)


def fused(k):
    ctx.tagc_reduce_shards_step(shards, grad, acc, params, "adamw_nm", 1e-3, k, adam_v=v, weight_decay=wd)


for name, fn in (("unfused", unfused), ("fused", fused), ("unfused", unfused), ("fused", fused)):
    ts = []
    for k in range(1, 9):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        fn(k)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 3))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(10):
        fn(k + 9)
    e1.record(stream)
    torch.cuda.synchronize()
    print(name, "isolated:", ts, "back-to-back ms/step:", round(e0.elapsed_time(e1) / 10, 4))
