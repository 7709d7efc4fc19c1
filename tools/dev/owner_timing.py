"""Per-call device time of the owner step (unfused vs fused), mirroring
bench.py's owner_step block, with a kernel timeline of the fused calls."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
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
fresh = len(sys.argv) > 2 and sys.argv[2] == "fresh"
grads = [grad]
if fresh:  # a different gradient every step (rotating through 4 draws)
    for i in range(3):
        gen.manual_seed(2000 + i)
        m = torch.randn(total, device="cuda", generator=gen).exp_()
        sg = torch.randint(0, 2, (total,), device="cuda", generator=gen, dtype=torch.int8)
        grads.append(torch.where(sg.bool(), -m, m))


def unfused(k):
    ctx.tagc_reduce_shards(shards, grads[k % len(grads)], acc, out, stats=False)
    ctx.apply_optimizer("adamw_nm", 1e-3, params, out, 1, k, v, weight_decay=wd)


def fused(k):
    ctx.tagc_reduce_shards_step(shards, grads[k % len(grads)], acc, params, "adamw_nm", 1e-3, k, adam_v=v, weight_decay=wd)


def plain(k):
    ctx.tagc_reduce_shards(shards, grads[k % len(grads)], acc, out, stats=False)


for name, fn in (("unfused", unfused), ("fused", fused), ("unfused", unfused), ("fused", fused), ("plain", plain)):
    ts, hs = [], []
    import time
    for k in range(1, 9):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        h0 = time.perf_counter()
        fn(k)
        hs.append(round((time.perf_counter() - h0) * 1e3, 3))
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 3))
        if ts[-1] > 1.4 and name == "plain":
            ctx.set_timing(True)
            ctx.sync()
            acc_save = acc.clone()
            fn(k)
            ctx.sync()
            print("  slow plain step", k, "stages", [round(x, 3) for x in ctx.last_timing()])
            acc.copy_(acc_save)
            ctx.set_timing(False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time
    e0.record(stream)
    t0 = time.perf_counter()
    for k in range(10):
        fn(k + 9)
    t1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    print(name, "isolated:", ts, "back-to-back ms/step:", round(e0.elapsed_time(e1) / 10, 4),
          "host enqueue ms/step:", round((t1 - t0) * 100, 4))
