"""Isolated exchange steps over rotating fresh gradients (error feedback
accumulating), eager (no graphs), with per-stage device timing of each."""
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
ctx.set_graphs(len(sys.argv) > 1 and sys.argv[1] == "graphs")
gen = torch.Generator(device="cuda")
grads = []
for i in range(4):
    gen.manual_seed(2000 + i)
    m = torch.randn(total, device="cuda", generator=gen).exp_()
    sg = torch.randint(0, 2, (total,), device="cuda", generator=gen, dtype=torch.int8)
    grads.append(torch.where(sg.bool(), -m, m))
acc = torch.zeros(total, device="cuda")
out = torch.empty(total, device="cuda")
torch.cuda.synchronize()
timing = len(sys.argv) > 2 and sys.argv[2] == "timing"
ctx.set_timing(timing)
for k in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    ctx.tagc_reduce_shards(shards, grads[k % 4], acc, out, stats=False)
    b.record(stream)
    torch.cuda.synchronize()
    line = f"step {k}: {a.elapsed_time(b):.3f} ms"
    if timing:
        line += " stages " + str([round(x, 3) for x in ctx.last_timing()]) + " spans " + str(
            [round(x, 3) for x in ctx.last_kernel_spans()])
    print(line, flush=True)
