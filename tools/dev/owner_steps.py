"""8 fused adamw_nm owner steps on the bench workload (for an ncu launch list)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2504_05638_b200 as tagc  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fused"
specs = bench.workload_specs()
shards = tagc.make_shards(specs, 1, 1)
total = shards[-1].end
ctx = tagc.Context(bench.cfg_obj(), device=0)
ctx.set_graphs(False)
gen = torch.Generator(device="cuda")
gen.manual_seed(1000)
mag = torch.randn(total, device="cuda", generator=gen).exp_()
sign = torch.randint(0, 2, (total,), device="cuda", generator=gen, dtype=torch.int8)
grad = torch.where(sign.bool(), -mag, mag)
acc = torch.zeros(total, device="cuda")
out = torch.empty(total, device="cuda")
params = torch.randn(total, device="cuda")
v = torch.zeros(total, device="cuda")
for k in range(1, 9):
    if mode == "fused":
        ctx.tagc_reduce_shards_step(shards, grad, acc, params, "adamw_nm", 1e-3, k, adam_v=v, weight_decay=0.01)
    else:
        ctx.tagc_reduce_shards(shards, grad, acc, out, stats=False)
ctx.sync()
print("ok")
