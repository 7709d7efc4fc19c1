"""Owner-step probe: GPT-2 W=1, a few unfused (reduce_shards + apply_optimizer)
and fused (reduce_shards_step) adamw_nm steps, for an ncu launch list."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2504_05638_b200 as tagc  # noqa: E402

specs = bench.workload_specs()
shards = tagc.make_shards(specs, 1, 1)
total = shards[-1].end
ctx = tagc.Context(bench.cfg_obj(), device=0)
g = torch.randn(total, device="cuda").exp_()
acc = torch.zeros(total, device="cuda")
out = torch.empty(total, device="cuda")
params = torch.randn(total, device="cuda")
v = torch.zeros(total, device="cuda")
mode = sys.argv[1] if len(sys.argv) > 1 else "both"
for k in range(1, 4):
    if mode in ("both", "unfused"):
        ctx.tagc_reduce_shards(shards, g, acc, out, stats=False)
        ctx.apply_optimizer("adamw_nm", 1e-3, params, out, 1, k, v, weight_decay=0.01)
    if mode in ("both", "fused"):
        ctx.tagc_reduce_shards_step(shards, g, acc, params, "adamw_nm", 1e-3, k, adam_v=v, weight_decay=0.01)
ctx.sync()
torch.cuda.synchronize()
print("ok")
