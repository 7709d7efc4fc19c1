"""Select outcomes over a run of steps with fresh gradients (error feedback
accumulating): prints items whose speculative window missed
(TAGC_DEBUG_SELECT=1 must be set)."""
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
ctx.set_graphs(False)
gen = torch.Generator(device="cuda")
acc = torch.zeros(total, device="cuda")
out = torch.empty(total, device="cuda")
for step in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    gen.manual_seed(3000 + (0 if os.environ.get("SAME_GRAD") else step))
    m = torch.randn(total, device="cuda", generator=gen).exp_()
    sg = torch.randint(0, 2, (total,), device="cuda", generator=gen, dtype=torch.int8)
    g = torch.where(sg.bool(), -m, m)
    print("step", step, flush=True)
    ctx.set_timing(True)
    ctx.tagc_reduce_shards(shards, g, acc, out, stats=False)
    ctx.sync()
    print("  stages", [round(x, 3) for x in ctx.last_timing()], flush=True)
