"""GPT-2 exchange at the paper's 1-bit setting (theta 98.75, ratio 10, w=1),
W = 2 simulated on one GPU (tagc_reduce_shard_sim per shard): step time with
per-stage timing, versus w = 4 at the same theta (ordered FIFO peel vs the
unordered one)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_05638_b200 as tagc  # noqa: E402

specs = tagc.gpt2_specs()
W = 2
shards = tagc.make_shards(specs, W, W)
total = shards[-1].end
gen = torch.Generator(device="cuda")
gen.manual_seed(3)
grads = []
for r in range(W):
    m = torch.randn(total, device="cuda", generator=gen).exp_()
    s = torch.randint(0, 2, (total,), device="cuda", generator=gen, dtype=torch.int8)
    grads.append(torch.where(s.bool(), -m, m))
for width in (1, 4):
    cfg = tagc.CompressionConfig(theta=98.75, ratio=10, index_width=width, policy="non_attention_linear",
                                 include_out_proj=True, seed=77)
    ctx = tagc.Context(cfg, device=0)
    accs = [torch.zeros(total, device="cuda") for _ in range(W)]
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st_all = []
        for sh in shards:
            g = [x[sh.begin:sh.end] for x in grads]
            a = [x[sh.begin:sh.end] for x in accs]
            _, st = ctx.tagc_reduce_shard_sim(sh, g, a)
            st_all.append(st)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
    print(f"w={width}: {dt:.2f} ms per step (both shards, W={W} simulated); "
          f"presence={sum(s.presence for s in st_all)} unresolved={sum(s.unresolved for s in st_all)} "
          f"lost={sum(s.index_lost for s in st_all)} spurious={sum(s.index_spurious for s in st_all)} "
          f"rounds={ctx.last_peel_rounds()}", flush=True)
