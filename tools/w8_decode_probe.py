"""Decode cost at W = 8 on the GPT-2 layout (make_shards(gpt2, 8, 8), theta
99, r 10, w 4): 8 rank contexts on one GPU encode through the split API, the
test harness reduce-scatters (fp32 / wrapping u32 sums), and each owner's
tagc_reduce_shards_end (decode of 1/8 of the model at union density ~7.7 %,
peel load ~0.77) is timed with CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_05638_b200 as tagc  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
specs = tagc.gpt2_specs()
shards = tagc.make_shards(specs, W, W)
total = shards[-1].end
cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="non_attention_linear",
                             include_out_proj=True, seed=77)
_, Bf, Bu = tagc.plan_exchange(cfg, shards, W, 0)
ctxs = [tagc.Context(cfg, world_size=W, rank=r, device=0) for r in range(W)]
gen = torch.Generator(device="cuda")
accs = [torch.zeros(total, device="cuda") for _ in range(W)]
send_f = [torch.zeros(W * Bf, device="cuda") for _ in range(W)]
send_u = [torch.zeros(W * Bu, dtype=torch.int32, device="cuda") for _ in range(W)]
outs = [torch.empty(sum(s.size() for s in shards if s.owner == r), device="cuda") for r in range(W)]
for step in range(3):
    for r in range(W):
        gen.manual_seed(100 * step + r)
        m = torch.randn(total, device="cuda", generator=gen).exp_()
        g = torch.where(torch.randint(0, 2, (total,), device="cuda", generator=gen, dtype=torch.int8).bool(), -m, m)
        ctxs[r].reduce_shards_begin(shards, g, accs[r], outs[r], send_f[r], send_u[r])
    torch.cuda.synchronize()
    times, stats = [], []
    for o in range(W):
        rf = send_f[0][o * Bf:(o + 1) * Bf].clone()
        ru = send_u[0][o * Bu:(o + 1) * Bu].to(torch.int64)
        for r in range(1, W):
            rf += send_f[r][o * Bf:(o + 1) * Bf]
            ru += send_u[r][o * Bu:(o + 1) * Bu].to(torch.int64)
        ru = ((ru & 0xFFFFFFFF) ^ 0x80000000).sub(0x80000000).to(torch.int32)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(torch.cuda.current_stream())
        st = ctxs[o].reduce_shards_end(rf, ru)
        b.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        stats.append(st)
    print("unresolved per owner", [s.unresolved for s in stats], "presence", [s.presence for s in stats])
    print(f"step {step}: decode ms per owner {[round(t, 3) for t in times]}; presence {stats[0].presence} "
          f"unresolved {stats[0].unresolved} rounds {ctxs[0].last_peel_rounds()}", flush=True)
