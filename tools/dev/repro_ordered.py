"""Small multi-segment 1-bit exchange (ordered peel) for compute-sanitizer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import oracle as O
import paper_2504_05638_b200 as tagc

specs = tagc.gpt2_specs(layers=int(os.environ.get("L", 2)), d_model=int(os.environ.get("D", 64)), ffn_mult=4, vocab=int(os.environ.get("V", 700)), ctx=64)
shards = tagc.make_shards(specs, 2, 2)
total = shards[-1].end
orc = O.Oracle()
grads = orc.stream(total, 99, count=2)
cfg = tagc.CompressionConfig(theta=98.75, ratio=10, index_width=1, policy="non_attention_linear", seed=77,
                             min_compress_segment=1024)
ctx = tagc.Context(cfg, device=0)
for sh in shards:
    g = [torch.from_numpy(x[sh.begin:sh.end].copy()).cuda() for x in grads]
    a = [torch.zeros(sh.size(), device="cuda") for _ in g]
    out, st = ctx.tagc_reduce_shard_sim(sh, g, a)
    torch.cuda.synchronize()
    ref, rst = orc.tagc_reduce_shard(O.Shard(sh.id, sh.owner, sh.begin, sh.end,
                                             [O.Segment(s.kind, s.begin, s.end, s.name) for s in sh.segments]),
                                     [x[sh.begin:sh.end] for x in grads],
                                     [np.zeros(sh.size(), np.float32) for _ in g],
                                     O.Config(98.75, 10, 1, "non_attention_linear", True, 77, 3, False, 1024))
    o = out.cpu().numpy()
    print(sh.id, st, rst, float(np.abs(o - ref).max()), float(np.abs(ref).max()))
