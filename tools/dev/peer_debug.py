"""Debug: W contexts on one GPU with the peer exchange; per-call host timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2504_05638_b200 as tagc
W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
specs = [tagc.LayerSpec("ffn", "feed_forward", 1 << 20), tagc.LayerSpec("b", "bias", 4096)]
shards = tagc.make_shards(specs, W, W)
total = shards[-1].end
cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="non_attention_linear", seed=77)
streams = [torch.cuda.Stream() for _ in range(W)]
ctxs = []
for r in range(W):
    with torch.cuda.stream(streams[r]):
        ctxs.append(tagc.Context(cfg, world_size=W, rank=r, device=0))
for c in ctxs:
    c.peer_prepare(shards)
for c in ctxs:
    c.peer_attach_local(ctxs)
print("prepared", flush=True)
g = [torch.randn(total, device="cuda") for _ in range(W)]
a = [torch.zeros(total, device="cuda") for _ in range(W)]
o = [torch.empty(total, device="cuda") for _ in range(W)]
torch.cuda.synchronize()
order = list(range(W))[::-1] if os.environ.get("REVERSE") else list(range(W))
for step in range(3):
    for r in order:
        t = time.time()
        ctxs[r].tagc_reduce_shards(shards, g[r], a[r], o[r], stats=False)
        print(f"step {step} rank {r} enqueue {1e3 * (time.time() - t):.1f} ms", flush=True)
    for r, c in enumerate(ctxs):
        t = time.time()
        try:
            c.sync()
            print(f"step {step} rank {r} sync ok {1e3 * (time.time() - t):.1f} ms", flush=True)
        except Exception as e:
            print(f"step {step} rank {r} sync FAIL {e}", flush=True)
