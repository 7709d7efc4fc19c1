"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) that drives every kernel family of the library once:

* the NCCL-world exchange path at W=1 (select chain, k_fused_tma, k_fixup,
  the deferred region-ordered scatter (forced), k_list, k_r0_emit,
  k_r0_subtract_cnt, k_peel, k_final_fix) on a GPT-2-shaped layout,
* the owner step fused into k_emit (k_emit<opt>, k_copy_items<opt>),
* the simulated world with a 1-bit index at W=2 (ordered peel, index
  diagnostics, audit),
* the peer-memory exchange at W=2 (k_peer_signal / wait / pull), contexts of
  this process,
* the standalone codec entries (sparsify, index, sketch, peel, estimate).

Run:  compute-sanitizer --tool memcheck python tools/sanitize_workload.py
Checks results against nothing (the parity tests do that); it exists so the
sanitizer sees every kernel on a real launch configuration."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_05638_b200 as tagc  # noqa: E402

DEV = "cuda:0"


def lognormal(n, seed):
    g = torch.Generator(device=DEV)
    g.manual_seed(seed)
    x = torch.randn(n, device=DEV, generator=g).exp_()
    s = torch.randint(0, 2, (n,), device=DEV, generator=g).float() * 2 - 1
    return (x * s).contiguous()


def exchange_w1():
    specs = tagc.gpt2_specs(layers=2, d_model=128, ffn_mult=4, vocab=3000, ctx=128)
    shards = tagc.make_shards(specs, 1, 1)
    total = shards[-1].end
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="non_attention_linear", seed=77)
    ctx = tagc.Context(cfg, device=0)
    acc = torch.zeros(total, device=DEV)
    for step in range(2):
        out, st = ctx.tagc_reduce_shards(shards, lognormal(total, 10 + step), acc, stats=True)
    torch.cuda.synchronize()
    print("w1 exchange", st)
    # owner step fused into the emit
    params = torch.zeros(total, device=DEV)
    adam_v = torch.zeros(total, device=DEV)
    ctx.tagc_reduce_shards_step(shards, lognormal(total, 20), acc, params, "adamw_nm", 1e-3, 1,
                                adam_v=adam_v, weight_decay=0.01)
    torch.cuda.synchronize()
    print("owner step ok")


def exchange_deferred():
    os.environ["TAGC_DEFER_SCATTER_BYTES"] = "0"  # read at context creation
    n = 1 << 20
    shards = [tagc.ShardSpec(0, 0, 0, n, [tagc.LayerSegment("ffn", "feed_forward", 0, n)])]
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="all_layers", seed=5,
                                 min_compress_segment=1)
    ctx = tagc.Context(cfg, device=0)
    acc = torch.zeros(n, device=DEV)
    out, st = ctx.tagc_reduce_shards(shards, lognormal(n, 3), acc, stats=True)
    torch.cuda.synchronize()
    del os.environ["TAGC_DEFER_SCATTER_BYTES"]
    print("deferred scatter", st)


def sim_w2_onebit():
    n = 1 << 16
    shard = tagc.ShardSpec(0, 0, 0, n, [tagc.LayerSegment("ffn", "feed_forward", 0, n)])
    cfg = tagc.CompressionConfig(theta=98.75, ratio=10, index_width=1, policy="all_layers", seed=77,
                                 min_compress_segment=1)
    ctx = tagc.Context(cfg, device=0)
    grads = [lognormal(n, 30 + r) for r in range(2)]
    accs = [torch.zeros(n, device=DEV) for _ in range(2)]
    out, st, audit = ctx.tagc_reduce_shard_sim_audit(shard, grads, accs)
    torch.cuda.synchronize()
    print("sim w=1", st)


def peer_w2():
    specs = tagc.gpt2_specs(layers=1, d_model=64, ffn_mult=4, vocab=1000, ctx=64)
    world = 2
    shards = tagc.make_shards(specs, world, world)
    total = shards[-1].end
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="non_attention_linear", seed=77)
    streams = [torch.cuda.Stream() for _ in range(world)]
    ctxs = []
    for r in range(world):
        with torch.cuda.stream(streams[r]):
            ctxs.append(tagc.Context(cfg, world_size=world, rank=r, device=0))
    for c in ctxs:
        c.peer_prepare(shards)
    for c in ctxs:
        c.peer_attach_local(ctxs)
    g = [lognormal(total, 40 + r) for r in range(world)]
    acc = [torch.zeros(total, device=DEV) for _ in range(world)]
    outs = [None] * world

    def run(r):
        outs[r], _ = ctxs[r].tagc_reduce_shards(shards, g[r], acc[r], stats=False)
        ctxs[r].sync()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    print("peer exchange ok")


def codec():
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="all_layers", seed=1)
    ctx = tagc.Context(cfg, device=0)
    n = 100_003
    v = lognormal(n, 50)
    sparse, residual, tau, _ = ctx.sparsify(v, 99.0)
    words = ctx.index_create(sparse, 4)
    pos = ctx.index_presence(words, n, 4)
    sk = ctx.sketch_compress(sparse, 10, 7)
    vals, unres, pf = ctx.peeling_decompress(pos, sk, n, 10, 7)
    torch.cuda.synchronize()
    print("codec ok", int(pos.numel()), pf)


if __name__ == "__main__":
    exchange_w1()
    exchange_deferred()
    sim_w2_onebit()
    peer_w2()
    codec()
    print("sanitize workload done")
