"""BASELINE config 4 at N = 1: a 2^28-element single bucket (feed_forward,
min_compress_segment = 1), density 0.1 % - 10 % (theta 99.9 ... 90, ratio
= the largest Table-1 ratio whose floor <= theta), error feedback carried
across steps. Reports exchange GB/s, k_fused_tma span and peel statistics.

    python tools/density_sweep.py [--steps 5] [--n-log2 28]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_05638_b200 as tagc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--n-log2", type=int, default=28)
    ap.add_argument("--theta", type=float, default=None, help="only this operating point")
    args = ap.parse_args()
    n = 1 << args.n_log2
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    grad = torch.randn(n, device="cuda", generator=g).exp_()
    grad.mul_(torch.randint(0, 2, (n,), device="cuda", generator=g, dtype=torch.int8).float().mul_(2).sub_(1))
    shards = [tagc.ShardSpec(0, 0, 0, n, [tagc.LayerSegment("bucket", "feed_forward", 0, n)])]
    out = torch.empty(n, device="cuda")
    rows = []
    for theta, ratio in ((99.9, 10), (99.5, 10), (99.0, 10), (98.0, 4), (95.0, 4), (90.0, 4)):
        if args.theta is not None and theta != args.theta:
            continue
        cfg = tagc.CompressionConfig(theta=theta, ratio=ratio, index_width=4, policy="all_layers", seed=77,
                                     min_compress_segment=1)
        ctx = tagc.Context(cfg, device=0)
        acc = torch.zeros(n, device="cuda")
        for _ in range(3):
            ctx.tagc_reduce_shards(shards, grad, acc, out, stats=False)
        _, st = ctx.tagc_reduce_shards(shards, grad, acc, out, stats=True)
        ctx.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            ctx.tagc_reduce_shards(shards, grad, acc, out, stats=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        ctx.set_timing(True)
        ctx.sync()
        ctx.tagc_reduce_shards(shards, grad, acc, out, stats=False)
        ctx.sync()
        spans = ctx.last_kernel_spans()
        rows.append({"theta": theta, "ratio": ratio, "ms_per_step": round(ms, 3),
                     "gbs": round(n * 4 / (ms * 1e-3) / 1e9, 1), "k_fused_ms": round(spans[0], 3),
                     "decode_ms": round(spans[1], 3), "presence": st.presence, "peeled": st.peeled,
                     "unresolved": st.unresolved, "rounds": list(ctx.last_peel_rounds())})
        print(json.dumps(rows[-1]), flush=True)
        del ctx, acc
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
