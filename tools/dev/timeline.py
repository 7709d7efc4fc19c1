"""Kernel timeline of the bench step (CUPTI via torch.profiler): per launch the
start offset from the step's first kernel, its duration and the idle gap before
it. Shows launch gaps and host stalls that per-kernel ncu times hide.

    python tools/timeline.py [--steps 2] [--world 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--host", action="store_true", help="profile the host-buffer entry (e2e path)")
    ap.add_argument("--own-stream", action="store_true", help="context-owned stream instead of torch's")
    ap.add_argument("--graph", type=int, default=-1, help="force graph mode 0/1 (-1: library default)")
    ap.add_argument("--opt", default="", choices=["", "fused", "unfused"],
                    help="add the owner's adamw_nm step (fused: tagc_reduce_shards_step)")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    import paper_2504_05638_b200 as tagc

    dev = "cuda:0"
    specs = bench.workload_specs()
    shards = tagc.make_shards(specs, 1, 1)
    total = shards[-1].end
    cfg = bench.cfg_obj()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = tagc.Context(cfg, device=0, stream=0 if args.own_stream else stream.cuda_stream)
    if args.graph >= 0 and hasattr(ctx, "set_graphs"):
        ctx.set_graphs(bool(args.graph))
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000)
    mag = torch.randn(total, device=dev, generator=gen).exp_()
    sign = torch.randint(0, 2, (total,), device=dev, generator=gen, dtype=torch.int8)
    grad = torch.where(sign.bool(), -mag, mag)
    del mag, sign
    acc = torch.zeros(total, device=dev)
    out = torch.empty(total, device=dev)
    params, adam_v = torch.randn(total, device=dev), torch.zeros(total, device=dev)
    k = [0]

    def step():
        k[0] += 1
        if args.opt == "fused":
            ctx.tagc_reduce_shards_step(shards, grad, acc, params, "adamw_nm", 1e-3, k[0], adam_v=adam_v)
            return
        ctx.tagc_reduce_shards(shards, grad, acc, out, stats=False)
        if args.opt == "unfused":
            ctx.apply_optimizer("adamw_nm", 1e-3, params, out, 1, k[0], adam_v)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    if args.host:
        hg = grad.cpu().pin_memory()
        ho = torch.empty(total, dtype=torch.float32, pin_memory=True)
        for _ in range(2):
            ctx.tagc_reduce_shards_host(shards, hg, acc, ho)
        ctx.sync()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            if args.host:
                ctx.tagc_reduce_shards_host(shards, hg, acc, ho)
            else:
                step()
        ctx.sync()
        torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.sync()
    ctx.tagc_reduce_shards(shards, grad, acc, out, stats=False)
    ctx.sync()
    print("stage ms (prep, select_fused, select_finish, exchange, decode):",
          [round(x, 4) for x in ctx.last_timing()], "kernel spans (fused, decode):",
          [round(x, 4) for x in ctx.last_kernel_spans()])
    ctx.set_timing(False)
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    if not evs:
        print("no CUDA events")
        return
    t0 = evs[0].time_range.start
    prev_end = t0
    busy = 0.0
    for e in evs:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        busy += d
        print(f"{(s - t0):9.1f}us  dur {d:8.1f}us  gap {s - prev_end:7.1f}us  {e.name[:70]}")
        prev_end = max(prev_end, e.time_range.end)
    span = prev_end - t0
    print(f"span {span:.1f}us for {args.steps} steps ({span / args.steps:.1f}us/step), "
          f"busy {busy / args.steps:.1f}us/step, {len(evs) / args.steps:.0f} device ops/step")


if __name__ == "__main__":
    main()
