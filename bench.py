#!/usr/bin/env python
"""Benchmark: uncompressed-equivalent gradient GB/s per sync (encode + exchange +
decode) of the B200 TAGC exchange, BASELINE.json's metric.

Workload (BASELINE config 2, "GPT-2 small (124M) shaped per-layer gradient
buckets, layer-selective compression"): every rank holds a full GPT-2-small
(tied head, 124,439,808 fp32) gradient laid out by the reference's own layer
list (model.cpp:39-64); make_shards(specs, N, N) gives one shard per rank;
non_attention_linear policy (+ out-proj), theta = 99 per rank, ratio 10,
4-bit index, seed 77. A step is one full exchange: every rank sparsifies and
encodes all shards, the index/sketch/raw blocks are reduce-scattered over
NCCL, and every owner peels its shard back to dense fp32. Accumulators carry
error feedback across steps. Gradients are synthetic log-normal magnitudes with
fair signs (the distribution of the reference's SyntheticStream,
train.cpp:445-459), generated on device; 498 MB per rank, > L2 (126 MB).

value = N * 124,439,808 * 4 B / (device time per step, max over ranks).

--impl reference times the reference's own CPU implementation
(oracle/_ref/libtagc_ref.so: tagc_reduce_shard with World(N, parallel), all
host threads) on a bounded sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

THETA, RATIO, WIDTH, SEED = 99.0, 10, 4, 77
WORKLOADS = {  # --workload: BASELINE config 2 (default) and config 3's layer layout
    "gpt2": "gpt2-small-124M-tied/non_attention_linear/theta99/r10/w4",
    "llama3-8b": "llama3-8b-8.03B/non_attention_linear/theta99/r10/w4",
}
WORKLOAD = WORKLOADS["gpt2"]
METRIC = "uncompressed-equivalent gradient GB/s per sync (encode+RS+decode)"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for i, nm in enumerate(names):
                    if "Active" in r[2 + i] and "Not" not in r[2 + i]:
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload_specs(name="gpt2"):
    import paper_2504_05638_b200 as tagc

    return tagc.llama3_8b_specs() if name == "llama3-8b" else tagc.gpt2_specs()


def cfg_obj():
    import paper_2504_05638_b200 as tagc

    return tagc.CompressionConfig(theta=THETA, ratio=RATIO, index_width=WIDTH,
                                  policy="non_attention_linear", include_out_proj=True, seed=SEED)


def algorithmic_bytes(shards, rank, world):
    """SURVEY.md §8(d) bytes for this rank's dominant kernel, the fused
    select + encode pass (k_fused_tma): per compressed element it reads g and
    acc (8 B) and writes the residual (4 B) and the packed index (w/8 B), plus
    a 24*d sketch read-modify-write (d = kept density = 1 - theta/100). The
    separate select pass of the survey's model (8 B) is gone: selection rides
    on the same pass, bracketed by two small passes over a 1/32 sample (2 x
    8/32 B, separate kernels, not in this figure)."""
    import paper_2504_05638_b200 as tagc

    comp = 0
    for sh in shards:
        for s in sh.segments:
            if tagc.kind_compressible(s.kind, "non_attention_linear", True) and s.size() >= 1024:
                comp += s.size()
    dens = 1.0 - THETA / 100.0
    fused = comp * (12.0 + WIDTH / 8.0 + 24.0 * dens)
    return comp, fused


def extra_sections(args, tagc, ctx, shards, grad, acc, out, owned, total, n_params, specs, stream, dev, local,
                   world, step, barrier, max_over_ranks, e0, e1):
    """Uncompressed comparator, owner step, overlap and e2e (GPT-2 workload)."""
    import torch

    # uncompressed comparator: ncclReduceScatter fp32 of the same shards (a
    # peer-exchange context has no NCCL communicator: no comparator then)
    base_ms = None
    if world == 1 or args.exchange == "nccl":
        base_out = torch.empty(shards[0].size(), device=dev)
        for _ in range(args.warmup):
            ctx.baseline_reduce_shards(shards, grad, base_out)
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            ctx.baseline_reduce_shards(shards, grad, base_out)
        e1.record(stream)
        barrier()
        base_ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
        del base_out

    # owner-side consumer: exchange + adamw_nm step on the
    # owned shard, unfused (tagc_reduce_shards then tagc_apply_optimizer,
    # which re-reads the decoded shard) vs fused (tagc_reduce_shards_step,
    # the update inside the decode emit / raw unpack, decoded not stored)
    params = torch.randn(max(owned, 1), device=dev)
    adam_v = torch.zeros(max(owned, 1), device=dev)
    opt_steps = max(3, min(args.steps, 10))

    def timed(fn):
        for i in range(max(3, args.warmup)):  # eager, capture, first replay
            fn(i + 1)
        barrier()
        e0.record(stream)
        for i in range(opt_steps):
            fn(i + 2)
        e1.record(stream)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1)) / opt_steps

    def unfused(k):
        step()
        ctx.apply_optimizer("adamw_nm", 1e-3, params, out, world, k, adam_v, weight_decay=0.01)

    def fused(k):
        ctx.tagc_reduce_shards_step(shards, grad, acc, params, "adamw_nm", 1e-3, k, adam_v=adam_v,
                                    weight_decay=0.01)

    owner_step = {"optimizer": "adamw_nm",
                  "apply_only_ms": round(timed(lambda k: ctx.apply_optimizer(
                      "adamw_nm", 1e-3, params, out, world, k, adam_v, weight_decay=0.01)), 4),
                  "unfused_ms": round(timed(unfused), 4), "fused_ms": round(timed(fused), 4)}

    # backward / exchange overlap: a synthetic backward
    # pass on a producer stream (3 bf16 GEMMs 8192x768 @ 768x3072 per GPT-2
    # block, then the block's gradient lands in the buffer), in reverse layer
    # order. one_shot: tagc_reduce_shards after the backward; overlapped:
    # tagc_overlap_* encoding each block as it lands. Times from backward start
    # to the decoded shard, device events.
    groups, off = [], 0
    for sp in specs:
        key = sp.name.split(".")[0] if sp.name.startswith("h") else ("final" if sp.name.startswith("ln_f") else "embed")
        if not groups or groups[-1][0] != key:
            groups.append([key, off, off])
        off += sp.param_count
        groups[-1][2] = off
    ranges = [(lo, hi) for _, lo, hi in groups]
    ranges[-1] = (ranges[-1][0], total)  # the make_shards pad tail lands with the last block
    ga = torch.randn(8192, 768, device=dev, dtype=torch.bfloat16)
    gb = torch.randn(768, 3072, device=dev, dtype=torch.bfloat16)
    gc = torch.empty(8192, 3072, device=dev, dtype=torch.bfloat16)
    grad_bw = torch.empty_like(grad)
    prod = torch.cuda.Stream(device=local)

    def backward(on_ready=None):
        for lo, hi in reversed(ranges):
            with torch.cuda.stream(prod):
                for _ in range(3):
                    torch.mm(ga, gb, out=gc)
                grad_bw[lo:hi].copy_(grad[lo:hi])
                ev = torch.cuda.Event()
                ev.record(prod)
            if on_ready:
                on_ready(lo, hi, ev)
        done = torch.cuda.Event()
        done.record(prod)
        return done

    def run_overlap(mode):
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        prod.wait_stream(stream)  # iterations do not overlap each other
        b0.record(prod)
        if mode == "backward":
            backward()
            b1.record(prod)
        elif mode == "one_shot":
            stream.wait_event(backward())
            ctx.tagc_reduce_shards(shards, grad_bw, acc, out, stats=False)
            b1.record(stream)
        else:
            stream.wait_event(b0)
            ctx.overlap_begin(shards, grad_bw, acc, out)
            backward(ctx.overlap_ready)
            ctx.overlap_finish()
            b1.record(stream)
        return b0, b1

    overlap = {"producer": "3x bf16 mm 8192x768@768x3072 per block, 14 blocks, reverse order"}
    for mode in ("backward", "one_shot", "overlapped"):
        for _ in range(max(3, args.warmup)):
            run_overlap(mode)
        barrier()
        evs = [run_overlap(mode) for _ in range(opt_steps)]
        barrier()
        overlap[mode + "_ms"] = round(max_over_ranks(sum(a.elapsed_time(b) for a, b in evs) / opt_steps), 4)
    del ga, gb, gc, grad_bw

    # e2e through the C-ABI host-buffer entry (tagc_reduce_shards_host): every
    # step copies this step's gradient H2D from pinned memory and the owner's
    # decoded shard D2H; consecutive calls overlap their copies with each
    # other and with the exchange (two copy streams, double-buffered device
    # buffers). host_join() makes the timing stream wait for the last D2H.
    host_grad = torch.empty(total, dtype=torch.float32, pin_memory=True)
    host_grad.copy_(grad.cpu())
    host_out = torch.empty(max(owned, 1), dtype=torch.float32, pin_memory=True)
    e2e_steps = min(max(30, args.steps), 60)  # ~10 ms a step (PCIe-bound): pipeline fill + drain once
    for _ in range(2):
        ctx.tagc_reduce_shards_host(shards, host_grad, acc, host_out)
    ctx.host_join()
    barrier()
    e0.record(stream)
    for _ in range(e2e_steps):
        ctx.tagc_reduce_shards_host(shards, host_grad, acc, host_out)
    ctx.host_join()
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / e2e_steps
    # the PCIe bound of that path: both directions at once (torch copies of the
    # same buffers on two streams), gradient-equivalent GB/s
    s_in, s_out = torch.cuda.Stream(device=local), torch.cuda.Stream(device=local)
    pc0, pc1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        barrier()
        pc0.record(stream)
        s_in.wait_stream(stream)
        s_out.wait_stream(stream)
        with torch.cuda.stream(s_in):
            grad_bw_probe = grad.copy_(host_grad, non_blocking=True)
        with torch.cuda.stream(s_out):
            host_out.copy_(out, non_blocking=True)
        stream.wait_stream(s_in)
        stream.wait_stream(s_out)
        pc1.record(stream)
        barrier()
    pcie_ms = max_over_ranks(pc0.elapsed_time(pc1))
    del grad_bw_probe

    uncompressed = n_params * 4.0
    e2e = {"value": round(world * uncompressed / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
           "h2d_bytes_per_step": int(total * 4), "d2h_bytes_per_step": int(owned * 4), "steps": e2e_steps,
           "pcie_bound": round(world * uncompressed / (pcie_ms * 1e-3) / 1e9, 3),
           "pcie_bound_note": "the same H2D + D2H bytes as plain concurrent copies, no exchange"}
    return base_ms, owner_step, overlap, e2e


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2504_05638_b200 as tagc

    world = args.gpus
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    # TAGC_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo host plumbing -
    # a plumbing check of the N > 1 code on a one-GPU box (--exchange peer;
    # NCCL refuses two ranks on one device). Never a measurement.
    share = world > 1 and os.environ.get("TAGC_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = f"cuda:{local}"
    specs = workload_specs(args.workload)
    big = args.workload != "gpt2"  # 8B parameters: no room for the owner-step / overlap / e2e buffers
    shards = tagc.make_shards(specs, world, world)
    total = shards[-1].end
    n_params = sum(s.param_count for s in specs)
    cfg = cfg_obj()

    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ctx = tagc.Context(cfg, world_size=world, rank=rank, device=local, stream=stream.cuda_stream)
    if world > 1 and args.exchange == "peer":  # pulls over NVLink peer memory (CUDA IPC), no NCCL
        handles = [None] * world
        dist.all_gather_object(handles, ctx.peer_prepare(shards))
        ctx.peer_open(handles)
    elif world > 1:
        obj = [tagc.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.init_nccl(obj[0])

    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    grad = torch.empty(total, device=dev)
    chunk = 1 << 26  # generated in chunks: the temporaries of an 8B-element draw would not fit
    for c0 in range(0, total, chunk):
        c1 = min(total, c0 + chunk)
        mag = torch.randn(c1 - c0, device=dev, generator=gen).exp_()
        sign = torch.randint(0, 2, (c1 - c0,), device=dev, generator=gen, dtype=torch.int8)
        grad[c0:c1] = torch.where(sign.bool(), -mag, mag)
    del mag, sign
    if total > n_params:
        grad[n_params:] = 0.0  # make_shards pad tail
    acc = torch.zeros(total, device=dev)
    owned = sum(s.size() for s in shards if s.owner == rank)
    out = torch.empty(max(owned, 1), device=dev)
    torch.cuda.synchronize()

    def step(stats=False):
        return ctx.tagc_reduce_shards(shards, grad, acc, out, stats=stats)

    for _ in range(args.warmup):
        step()
    _, st = step(stats=True)  # untimed: peel statistics of this config
    rounds = ctx.last_peel_rounds()
    ctx.set_timing(True)
    step()
    stage_ms = ctx.last_timing()
    launches_per_step = ctx.last_launches()
    ctx.set_timing(False)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            if share:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if share else dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    clk = clocks.stop()

    # per-stage device time of one step with stage events (prep, sampled select +
    # fused split/encode, select finish, exchange, decode)
    # (each timed call starts on an idle stream: stage events recorded behind a
    # queue of earlier calls were seen to be stamped late)
    # The roofline kernel's duration comes from device-side %globaltimer
    # stamps the kernels write in timing mode (earliest CTA start of k_sample
    # to latest CTA end of k_fused), averaged over the timed launches.
    ctx.set_timing(True)
    stage_acc = [0.0] * 5
    span_acc = [0.0, 0.0]
    for _ in range(args.steps):
        ctx.sync()
        step()
        t = ctx.last_timing()
        stage_acc = [a + b for a, b in zip(stage_acc, t)]
        span_acc = [a + b for a, b in zip(span_acc, ctx.last_kernel_spans())]
    ctx.set_timing(False)
    stage_ms = [a / args.steps for a in stage_acc]
    span_ms = [a / args.steps for a in span_acc]

    base_ms = owner_step = overlap = e2e = None
    if not big:
        base_ms, owner_step, overlap, e2e = extra_sections(
            args, tagc, ctx, shards, grad, acc, out, owned, total, n_params, specs, stream, dev, local, world,
            step, barrier, max_over_ranks, e0, e1)
    comp, fused_bytes = algorithmic_bytes(shards, rank, world)
    hbm, peak_kind = peaks()
    fused_ms = span_ms[0]
    achieved = fused_bytes / (fused_ms * 1e-3) / 1e9 if fused_ms > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "fused_traffic.json")
    if os.path.exists(tpath) and args.workload == "gpt2":  # captured on the default workload
        try:
            with open(tpath) as f:
                traffic = json.load(f).get("bytes_per_launch")
        except Exception:
            traffic = None

    uncompressed = n_params * 4.0
    value = world * uncompressed / (ms * 1e-3) / 1e9
    result = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic log-normal gradients (SyntheticStream distribution), generated on device",
        "config": {
            "workload": WORKLOADS[args.workload],
            "params_per_rank": n_params,
            "shards": f"make_shards({args.workload}, {world}, {world})",
            "compressed_params_per_rank": comp,
            "peel": {"presence": st.presence, "peeled": st.peeled, "unresolved": st.unresolved,
                     "rounds": rounds[0], "tail_rounds": rounds[1]},
            "l2": f"inputs larger than L2 ({total * 4 / 1e6:.0f} MB per rank)",
            "parallelism": f"dp{world} (one process per GPU, "
                           f"{'peer-memory pulls' if args.exchange == 'peer' else 'NCCL reduce-scatter'})",
        },
        "e2e": e2e if e2e is not None else {"skipped": "8B-parameter workload: host buffers not allocated"},
        "roofline": {"kernel": "k_fused_tma (TMA-staged select/split/index/sketch scatter)",
                     "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": int(fused_bytes),
                     "kernel_ms": round(fused_ms, 4),
                     "timed": "k_fused_tma launches: device span from %globaltimer stamps written by the "
                              "kernel (first CTA start to last CTA end), mean of the timed launches"},
        "decode_span_ms": round(span_ms[1], 4),
        "stages_ms": {"prep": round(stage_ms[0], 4), "select_fused": round(stage_ms[1], 4),
                      "select_finish": round(stage_ms[2], 4), "exchange": round(stage_ms[3], 4),
                      "decode": round(stage_ms[4], 4)},
        "uncompressed_rs": ({"value": round(world * uncompressed / (base_ms * 1e-3) / 1e9, 3),
                             "unit": "GB/s", "ms_per_step": round(base_ms, 4)} if base_ms else None),
        "owner_step": owner_step,
        "overlap": overlap,
        "gpu_launches": int(launches_per_step * args.steps),
        "clocks": clk,
    }
    if share:
        result["config"]["shared_gpu_plumbing_check"] = "all ranks on cuda:0 (TAGC_BENCH_SHARE_GPU=1): not a measurement"
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not big:
        result["cpu_baseline"] = cpu_baseline(args, specs, world, budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        barrier()
        dist.destroy_process_group()


def sample_shards(specs, world, budget_elems):
    """A bounded sample of the workload: the shard plan of make_shards(specs,
    W, W) restricted to its first segments up to ~budget_elems per rank."""
    import oracle as O
    import paper_2504_05638_b200 as tagc

    shards = tagc.make_shards(specs, world, world)
    out, used = [], 0
    for sh in shards:
        segs = []
        for s in sh.segments:
            if used >= budget_elems:
                break
            segs.append(O.Segment(s.kind, s.begin, s.end, s.name))
            used += s.size()
        if segs:
            out.append(O.Shard(sh.id, sh.owner, segs[0].begin, segs[-1].end, segs))
    return out, used


def cpu_baseline(args, specs, world, budget_s=20.0):
    """The reference's own CPU path (oracle/_ref) on the host cores, bounded."""
    import numpy as np

    import oracle as O

    if not O.Ref.available():
        return {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    ref = O.Ref()
    budget = args.cpu_elems
    shards, used = sample_shards(specs, world, budget)
    end = max(s.end for s in shards)
    grads = list(O.Oracle().stream(end, 2024, count=world))
    cfg = O.Config(THETA, RATIO, WIDTH, "non_attention_linear", True, SEED, 3, False, 1024)
    # each shard's grads are sliced by the reference wrapper from the flat buffers
    secs = ref.time_reduce_shards(shards, grads, cfg, reps=1)
    t = float(secs.min())
    return {"value": round(world * used * 4 / t / 1e9, 5), "unit": "GB/s",
            "cores": os.cpu_count(), "kind": "reference",
            "sample": f"first {used} params per rank of the workload ({len(shards)} shard(s)), "
                      f"tagc_reduce_shard World({world}, parallel), OMP_NUM_THREADS={os.environ['OMP_NUM_THREADS']}",
            "seconds": round(t, 3)}


def run_reference(args):
    world = args.gpus
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    import numpy as np

    import oracle as O

    if not O.Ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtagc_ref.so not built"}))
        return
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    specs = workload_specs()
    shards, used = sample_shards(specs, world, args.cpu_elems)
    end = max(s.end for s in shards)
    grads = list(O.Oracle().stream(end, 2024, count=world))
    cfg = O.Config(THETA, RATIO, WIDTH, "non_attention_linear", True, SEED, 3, False, 1024)
    ref = O.Ref()
    ref.time_reduce_shards(shards, grads, cfg, reps=max(0, min(args.warmup, 1)) or 1)
    secs = ref.time_reduce_shards(shards, grads, cfg, reps=args.steps)
    t = float(secs.mean())
    value = world * used * 4 / t / 1e9
    sample = (f"first {used} params per rank of {WORKLOAD} ({len(shards)} shard(s)), "
              f"tagc_reduce_shard World({world}, parallel)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic SyntheticStream gradients (reference generator)",
        "config": {"workload": WORKLOAD, "sample_params_per_rank": used},
        "cpu_baseline": {"value": round(value, 5), "unit": "GB/s", "cores": os.cpu_count(),
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 5), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-elems", type=int, default=24_000_000,
                    help="params per rank in the bounded CPU-reference sample")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="gpt2", choices=sorted(WORKLOADS),
                    help="gpt2 (BASELINE config 2, the default line) or llama3-8b (config 3's layout)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="N>1 collective: grouped ncclReduceScatter, or pulls over peer memory")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
