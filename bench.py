#!/usr/bin/env python
"""Benchmark: uncompressed-equivalent gradient GB/s per sync (encode + exchange +
decode) of the B200 TAGC exchange, BASELINE.json's metric.

Headline workload (BASELINE config 4, the largest single-GPU configuration):
every rank holds ONE 2^28-element fp32 gradient bucket (a single
`feed_forward` segment, min_compress_segment = 1), theta = 99 per rank
(1 % density), ratio 10, 4-bit index, seed 77; make_shards(bucket, N, N)
gives one shard per rank. A step is one full exchange: every rank sparsifies
and encodes its whole bucket, the index / sketch blocks are reduce-scattered
(NCCL over NVLink), and every owner peels its shard back to dense fp32.
Accumulators carry error feedback across steps. Gradients are synthetic
log-normal magnitudes with fair signs (the distribution of the reference's
SyntheticStream, train.cpp:445-459), generated on device; 1 GiB per rank,
> L2 (126 MB), so every step streams from HBM.

value = N * 2^28 * 4 B / (device time per step, max over ranks).

Extra keys (same line): the GPT-2-small layer layout (config 2) at theta 99 /
4-bit and at the paper setting theta 98.75 / 1-bit, the uncompressed
ncclReduceScatter comparator with its bus bandwidth, the owner step and the
backward overlap. --workload llama3-8b runs config 3's layout as the headline.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libtagc_ref.so, compiled from /root/reference by
oracle/Makefile: tagc_reduce_shard with World(N, parallel), all host threads)
on a bounded sample of the same workload, rank 0 only. That arm never imports
the product package: its shard plan comes from the reference's own
make_shards.

--gpus N without torchrun re-launches itself under torch.distributed.run.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "uncompressed-equivalent gradient GB/s per sync (encode+RS+decode)"
SEED = 77
C4_N = 1 << 28


# --------------------------------------------------------------------------- workloads
# Pure host data (name, kind, count) so the reference arm never loads the
# product library.
def gpt2_layers(layers=12, d=768, mu=4, vocab=50257, ctx=1024):
    """GPT-2 small, tied head (reference model.cpp:39-64 order): 124,439,808."""
    out = [("wte", "embedding", vocab * d), ("wpe", "positional_embedding", ctx * d)]
    for l in range(layers):
        p = f"h{l}."
        out += [(p + "ln1.g", "norm", d), (p + "ln1.b", "norm", d),
                (p + "attn.qkv.w", "attention_qkv", d * 3 * d), (p + "attn.qkv.b", "bias", 3 * d),
                (p + "attn.proj.w", "attention_out_proj", d * d), (p + "attn.proj.b", "bias", d),
                (p + "ln2.g", "norm", d), (p + "ln2.b", "norm", d),
                (p + "mlp.fc.w", "feed_forward", d * mu * d), (p + "mlp.fc.b", "bias", mu * d),
                (p + "mlp.proj.w", "feed_forward", mu * d * d), (p + "mlp.proj.b", "bias", d)]
    return out + [("ln_f.g", "norm", d), ("ln_f.b", "norm", d)]


def llama3_8b_layers(layers=32, d=4096, kv=1024, ffn=14336, vocab=128256):
    out = [("embed_tokens", "embedding", vocab * d)]
    for l in range(layers):
        p = f"layers.{l}."
        out += [(p + "q_proj", "attention_qkv", d * d), (p + "k_proj", "attention_qkv", d * kv),
                (p + "v_proj", "attention_qkv", d * kv), (p + "o_proj", "attention_out_proj", d * d),
                (p + "gate_proj", "feed_forward", d * ffn), (p + "up_proj", "feed_forward", d * ffn),
                (p + "down_proj", "feed_forward", ffn * d),
                (p + "input_layernorm", "norm", d), (p + "post_attention_layernorm", "norm", d)]
    return out + [("norm", "norm", d), ("lm_head", "lm_head", d * vocab)]


WORKLOADS = {
    # name: (description, layers(), theta, ratio, width, policy, min_compress_segment)
    "c4": ("bucket-2^28-f32/feed_forward/theta99/r10/w4",
           lambda: [("bucket", "feed_forward", C4_N)], 99.0, 10, 4, "all_layers", 1),
    "gpt2": ("gpt2-small-124M-tied/non_attention_linear/theta99/r10/w4",
             gpt2_layers, 99.0, 10, 4, "non_attention_linear", 1024),
    "gpt2-paper": ("gpt2-small-124M-tied/non_attention_linear/theta98.75/r10/w1 (paper setting)",
                   gpt2_layers, 98.75, 10, 1, "non_attention_linear", 1024),
    "llama3-8b": ("llama3-8b-8.03B/non_attention_linear/theta99/r10/w4",
                  llama3_8b_layers, 99.0, 10, 4, "non_attention_linear", 1024),
}


def workload_config(name, world):
    """The `config` object of the JSON line: identical in both arms."""
    desc, layers, theta, ratio, width, policy, mcs = WORKLOADS[name]
    n = sum(c for _, _, c in layers())
    return {"workload": desc, "params_per_rank": n, "shards": f"make_shards({name}, {world}, {world})",
            "theta": theta, "ratio": ratio, "index_width": width, "policy": policy,
            "include_out_proj": True, "min_compress_segment": mcs, "seed": SEED,
            "l2": f"inputs larger than L2 ({n * 4 / 1e6:.0f} MB of gradient per rank, streamed every step)"}


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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
                 "--format=csv,noheader,nounits", "-lms", "50"],
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


# --------------------------------------------------------------------------- B200 arm
class Rig:
    """Per-rank plumbing: device, stream, context, barrier, max over ranks."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.world = args.gpus
        self.rank = env_int("RANK", 0)
        self.local = env_int("LOCAL_RANK", 0)
        # TAGC_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo host plumbing
        # and the peer-memory exchange - a check of the N > 1 code on a one-GPU
        # box (NCCL refuses two ranks on one device). Never a measurement.
        self.share = self.world > 1 and os.environ.get("TAGC_BENCH_SHARE_GPU") == "1"
        if self.share:
            self.local = 0
            args.exchange = "peer"
        self.exchange = args.exchange
        torch.cuda.set_device(self.local)
        if self.world > 1:
            if self.share:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device(f"cuda:{self.local}"))
        self.dev = f"cuda:{self.local}"
        self.stream = torch.cuda.Stream(device=self.local)
        torch.cuda.set_stream(self.stream)
        self.e0 = torch.cuda.Event(enable_timing=True)
        self.e1 = torch.cuda.Event(enable_timing=True)

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.world > 1:
            if self.share:
                self.dist.barrier()
            else:
                self.dist.barrier(device_ids=[self.local])
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], device="cpu" if self.share else self.dev, dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def timed(self, fn, steps):
        """Device time of `steps` calls (ms per call), CUDA events on the
        context stream bracketed by barrier + synchronize, max over ranks."""
        self.barrier()
        self.e0.record(self.stream)
        for i in range(steps):
            fn(i)
        self.e1.record(self.stream)
        self.barrier()
        return self.max_over_ranks(self.e0.elapsed_time(self.e1)) / steps

    def context(self, tagc, cfg, shards):
        ctx = tagc.Context(cfg, world_size=self.world, rank=self.rank, device=self.local,
                           stream=self.stream.cuda_stream)
        if self.world > 1 and self.exchange == "peer":  # pulls over NVLink peer memory (CUDA IPC)
            handles = [None] * self.world
            self.dist.all_gather_object(handles, ctx.peer_prepare(shards))
            ctx.peer_open(handles)
        elif self.world > 1:
            obj = [tagc.Context.nccl_unique_id() if self.rank == 0 else None]
            self.dist.broadcast_object_list(obj, src=0)
            ctx.init_nccl(obj[0])
        return ctx


def make_workload(tagc, name, world):
    desc, layers, theta, ratio, width, policy, mcs = WORKLOADS[name]
    specs = [tagc.LayerSpec(nm, kind, cnt) for nm, kind, cnt in layers()]
    cfg = tagc.CompressionConfig(theta=theta, ratio=ratio, index_width=width, policy=policy,
                                 include_out_proj=True, seed=SEED, min_compress_segment=mcs)
    shards = tagc.make_shards(specs, world, world)
    return specs, cfg, shards


def synthetic_grad(torch, total, n_params, dev, seed):
    """Log-normal magnitudes with fair signs (SyntheticStream's distribution),
    drawn on the device in chunks; the make_shards pad tail is zero."""
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    grad = torch.empty(total, device=dev)
    chunk = 1 << 26
    for c0 in range(0, total, chunk):
        c1 = min(total, c0 + chunk)
        mag = torch.randn(c1 - c0, device=dev, generator=gen).exp_()
        sign = torch.randint(0, 2, (c1 - c0,), device=dev, generator=gen, dtype=torch.int8)
        grad[c0:c1] = torch.where(sign.bool(), -mag, mag)
    if total > n_params:
        grad[n_params:] = 0.0
    return grad


def compressed_elems(tagc, shards, cfg):
    n = 0
    for sh in shards:
        for s in sh.segments:
            if tagc.kind_compressible(s.kind, cfg.policy, cfg.include_out_proj) and \
                    s.size() >= cfg.min_compress_segment and cfg.ratio > 1:
                n += s.size()
    return n


DEFER_SCATTER_BYTES = 32 << 20  # engine default (TAGC_DEFER_SCATTER_BYTES): larger sketches are deferred


def fused_bytes_per_elem(cfg, deferred=False):
    """SURVEY.md §8(d) bytes per compressed element of the dominant kernel, the
    fused select + split + encode pass (k_fused_tma): read g and acc (8 B),
    write the residual (4 B) and the packed index (w/8 B), plus a 24*d sketch
    read-modify-write (d = 1 - theta/100), or, for a segment whose sketch is
    deferred to the region-sorted scatter (> 32 MB), an 8*d (pos, v) log
    write instead. The separate select pass of the survey's model (8 B) is
    gone: selection rides on the same pass, bracketed by two small passes over
    a 1/32 sample (separate kernels, not counted)."""
    d = 1.0 - cfg.theta / 100.0
    return 12.0 + cfg.index_width / 8.0 + (8.0 if deferred else 24.0) * d


def fused_bytes(tagc, shards, cfg):
    """Algorithmic bytes of one k_fused_tma launch over every compressed
    segment of this rank (every shard is encoded by every rank)."""
    total = 0.0
    for sh in shards:
        for s in sh.segments:
            if tagc.kind_compressible(s.kind, cfg.policy, cfg.include_out_proj) and \
                    s.size() >= cfg.min_compress_segment and cfg.ratio > 1:
                g = tagc.sketch_geometry(s.size(), cfg.ratio, cfg.sketch_rows)
                sketch = 4 * g["rows"] * g["buckets_per_row"]
                total += s.size() * fused_bytes_per_elem(cfg, sketch > DEFER_SCATTER_BYTES)
    return total


def decode_bytes_per_elem(cfg):
    """SURVEY.md §8(d) decode bytes per owned compressed element: read the
    merged index (w/8 B) and the reduced sketch (4/r B), write the dense
    shard (4 B)."""
    return cfg.index_width / 8.0 + 4.0 / cfg.ratio + 4.0


def measure_exchange(rig, tagc, name, args, full=True):
    """One workload: warm-up, peel statistics, K timed steps (+ clocks), then
    the per-stage and kernel-span breakdown. Returns (result dict, state)."""
    torch = rig.torch
    specs, cfg, shards = make_workload(tagc, name, rig.world)
    total = shards[-1].end
    n_params = sum(s.param_count for s in specs)
    ctx = rig.context(tagc, cfg, shards)
    grad = synthetic_grad(torch, total, n_params, rig.dev, 1000 + rig.rank)
    acc = torch.zeros(total, device=rig.dev)
    owned = sum(s.size() for s in shards if s.owner == rig.rank)
    out = torch.empty(max(owned, 1), device=rig.dev)
    torch.cuda.synchronize()

    def step(i=0):
        ctx.tagc_reduce_shards(shards, grad, acc, out, stats=False)

    for _ in range(args.warmup):
        step()
    _, st = ctx.tagc_reduce_shards(shards, grad, acc, out, stats=True)  # untimed: peel statistics
    rounds = ctx.last_peel_rounds()

    clocks = ClockSampler(rig.local) if full else None
    if clocks:
        rig.barrier()
        clocks.start()
    ms = rig.timed(step, args.steps)
    clk = clocks.stop() if clocks else None
    launches = ctx.last_launches()

    # stage breakdown and kernel-written spans (each timed call starts on an
    # idle stream: stage events recorded behind a queue were stamped late)
    ctx.set_timing(True)
    stage_acc, span_acc = [0.0] * 5, [0.0, 0.0]
    reps = max(3, min(args.steps, 10))
    for _ in range(reps):
        ctx.sync()
        step()
        stage_acc = [a + b for a, b in zip(stage_acc, ctx.last_timing())]
        span_acc = [a + b for a, b in zip(span_acc, ctx.last_kernel_spans())]
    ctx.set_timing(False)
    stage_ms = [a / reps for a in stage_acc]
    span_ms = [rig.max_over_ranks(a / reps) for a in span_acc]

    comp = compressed_elems(tagc, shards, cfg)
    owned_comp = compressed_elems(tagc, [s for s in shards if s.owner == rig.rank], cfg)
    value = rig.world * n_params * 4.0 / (ms * 1e-3) / 1e9
    res = {
        "value": round(value, 3), "ms_per_step": round(ms, 4),
        "peel": {"presence": st.presence, "peeled": st.peeled, "unresolved": st.unresolved,
                 "index_lost": st.index_lost, "index_spurious": st.index_spurious,
                 "grid_rounds": rounds[0], "tail_rounds": rounds[1]},
        "k_fused_tma_ms": round(span_ms[0], 4), "decode_span_ms": round(span_ms[1], 4),
        "stages_ms": dict(zip(("prep", "select_fused", "select_finish", "exchange", "decode"),
                              (round(x, 4) for x in stage_ms))),
        "launches_per_step": int(launches),
    }
    state = dict(specs=specs, cfg=cfg, shards=shards, total=total, n_params=n_params, ctx=ctx, grad=grad,
                 acc=acc, out=out, owned=owned, comp=comp, owned_comp=owned_comp, ms=ms, span_ms=span_ms,
                 fused_bytes=fused_bytes(tagc, shards, cfg),
                 clk=clk, step=step)
    return res, state


def uncompressed_comparator(rig, S, args):
    """ncclReduceScatter fp32 of the same shards (baseline_reduce_shard,
    hook.cpp:90-96): time and NCCL bus bandwidth ((W-1)/W x payload / t)."""
    if rig.world > 1 and rig.exchange != "nccl":
        return None  # a peer-exchange context has no NCCL communicator
    torch, ctx, shards = rig.torch, S["ctx"], S["shards"]
    base_out = torch.empty(max(S["owned"], 1), device=rig.dev)
    for _ in range(args.warmup):
        ctx.baseline_reduce_shards(shards, S["grad"], base_out)
    ms = rig.timed(lambda i: ctx.baseline_reduce_shards(shards, S["grad"], base_out), args.steps)
    payload = S["total"] * 4.0
    bus = (rig.world - 1) / rig.world * payload / (ms * 1e-3) / 1e9 if rig.world > 1 else None
    return {"value": round(rig.world * S["n_params"] * 4.0 / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "ms_per_step": round(ms, 4),
            "nccl_bus_gbs": round(bus, 1) if bus is not None else None,
            "what": "ncclReduceScatter fp32 of the same buffers" if rig.world > 1
                    else "N=1: the reduce-scatter degenerates to a device copy"}


def end_to_end(rig, S, args):
    """The same metric through the C-ABI host-buffer entry
    (tagc_reduce_shards_host): every step copies this step's gradient H2D from
    pinned memory and the owner's decoded shard D2H; consecutive calls overlap
    their copies with each other and with the exchange (two copy streams,
    double-buffered device buffers). host_join() makes the timing stream wait
    for the last D2H."""
    torch, ctx, shards = rig.torch, S["ctx"], S["shards"]
    host_grad = torch.empty(S["total"], dtype=torch.float32, pin_memory=True)
    host_grad.copy_(S["grad"].cpu())
    host_out = torch.empty(max(S["owned"], 1), dtype=torch.float32, pin_memory=True)
    steps = max(args.steps, 60)  # the pipeline's fill and drain (about one step) are paid once
    for _ in range(2):
        ctx.tagc_reduce_shards_host(shards, host_grad, S["acc"], host_out)
    ctx.host_join()

    def one(i):
        ctx.tagc_reduce_shards_host(shards, host_grad, S["acc"], host_out)
        if i == steps - 1:
            ctx.host_join()

    ms = rig.timed(one, steps)
    # the PCIe bound of that path: both directions at once (plain copies of
    # the same buffers on two streams)
    s_in, s_out = torch.cuda.Stream(device=rig.local), torch.cuda.Stream(device=rig.local)
    scratch = torch.empty_like(S["grad"])

    def copies(i):
        s_in.wait_stream(rig.stream)
        s_out.wait_stream(rig.stream)
        with torch.cuda.stream(s_in):
            scratch.copy_(host_grad, non_blocking=True)
        with torch.cuda.stream(s_out):
            host_out.copy_(S["out"], non_blocking=True)
        rig.stream.wait_stream(s_in)
        rig.stream.wait_stream(s_out)

    pcie_ms = rig.timed(copies, 3)
    del scratch
    u = rig.world * S["n_params"] * 4.0
    return {"value": round(u / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": int(S["total"] * 4), "d2h_bytes_per_step": int(S["owned"] * 4),
            "steps": steps, "ms_per_step": round(ms, 3),
            "pcie_bound": round(u / (pcie_ms * 1e-3) / 1e9, 3),
            "pcie_bound_note": "the same H2D + D2H bytes as plain concurrent copies, no exchange"}


def owner_step_and_overlap(rig, tagc, S, args):
    """SURVEY §8f rows 2 and 4 on the GPT-2 layout: exchange + adamw_nm step
    on the owned shard, unfused vs fused into the decode emit; and a synthetic
    backward pass (3 bf16 GEMMs per block) with the exchange one-shot after it
    vs overlapped with it (tagc_overlap_*)."""
    torch, ctx, shards, world = rig.torch, S["ctx"], S["shards"], rig.world
    grad, acc, out, owned = S["grad"], S["acc"], S["out"], S["owned"]
    params = torch.randn(max(owned, 1), device=rig.dev)
    adam_v = torch.zeros(max(owned, 1), device=rig.dev)
    reps = max(3, min(args.steps, 10))

    def timed(fn):
        for i in range(max(3, args.warmup)):  # eager, capture, first replay
            fn(i + 1)
        return rig.timed(lambda i: fn(i + 2), reps)

    def apply_only(k):
        ctx.apply_optimizer("adamw_nm", 1e-3, params, out, world, k, adam_v, weight_decay=0.01)

    def unfused(k):
        S["step"]()
        apply_only(k)

    def fused(k):
        ctx.tagc_reduce_shards_step(shards, grad, acc, params, "adamw_nm", 1e-3, k, adam_v=adam_v,
                                    weight_decay=0.01)

    owner = {"optimizer": "adamw_nm", "apply_only_ms": round(timed(apply_only), 4),
             "unfused_ms": round(timed(unfused), 4), "fused_ms": round(timed(fused), 4)}

    groups, off = [], 0
    for sp in S["specs"]:
        key = sp.name.split(".")[0] if sp.name.startswith("h") else ("final" if sp.name.startswith("ln_f") else "embed")
        if not groups or groups[-1][0] != key:
            groups.append([key, off, off])
        off += sp.param_count
        groups[-1][2] = off
    ranges = [(lo, hi) for _, lo, hi in groups]
    ranges[-1] = (ranges[-1][0], S["total"])  # the make_shards pad tail lands with the last block
    ga = torch.randn(8192, 768, device=rig.dev, dtype=torch.bfloat16)
    gb = torch.randn(768, 3072, device=rig.dev, dtype=torch.bfloat16)
    gc = torch.empty(8192, 3072, device=rig.dev, dtype=torch.bfloat16)
    grad_bw = torch.empty_like(grad)
    prod = torch.cuda.Stream(device=rig.local)

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

    def run(mode):
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        prod.wait_stream(rig.stream)
        b0.record(prod)
        if mode == "backward":
            backward()
            b1.record(prod)
        elif mode == "one_shot":
            rig.stream.wait_event(backward())
            ctx.tagc_reduce_shards(shards, grad_bw, acc, out, stats=False)
            b1.record(rig.stream)
        else:
            rig.stream.wait_event(b0)
            ctx.overlap_begin(shards, grad_bw, acc, out)
            backward(ctx.overlap_ready)
            ctx.overlap_finish()
            b1.record(rig.stream)
        return b0, b1

    overlap = {"producer": "3x bf16 mm 8192x768@768x3072 per block, 14 blocks, reverse order"}
    for mode in ("backward", "one_shot", "overlapped"):
        for _ in range(max(3, args.warmup)):
            run(mode)
        rig.barrier()
        evs = [run(mode) for _ in range(reps)]
        rig.barrier()
        overlap[mode + "_ms"] = round(rig.max_over_ranks(sum(a.elapsed_time(b) for a, b in evs) / reps), 4)
    return owner, overlap


def paper_w2_simulated(rig, tagc, args):
    """The paper setting (GPT-2, theta 98.75, r 10, 1-bit index) at W = 2 with
    both ranks simulated on this one GPU (tagc_reduce_shard_sim per shard:
    both ranks' encode, the rank-ordered sums, and the 1-bit merged index's
    FIFO-ordered peel, k_ord_loop). Not a multi-GPU number: the two ranks'
    work runs back to back on one device, so value = 2 x params x 4 B / t is
    a lower bound for two GPUs."""
    torch = rig.torch
    W = 2
    specs, cfg, shards = make_workload(tagc, "gpt2-paper", W)
    total = shards[-1].end
    n_params = sum(sp.param_count for sp in specs)
    grads = [synthetic_grad(torch, total, n_params, rig.dev, 2000 + r) for r in range(W)]
    accs = [torch.zeros(total, device=rig.dev) for _ in range(W)]
    ctx = tagc.Context(cfg, device=rig.local, stream=rig.stream.cuda_stream)

    def step():
        st = None
        for sh in shards:
            _, st = ctx.tagc_reduce_shard_sim(sh, [g[sh.begin:sh.end] for g in grads],
                                              [a[sh.begin:sh.end] for a in accs])
        return st

    for _ in range(max(args.warmup, 3)):
        st = step()
    rig.torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    n = max(args.steps, 5)
    ev[0].record(rig.stream)
    for _ in range(n):
        st = step()
    ev[1].record(rig.stream)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / n
    res = {"workload": WORKLOADS["gpt2-paper"][0] + ", W=2 simulated on one GPU (tagc_reduce_shard_sim)",
           "value": round(W * total * 4.0 / (ms * 1e-3) / 1e9, 3), "ms_per_step": round(ms, 4),
           "last_shard_peel": {"presence": st.presence, "unresolved": st.unresolved,
                               "index_lost": st.index_lost, "index_spurious": st.index_spurious,
                               "ordered_generations": ctx.last_peel_rounds()},
           "note": "both ranks on one device back to back (not a scaling point); the FIFO-ordered 1-bit peel "
                   "runs on the device (k_ord_loop)"}
    ctx.close()
    del grads, accs
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return res


def free_state(rig, S):
    S["ctx"].sync()
    S["ctx"].close()
    S.clear()
    rig.torch.cuda.synchronize()
    rig.torch.cuda.empty_cache()


def run_b200(args):
    rig = Rig(args)
    torch = rig.torch
    import paper_2504_05638_b200 as tagc

    head, S = measure_exchange(rig, tagc, args.workload, args)
    cfg, world = S["cfg"], rig.world
    hbm, peak_kind = peaks()
    fused_ms = S["span_ms"][0]
    fused_bytes = S["fused_bytes"]
    fused_bpe = fused_bytes / max(S["comp"], 1)
    achieved = fused_bytes / (fused_ms * 1e-3) / 1e9 if fused_ms > 0 else 0.0
    dec_bytes = S["owned_comp"] * decode_bytes_per_elem(cfg)
    dec_ms = S["span_ms"][1]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"fused_traffic_{args.workload}.json")
    if os.path.exists(tpath) and world == 1:  # captured on this workload at N=1
        try:
            with open(tpath) as f:
                traffic = json.load(f).get("bytes_per_launch")
        except Exception:
            traffic = None
    comparator = uncompressed_comparator(rig, S, args)
    e2e = end_to_end(rig, S, args) if not args.no_e2e and args.workload != "llama3-8b" else None
    clk = S["clk"]
    launches = head["launches_per_step"]
    config = workload_config(args.workload, world)
    config["parallelism"] = (f"dp{world}: one process per GPU, "
                             f"{'peer-memory pulls' if rig.exchange == 'peer' else 'NCCL reduce-scatter'}")
    free_state(rig, S)

    extras = {}
    if not args.no_extras and args.workload == "c4":
        for name in ("gpt2", "gpt2-paper"):
            r, S2 = measure_exchange(rig, tagc, name, args, full=False)
            r["workload"] = WORKLOADS[name][0]
            if name == "gpt2" and not args.no_owner_step:
                r["owner_step"], r["overlap"] = owner_step_and_overlap(rig, tagc, S2, args)
            free_state(rig, S2)
            extras[name] = r
        if world == 1:
            extras["gpt2-paper-w2-simulated"] = paper_w2_simulated(rig, tagc, args)

    result = {
        "metric": METRIC, "value": head["value"], "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic log-normal gradients (SyntheticStream distribution), generated on device",
        "config": config,
        "peel": head["peel"],
        "e2e": e2e if e2e is not None else {"skipped": "host buffers not allocated for this workload"},
        "roofline": {"kernel": "k_fused_tma (TMA-staged select / split / index / sketch scatter)",
                     "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": int(fused_bytes),
                     "bytes_per_elem": round(fused_bpe, 4),
                     "kernel_ms": round(fused_ms, 4),
                     "timed": "k_fused_tma launches: device span from %globaltimer stamps written by the "
                              "kernel (first CTA start to last CTA end), mean of the timed launches, max "
                              "over ranks"},
        "decode_roofline": {"kernels": "k_list .. k_emit (owner decode chain)", "bound": "hbm",
                            "achieved": round(dec_bytes / (dec_ms * 1e-3) / 1e9, 1) if dec_ms > 0 else None,
                            "peak": hbm, "unit": "GB/s",
                            "frac": round(dec_bytes / (dec_ms * 1e-3) / 1e9 / hbm, 4) if dec_ms > 0 else None,
                            "algorithmic_bytes": int(dec_bytes), "span_ms": round(dec_ms, 4)},
        "stages_ms": head["stages_ms"],
        "uncompressed_rs": comparator,
        "extras": extras,
        "gpu_launches": int(launches * args.steps),
        "clocks": clk,
    }
    if rig.share:
        result["config"]["shared_gpu_plumbing_check"] = \
            "all ranks on cuda:0 (TAGC_BENCH_SHARE_GPU=1): not a measurement"
    if not args.no_cpu_baseline:
        # rank 0 times the reference's CPU path on the host cores while the
        # other ranks wait (a reported baseline, outside every timed region)
        cb = cpu_baseline(args, world) if rig.rank == 0 else None
        rig.barrier()
        if cb is not None:
            result["cpu_baseline"] = cb
    if rig.rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        rig.barrier()
        rig.dist.destroy_process_group()


# --------------------------------------------------------------------------- reference arm
def reference_plan(name, world, sample_elems):
    """The reference's own make_shards (hook.cpp:30-61, through oracle/_ref) on
    the workload's layer list; for the single-bucket workload a bounded sample
    is the first `sample_elems` elements of each rank's bucket, sharded the
    same way. Returns (oracle Shards, elements per rank)."""
    import oracle as O

    ref = O.Ref()
    desc, layers, theta, ratio, width, policy, mcs = WORKLOADS[name]
    lay = layers()
    if name == "c4":
        lay = [("bucket", "feed_forward", min(sample_elems, C4_N))]
    counts = [c for _, _, c in lay]
    kinds = [O.KIND[k] for _, k, _ in lay]
    inv = {v: k for k, v in O.KIND.items()}
    slen, segs = ref.make_shards(counts, kinds, world, world)
    shards = []
    for sid in range(world):
        ss = [O.Segment(inv[k], b, e) for (s, k, b, e) in segs if s == sid]
        shards.append(O.Shard(sid, sid % world, sid * slen, (sid + 1) * slen, ss))
    per_rank = world * slen
    if name != "c4":  # layered workloads: the first segments up to the sample size
        out, used = [], 0
        for sh in shards:
            keep = []
            for s in sh.segments:
                if used >= sample_elems:
                    break
                keep.append(s)
                used += s.size
            if keep:
                out.append(O.Shard(sh.id, sh.owner, keep[0].begin, keep[-1].end, keep))
        shards, per_rank = out, used
    cfg = O.Config(theta, ratio, width, policy, True, SEED, 3, False, mcs)
    return ref, shards, per_rank, cfg


def reference_sample_elems(world):
    # ~2-3 s of reference work per step on 16 host cores: a quarter of the
    # 2^28 bucket at N = 1, the same total at every N
    return max(1 << 22, (1 << 26) // world)


def time_reference(name, world, steps, warmup, sample_elems):
    import oracle as O

    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    ref, shards, per_rank, cfg = reference_plan(name, world, sample_elems)
    end = max(s.end for s in shards)
    grads = list(ref.stream(end, 2024, count=world))  # the reference's SyntheticStream
    if warmup:
        ref.time_reduce_shards(shards, grads, cfg, reps=warmup)
    secs = ref.time_reduce_shards(shards, grads, cfg, reps=steps)
    t = float(secs.mean())
    value = world * per_rank * 4 / t / 1e9
    sample = (f"{'first ' if name != 'c4' else ''}{per_rank} elements per rank of {WORKLOADS[name][0]} "
              f"({'a 2^' + str(per_rank.bit_length() - 1) + '-element bucket' if name == 'c4' else 'leading segments'}"
              f", make_shards({world}, {world}) by the reference), tagc_reduce_shard with World({world}, "
              f"parallel), OMP_NUM_THREADS={os.environ['OMP_NUM_THREADS']}")
    return value, t, sample


def cpu_baseline(args, world):
    """The reference's own CPU path (oracle/_ref) on the host cores, bounded."""
    import oracle as O

    if not O.Ref.available():
        return {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    value, t, sample = time_reference(args.workload, world, 2, 0, reference_sample_elems(world))
    return {"value": round(value, 5), "unit": "GB/s", "cores": int(os.environ.get("OMP_NUM_THREADS")),
            "cpu_model": cpu_model(), "kind": "reference", "sample": sample, "seconds_per_step": round(t, 3)}


def run_reference(args):
    world = args.gpus
    if env_int("RANK", 0) != 0:
        return
    import oracle as O

    if not O.Ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtagc_ref.so not built"}))
        return
    value, t, sample = time_reference(args.workload, world, args.steps, max(0, min(args.warmup, 1)),
                                      reference_sample_elems(world))
    config = workload_config(args.workload, world)
    config["parallelism"] = f"reference World({world}, parallel): in-process ranks on the host cores"
    cores = int(os.environ.get("OMP_NUM_THREADS"))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic SyntheticStream gradients (the reference's own generator)",
        "config": config,
        "cpu_baseline": {"value": round(value, 5), "unit": "GB/s", "cores": cores, "cpu_model": cpu_model(),
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 5), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# --------------------------------------------------------------------------- launch
def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS),
                    help="c4 (BASELINE config 4: one 2^28 bucket, the default line), gpt2 / gpt2-paper "
                         "(config 2's layout), llama3-8b (config 3's layout)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="N>1 collective: grouped ncclReduceScatter, or pulls over peer memory")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the GPT-2 extra lines")
    ap.add_argument("--no-owner-step", action="store_true", help="skip the owner-step / overlap timings")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        # self-launch: one process per GPU under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
        sys.exit(subprocess.call(cmd + sys.argv[1:]))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
