"""Two (or more) processes, one GPU: the peer-memory exchange with its regions
mapped across processes through CUDA IPC (tagc_ctx_peer_open), the path
bench.py --exchange peer takes on an 8-GPU box, checked against the CPU
oracle on rank 0. Launched by tests/test_gpu_ipc.py:

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port P tools/peer_ipc_check.py [--steps 3] [--width 4]

Host plumbing (handle exchange, result gathering) uses gloo; every rank
uses cuda:0 (a test arrangement: production has one GPU per rank)."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402  (checker only)
import paper_2504_05638_b200 as tagc  # noqa: E402

SPECS = [
    ("wte", "embedding", 200_000), ("h0.ln_1", "norm", 512), ("h0.attn.c_attn", "attention_qkv", 98_304),
    ("h0.attn.c_proj", "attention_out_proj", 65_536), ("h0.mlp.c_fc", "feed_forward", 262_144),
    ("h0.mlp.c_fc.bias", "bias", 1_024), ("h0.mlp.c_proj", "feed_forward", 262_144), ("lm_head", "lm_head", 120_001),
]


def lognormal(n, seed):
    rng = np.random.default_rng(seed)
    mag = np.exp(rng.standard_normal(n, dtype=np.float32))
    return np.where(rng.integers(0, 2, n, dtype=np.int8) == 1, -mag, mag).astype(np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--width", type=int, default=4)
    args = ap.parse_args()
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    specs = [tagc.LayerSpec(n, k, c) for n, k, c in SPECS]
    shards = tagc.make_shards(specs, world, world)
    total = shards[-1].end
    theta = 99.0 if args.width == 4 else 98.75
    cfg = tagc.CompressionConfig(theta=theta, ratio=10, index_width=args.width, policy="non_attention_linear",
                                 include_out_proj=True, seed=77)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = tagc.Context(cfg, world_size=world, rank=rank, device=0, stream=stream.cuda_stream)
    handles = [None] * world
    dist.all_gather_object(handles, ctx.peer_prepare(shards))
    ctx.peer_open(handles)
    acc = torch.zeros(total, device="cuda")
    owned = [s for s in shards if s.owner == rank]
    outs = []
    for step in range(args.steps):
        g = torch.from_numpy(lognormal(total, 900 + 10 * step + rank)).cuda()
        out, st = ctx.tagc_reduce_shards(shards, g, acc, stats=True)
        outs.append(out.cpu().numpy().copy())
    accs = [None] * world
    all_outs = [None] * world
    dist.all_gather_object(accs, acc.cpu().numpy())
    dist.all_gather_object(all_outs, outs)
    if rank == 0:
        ocfg = O.Config(cfg.theta, cfg.ratio, cfg.index_width, cfg.policy, cfg.include_out_proj, cfg.seed,
                        cfg.sketch_rows, cfg.allow_low_theta, cfg.min_compress_segment)
        orc = O.Oracle()
        oacc = [np.zeros(total, np.float32) for _ in range(world)]
        worst = 0.0
        for step in range(args.steps):
            grads = [lognormal(total, 900 + 10 * step + r) for r in range(world)]
            refs = {}
            for sh in shards:
                osh = O.Shard(sh.id, sh.owner, sh.begin, sh.end,
                              [O.Segment(s.kind, s.begin, s.end, s.name) for s in sh.segments])
                a = [oacc[r][sh.begin:sh.end].copy() for r in range(world)]
                ref, _ = orc.tagc_reduce_shard(osh, [grads[r][sh.begin:sh.end] for r in range(world)], a, ocfg)
                for r in range(world):
                    oacc[r][sh.begin:sh.end] = a[r]
                refs[sh.id] = ref.copy()
            for o in range(world):
                mine = [s for s in shards if s.owner == o]
                ref = np.concatenate([refs[s.id] for s in mine])
                got = all_outs[o][step][:ref.size]
                scale = float(np.abs(ref).max())
                err = float(np.max(np.abs(got.astype(np.float64) - ref) / np.maximum(np.abs(ref), scale)))
                worst = max(worst, err)
                assert err <= 1e-5, (step, o, err)
        for r in range(world):
            assert np.array_equal(accs[r].view(np.uint32), oacc[r].view(np.uint32)), r
        print(f"IPC peer exchange OK: world={world} steps={args.steps} width={args.width} "
              f"max_rel_err={worst:.2e}", flush=True)
    dist.barrier()
    del owned
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
