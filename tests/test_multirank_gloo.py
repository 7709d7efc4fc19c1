"""CPU, world_size 2 over gloo: the N>1 exchange layout.

Each process plays one rank of tagc_reduce_shards: it lays out its encoded
compressed segments (index words + count sketch) and raw segments in the
owner-major send blocks the C++ planner (tagc_plan_exchange) assigns, the
blocks are summed across ranks (gloo all_reduce == reduce-scatter + slice),
and the owner decodes its slice. The codec arithmetic is done by the CPU
oracle (test infrastructure); what is under test is the planner's layout and
the exchange semantics, which must reproduce the single-process reference
world (tagc_reduce_shard, hook.cpp:98-200) bit-for-bit at W = 2."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2504_05638_b200 as tagc

WORLD = 2


def _specs():
    # a small GPT-2-shaped model: the reference's own layer kinds and order
    return tagc.gpt2_specs(layers=2, d_model=64, ffn_mult=4, vocab=700, ctx=64)


def _cfg(width):
    return tagc.CompressionConfig(theta=98.75, ratio=10, index_width=width,
                                  policy="non_attention_linear", seed=77)


def _ocfg(c):
    return O.Config(c.theta, c.ratio, c.index_width, c.policy, c.include_out_proj, c.seed,
                    c.sketch_rows, c.allow_low_theta, c.min_compress_segment)


def _grads(total):
    return list(O.Oracle().stream(total, 4242, count=WORLD))


def _worker(rank, port, width, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        orc = O.Oracle()
        cfg = _cfg(width)
        shards = tagc.make_shards(_specs(), WORLD, WORLD)
        total = shards[-1].end
        g = _grads(total)[rank]
        acc = np.zeros(total, np.float32)
        plan, bf, bu = tagc.plan_exchange(cfg, shards, WORLD, rank)
        send_f = np.zeros(WORLD * bf, np.float32)
        send_u = np.zeros(WORLD * bu, np.uint32)
        for p in plan:
            sh = shards[p["shard"]]
            lo, n, o = sh.begin + p["lo"], p["len"], p["owner"]
            if p["compressed"]:
                combined = g[lo:lo + n] + acc[lo:lo + n]
                sparse, residual, _, _ = orc.sparsify(combined, cfg.theta)
                acc[lo:lo + n] = residual
                words = orc.index_create(sparse, width)
                send_u[o * bu + p["word_off"]: o * bu + p["word_off"] + p["n_words"]] = words[: p["n_words"]]
                sk = orc.sketch_compress(sparse, cfg.ratio, cfg.seed, cfg.sketch_rows)
                send_f[o * bf + p["sk_off"]: o * bf + p["sk_off"] + sk.size] = sk
            else:
                send_f[o * bf + p["raw_off"]: o * bf + p["raw_off"] + n] = g[lo:lo + n]
        tf = torch.from_numpy(send_f)
        tu = torch.from_numpy(send_u.view(np.int32))
        dist.all_reduce(tf)  # wrapping int32 add == u32 word sum (kernels.cpp:65-84)
        dist.all_reduce(tu)
        recv_f = tf.numpy()[rank * bf:(rank + 1) * bf]
        recv_u = tu.numpy().view(np.uint32)[rank * bu:(rank + 1) * bu]
        owned = sum(s.size() for s in shards if s.owner == rank)
        out = np.zeros(owned, np.float32)
        for p in plan:
            if p["owner"] != rank:
                continue
            n = p["len"]
            if p["compressed"]:
                words = recv_u[p["word_off"]: p["word_off"] + p["n_words"]]
                pres = orc.presence(words, n, width)
                sk = recv_f[p["sk_off"]: p["sk_off"] + cfg.sketch_rows * p["buckets_per_row"]]
                vals, _, _ = orc.peeling_decompress(pres, sk, n, cfg.ratio, cfg.seed, cfg.sketch_rows)
                out[p["out_off"]: p["out_off"] + n] = vals
            else:
                out[p["out_off"]: p["out_off"] + n] = recv_f[p["raw_off"]: p["raw_off"] + n]
        results[rank] = (out, acc)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("width", [4, 1])
def test_two_rank_exchange_matches_single_process_reference(width):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(_free_port(), width, results), nprocs=WORLD, join=True)
    cfg = _cfg(width)
    shards = tagc.make_shards(_specs(), WORLD, WORLD)
    total = shards[-1].end
    grads = _grads(total)
    orc = O.Oracle()
    accs = [np.zeros(total, np.float32) for _ in range(WORLD)]
    for sh in shards:
        osh = O.Shard(sh.id, sh.owner, sh.begin, sh.end,
                      [O.Segment(s.kind, s.begin, s.end, s.name) for s in sh.segments])
        sl = [x[sh.begin:sh.end] for x in grads]
        ac = [a[sh.begin:sh.end].copy() for a in accs]
        ref, _ = orc.tagc_reduce_shard(osh, sl, ac, _ocfg(cfg))
        for r in range(WORLD):
            accs[r][sh.begin:sh.end] = ac[r]
        out, _ = results[sh.owner]
        off = sum(s.size() for s in shards[: sh.id] if s.owner == sh.owner)
        got = out[off: off + sh.size()]
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), sh.id
    for r in range(WORLD):
        assert np.array_equal(results[r][1].view(np.uint32), accs[r].view(np.uint32))
