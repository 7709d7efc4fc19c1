"""The reference's per-exchange diagnostics through the CUDA path
(hook.cpp:171-196): collect_audit / audit_exchanged_sum in the simulated world
and the one-process-per-GPU world, against the reference's own audit
(oracle/_ref ref_tagc_reduce_shard_audit), and the sticky error word: a NaN
found by an early encode batch survives later batches and calls until it is
reported (tagc_b200.h: tagc_ctx_sync)."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2504_05638_b200 as tagc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"

SPECS = [("wte", "embedding", 120_000), ("h0.qkv", "attention_qkv", 30_000), ("h0.ln", "norm", 700),
         ("h0.fc", "feed_forward", 90_000), ("h0.proj", "attention_out_proj", 20_000),
         ("h1.fc", "feed_forward", 65_536)]


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def lognormal(n, seed):
    rng = np.random.default_rng(seed)
    mag = np.exp(rng.standard_normal(n, dtype=np.float32))
    return np.where(rng.integers(0, 2, n, dtype=np.int8) == 1, -mag, mag).astype(np.float32)


def oshard(sh):
    return O.Shard(sh.id, sh.owner, sh.begin, sh.end, [O.Segment(s.kind, s.begin, s.end, s.name) for s in sh.segments])


@pytest.mark.parametrize("world,width", [(2, 4), (3, 1), (4, 4)])
def test_sim_audit_matches_reference(ref, world, width):
    specs = [tagc.LayerSpec(n, k, c) for n, k, c in SPECS]
    sh = tagc.make_shards(specs, 1, 1)[0]
    n = sh.size()
    theta = 99.0 if width == 4 else 98.75
    cfg = tagc.CompressionConfig(theta=theta, ratio=10, index_width=width, policy="non_attention_linear",
                                 include_out_proj=True, seed=77)
    ocfg = O.Config(theta, 10, width, "non_attention_linear", True, 77, 3, False, 1024)
    ctx = tagc.Context(cfg, device=0)
    acc = [torch.zeros(n, device=DEV) for _ in range(world)]
    oacc = [np.zeros(n, np.float32) for _ in range(world)]
    for step in range(2):  # the second step carries error feedback
        grads = [lognormal(n, 50 * step + r) for r in range(world)]
        out, st, audit = ctx.tagc_reduce_shard_sim_audit(sh, [torch.from_numpy(g).to(DEV) for g in grads], acc)
        _, raudit = ref.tagc_reduce_shard_audit(oshard(sh), grads, oacc, ocfg)
        torch.cuda.synchronize()
        for r in range(world):
            assert np.array_equal(bits(acc[r].cpu().numpy()), bits(oacc[r])), (step, r)
        # same fp32 adds in the same (ascending rank) order: bit-exact
        assert np.array_equal(bits(audit.cpu().numpy()), bits(raudit)), step
        assert np.count_nonzero(raudit) > 0


def test_world_audit_matches_reference(ref):
    """tagc_reduce_shards_audit at world size 1 (the NCCL-world code path):
    the owner's audit equals the reference's audit of the same shard."""
    specs = [tagc.LayerSpec(n, k, c) for n, k, c in SPECS]
    shards = tagc.make_shards(specs, 1, 1)
    total = shards[-1].end
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="non_attention_linear",
                                 include_out_proj=True, seed=77)
    ocfg = O.Config(99.0, 10, 4, "non_attention_linear", True, 77, 3, False, 1024)
    ctx = tagc.Context(cfg, device=0)
    acc = torch.zeros(total, device=DEV)
    oacc = [np.zeros(total, np.float32)]
    for step in range(2):
        g = lognormal(total, 900 + step)
        out, st, audit = ctx.tagc_reduce_shards_audit(shards, torch.from_numpy(g).to(DEV), acc)
        _, raudit = ref.tagc_reduce_shard_audit(oshard(shards[0]), [g], oacc, ocfg)
        assert np.array_equal(bits(audit.cpu().numpy()), bits(raudit)), step
        assert np.array_equal(bits(acc.cpu().numpy()), bits(oacc[0])), step


def test_nan_error_is_sticky_until_reported():
    """an encode batch must not clear the NaN flag an earlier batch
    (overlap) or an earlier asynchronous call raised."""
    n = 1 << 18
    specs = [tagc.LayerSpec("a", "feed_forward", n), tagc.LayerSpec("b", "feed_forward", n)]
    shards = tagc.make_shards(specs, 1, 1)
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="all_layers", seed=77)
    ctx = tagc.Context(cfg, device=0)
    grad = torch.ones(2 * n, device=DEV)
    grad[5] = float("nan")  # in the first segment
    acc = torch.zeros(2 * n, device=DEV)
    # overlap: the NaN batch first, a clean batch after it
    ctx.overlap_begin(shards, grad, acc)
    ctx.overlap_ready(0, n)
    ctx.overlap_ready(n, 2 * n)
    with pytest.raises(tagc.TagcInvalidArgument):
        ctx.overlap_finish(stats=True)
    # asynchronous calls without stats: the error survives the next clean call
    clean = torch.ones(2 * n, device=DEV)
    ctx.tagc_reduce_shards(shards, grad, acc, stats=False)
    ctx.tagc_reduce_shards(shards, clean, torch.zeros(2 * n, device=DEV), stats=False)
    with pytest.raises(tagc.TagcInvalidArgument):
        ctx.sync()
    # reported once: the context is clean again
    ctx.tagc_reduce_shards(shards, clean, torch.zeros(2 * n, device=DEV), stats=False)
    ctx.sync()


def test_api_rejects_bad_buffers():
    """wrong dtype / short / host tensors never reach the kernels."""
    n = 4096
    shards = tagc.make_shards([tagc.LayerSpec("a", "feed_forward", n)], 1, 1)
    ctx = tagc.Context(tagc.CompressionConfig(theta=99.0, ratio=10, seed=1, policy="all_layers"), device=0)
    good = torch.zeros(n, device=DEV)
    for bad in (torch.zeros(n // 2, device=DEV), torch.zeros(n, device=DEV, dtype=torch.float64),
                torch.zeros(n), torch.zeros(2 * n, device=DEV)[::2]):
        with pytest.raises(tagc.TagcInvalidArgument):
            ctx.tagc_reduce_shards(shards, bad, good.clone())
        with pytest.raises(tagc.TagcInvalidArgument):
            ctx.tagc_reduce_shards(shards, good, bad)
    with pytest.raises(tagc.TagcInvalidArgument):
        ctx.tagc_reduce_shards(shards, good, good.clone(), out=torch.zeros(10, device=DEV))
