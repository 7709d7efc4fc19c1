"""GPU parity of the owner-side consumer that follows the exchange in the
reference's training loop: the mean over ranks and the
optimizer step on the decoded shard (train.cpp:355-359, apply_optimizer
:202-220), bit-exact against the oracle's fp32 loop (which the CPU suite pins
to the reference's scale_sub_inplace and to an fp32 restatement of adamw_nm),
and the parameter all-gather's ledger row (train.cpp:364)."""
import numpy as np
import pytest
import torch

import paper_2504_05638_b200 as tagc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("optimizer,world,n", [("sgd", 1, 4097), ("sgd", 4, 1_000_003),
                                               ("adamw_nm", 2, 65_536), ("adamw_nm", 8, 3_000_017)])
def test_apply_optimizer_matches_oracle(orc, ctx, optimizer, world, n):
    kind = 0 if optimizer == "sgd" else 1
    rng = np.random.default_rng(n)
    p = rng.standard_normal(n).astype(np.float32)
    v = np.zeros(n, np.float32)
    p_d, v_d = torch.from_numpy(p.copy()).to(DEV), torch.zeros(n, device=DEV)
    lr, wd = 0.01, (0.1 if kind else 0.0)
    for step in range(1, 5):
        dec = (rng.standard_normal(n) * world).astype(np.float32)
        dec[rng.integers(0, n, n // 10)] = 0.0
        dec_d = torch.from_numpy(dec).to(DEV)
        ctx.apply_optimizer(optimizer, lr, p_d, dec_d, world, step, v_d if kind else None, weight_decay=wd)
        orc.apply_optimizer(kind, lr, wd, world, step, p, dec.copy(), v if kind else None)
        torch.cuda.synchronize()
        assert np.array_equal(bits(p_d.cpu().numpy()), bits(p)), (optimizer, step)
        if kind:
            assert np.array_equal(bits(v_d.cpu().numpy()), bits(v)), step
        # decoded is read only
        assert np.array_equal(bits(dec_d.cpu().numpy()), bits(dec))


def test_exchange_then_owner_step(orc):
    """One training-loop step at W = 1 through the public calls: exchange the
    shard, then the owner's adamw_nm step on the decoded gradient, then the
    (single-rank) parameter all-gather, which must leave params unchanged and
    record the reference's params/allgather row."""
    n = 1 << 20
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="all_layers", seed=77,
                                 min_compress_segment=1)
    shards = [tagc.ShardSpec(0, 0, 0, n, [tagc.LayerSegment("bucket", "feed_forward", 0, n)])]
    c = tagc.Context(cfg, device=0)
    rng = np.random.default_rng(11)
    grad = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).to(DEV)
    acc = torch.zeros(n, device=DEV)
    p0 = rng.standard_normal(n).astype(np.float32)
    params, v = torch.from_numpy(p0.copy()).to(DEV), torch.zeros(n, device=DEV)
    out, _ = c.tagc_reduce_shards(shards, grad, acc)
    dec = out.cpu().numpy()
    c.apply_optimizer("adamw_nm", 0.01, params, out, 1, 1, v, weight_decay=0.1)
    c.ledger_reset()
    c.allgather_params(params)
    c.sync()
    p_ref, v_ref = p0.copy(), np.zeros(n, np.float32)
    orc.apply_optimizer(1, 0.01, 0.1, 1, 1, p_ref, dec.copy(), v_ref)
    assert np.array_equal(bits(params.cpu().numpy()), bits(p_ref))
    assert np.array_equal(bits(v.cpu().numpy()), bits(v_ref))
    assert "params/allgather" in c.ledger_csv()
    with pytest.raises(tagc.TagcInvalidArgument):
        c.apply_optimizer("adamw_nm", 0.01, params, out, 1, 0, v)  # step counts from 1
    with pytest.raises(tagc.TagcInvalidArgument):
        c.apply_optimizer("lamb", 0.01, params, out, 1, 1, v)


SPECS = [
    ("wte", "embedding", 200_000), ("wpe", "positional_embedding", 16_384),
    ("h0.ln_1", "norm", 512), ("h0.attn.c_attn", "attention_qkv", 98_304),
    ("h0.attn.c_proj", "attention_out_proj", 65_536), ("h0.mlp.c_fc", "feed_forward", 262_144),
    ("h0.mlp.c_fc.bias", "bias", 1_024), ("h0.mlp.c_proj", "feed_forward", 262_144),
    ("ln_f", "norm", 512), ("lm_head", "lm_head", 120_001),
]


def _lognormal(n, seed):
    rng = np.random.default_rng(seed)
    mag = np.exp(rng.standard_normal(n, dtype=np.float32))
    return np.where(rng.integers(0, 2, n, dtype=np.int8) == 1, -mag, mag).astype(np.float32)


def _check_step(orc, ocfg, shards, owned, grads, oacc, outs, params0, v0, params, v, kind, world, step):
    """The fused step stored the decoded shard too (out given): the update
    must be exactly the oracle's optimizer applied to those values, and the
    values must be the oracle's decoded shard within the 1e-5 tolerance."""
    import oracle as O
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
        dec = outs[o].cpu().numpy()
        ref = np.concatenate([refs[s.id] for s in owned[o]])
        scale = float(np.abs(ref).max())
        assert float(np.max(np.abs(dec.astype(np.float64) - ref) / np.maximum(np.abs(ref), scale))) <= 1e-5
        p_ref, v_ref = params0[o].copy(), v0[o].copy()
        orc.apply_optimizer(kind, 0.01, 0.1 if kind else 0.0, world, step, p_ref, dec.copy(),
                            v_ref if kind else None)
        assert np.array_equal(bits(params[o].cpu().numpy()), bits(p_ref)), (o, step)
        if kind:
            assert np.array_equal(bits(v[o].cpu().numpy()), bits(v_ref)), (o, step)
        params0[o], v0[o] = p_ref, v_ref


@pytest.mark.parametrize("optimizer", ["sgd", "adamw_nm"])
def test_fused_step_w1(orc, optimizer):
    """tagc_reduce_shards_step at W = 1 (decode emit and the raw-segment side
    copy both carry the optimizer epilogue), two steps, then a third step
    without a decoded output (out=None) against the same update computed
    from a run that stores it (1e-5 tolerance: the sketch's float REDs are
    order-nondeterministic across runs)."""
    import oracle as O
    kind = 0 if optimizer == "sgd" else 1
    specs = [tagc.LayerSpec(n, k, c) for n, k, c in SPECS]
    shards = tagc.make_shards(specs, 1, 1)
    total = shards[-1].end
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="non_attention_linear",
                                 include_out_proj=True, seed=77)
    ocfg = O.Config(cfg.theta, cfg.ratio, cfg.index_width, cfg.policy, cfg.include_out_proj, cfg.seed,
                    cfg.sketch_rows, cfg.allow_low_theta, cfg.min_compress_segment)
    c = tagc.Context(cfg, device=0)
    rng = np.random.default_rng(5)
    params0 = [rng.standard_normal(total).astype(np.float32)]
    v0 = [np.zeros(total, np.float32)]
    params = [torch.from_numpy(params0[0].copy()).to(DEV)]
    v = [torch.zeros(total, device=DEV)]
    acc = torch.zeros(total, device=DEV)
    oacc = [np.zeros(total, np.float32)]
    out = torch.empty(total, device=DEV)
    for step in (1, 2):
        grads = [_lognormal(total, 40 + step)]
        c.tagc_reduce_shards_step(shards, torch.from_numpy(grads[0]).to(DEV), acc, params[0], optimizer, 0.01, step,
                                  adam_v=v[0] if kind else None, weight_decay=0.1 if kind else 0.0, out=out)
        c.sync()
        _check_step(orc, ocfg, shards, [shards], grads, oacc, [out], params0, v0, params, v, kind, 1, step)
    # out=None: same update as a twin that stores the decoded shard
    g = torch.from_numpy(_lognormal(total, 99)).to(DEV)
    acc2, p2, v2 = acc.clone(), params[0].clone(), v[0].clone()
    c.tagc_reduce_shards_step(shards, g, acc, params[0], optimizer, 0.01, 3, adam_v=v[0] if kind else None,
                              weight_decay=0.1 if kind else 0.0)
    c.tagc_reduce_shards_step(shards, g, acc2, p2, optimizer, 0.01, 3, adam_v=v2 if kind else None,
                              weight_decay=0.1 if kind else 0.0, out=out)
    c.sync()
    assert torch.equal(acc.view(torch.int32), acc2.view(torch.int32))
    d = (params[0] - p2).abs().max().item()
    assert d <= 1e-5 * max(1.0, p2.abs().max().item()), d


@pytest.mark.parametrize("optimizer", ["sgd", "adamw_nm"])
def test_fused_step_peer_w2(orc, optimizer):
    """W = 2 over the peer-memory exchange (both ranks in this process, one
    host thread each): the owners' raw-segment unpack and decode emit carry
    the optimizer with the mean over 2 ranks."""
    import threading

    import oracle as O
    kind = 0 if optimizer == "sgd" else 1
    world = 2
    specs = [tagc.LayerSpec(n, k, c) for n, k, c in SPECS]
    shards = tagc.make_shards(specs, world, world)
    total = shards[-1].end
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="non_attention_linear",
                                 include_out_proj=True, seed=77)
    ocfg = O.Config(cfg.theta, cfg.ratio, cfg.index_width, cfg.policy, cfg.include_out_proj, cfg.seed,
                    cfg.sketch_rows, cfg.allow_low_theta, cfg.min_compress_segment)
    streams = [torch.cuda.Stream() for _ in range(world)]
    ctxs = []
    for r in range(world):
        with torch.cuda.stream(streams[r]):
            ctxs.append(tagc.Context(cfg, world_size=world, rank=r, device=0))
    for c in ctxs:
        c.peer_prepare(shards)
    for c in ctxs:
        c.peer_attach_local(ctxs)
    owned = [[s for s in shards if s.owner == r] for r in range(world)]
    sizes = [sum(s.size() for s in owned[r]) for r in range(world)]
    rng = np.random.default_rng(8)
    params0 = [rng.standard_normal(sizes[r]).astype(np.float32) for r in range(world)]
    v0 = [np.zeros(sizes[r], np.float32) for r in range(world)]
    params = [torch.from_numpy(p.copy()).to(DEV) for p in params0]
    v = [torch.zeros(sizes[r], device=DEV) for r in range(world)]
    acc = [torch.zeros(total, device=DEV) for _ in range(world)]
    oacc = [np.zeros(total, np.float32) for _ in range(world)]
    outs = [torch.empty(sizes[r], device=DEV) for r in range(world)]
    g_d = [torch.empty(total, device=DEV) for _ in range(world)]
    torch.cuda.synchronize()
    for step in (1, 2):
        grads = [_lognormal(total, 300 + 10 * step + r) for r in range(world)]
        for r in range(world):
            g_d[r].copy_(torch.from_numpy(grads[r]))
        torch.cuda.synchronize()
        errs = [None] * world

        def run(r):
            try:
                ctxs[r].tagc_reduce_shards_step(shards, g_d[r], acc[r], params[r], optimizer, 0.01, step,
                                                adam_v=v[r] if kind else None, weight_decay=0.1 if kind else 0.0,
                                                out=outs[r])
                ctxs[r].sync()
            except Exception as e:  # surfaced below
                errs[r] = e

        threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for e in errs:
            if e is not None:
                raise e
        _check_step(orc, ocfg, shards, owned, grads, oacc, outs, params0, v0, params, v, kind, world, step)
