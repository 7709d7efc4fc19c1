"""GPU parity of the one-process-per-GPU exchange at W > 1, on one GPU: every
rank's context runs tagc_reduce_shards_begin / _end (the NCCL-world code
path with the collective supplied by the caller), and the test performs the
reduce-scatter the way the reference's World does - fp32 sums of the owner
blocks in ascending rank order and wrapping u32 sums of the index blocks
(collectives.cpp:127-166). Compared with the CPU oracle's tagc_reduce_shard
(reference hook.cpp:98-200) shard by shard: residual accumulators of every
rank bit-exact, peel statistics exact, the owner's decoded shards within the
reference's 1e-5 tolerance (roundtrip.cpp:119-137). With a 1-bit index the
merged words carry (index.cpp:80-93) and the decoder's FIFO-ordered peel must
reproduce the reference's carry-corrupted values."""
import threading

import numpy as np
import pytest
import torch

import oracle as O
import paper_2504_05638_b200 as tagc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"

SPECS = [
    ("wte", "embedding", 200_000), ("wpe", "positional_embedding", 16_384),
    ("h0.ln_1", "norm", 512), ("h0.attn.c_attn", "attention_qkv", 98_304),
    ("h0.attn.c_proj", "attention_out_proj", 65_536), ("h0.mlp.c_fc", "feed_forward", 262_144),
    ("h0.mlp.c_fc.bias", "bias", 1_024), ("h0.mlp.c_proj", "feed_forward", 262_144),
    ("h1.mlp.c_fc", "feed_forward", 131_072), ("ln_f", "norm", 512), ("lm_head", "lm_head", 120_000),
]


def lognormal(n, seed):
    rng = np.random.default_rng(seed)
    mag = np.exp(rng.standard_normal(n, dtype=np.float32))
    return np.where(rng.integers(0, 2, n, dtype=np.int8) == 1, -mag, mag).astype(np.float32)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def check_close(got, ref, tol=1e-5):
    scale = float(np.abs(ref).max())
    if scale == 0.0:
        assert np.array_equal(bits(got), bits(ref))
        return
    err = float(np.max(np.abs(got.astype(np.float64) - ref) / np.maximum(np.abs(ref), scale)))
    assert err <= tol, err


@pytest.mark.parametrize("world,width,theta,steps", [
    (2, 4, 99.0, 2), (4, 4, 99.0, 1), (8, 4, 99.5, 1), (3, 4, 98.0, 1), (2, 1, 98.75, 2), (4, 1, 99.0, 1),
])
def test_split_exchange_matches_oracle(orc, world, width, theta, steps):
    specs = [tagc.LayerSpec(n, k, c) for n, k, c in SPECS]
    shards = tagc.make_shards(specs, world, world)
    total = shards[-1].end
    ratio = 10 if theta >= 98.75 else 4
    cfg = tagc.CompressionConfig(theta=theta, ratio=ratio, index_width=width, policy="non_attention_linear",
                                 include_out_proj=True, seed=77)
    ocfg = O.Config(cfg.theta, cfg.ratio, cfg.index_width, cfg.policy, cfg.include_out_proj, cfg.seed,
                    cfg.sketch_rows, cfg.allow_low_theta, cfg.min_compress_segment)
    _, Bf, Bu = tagc.plan_exchange(cfg, shards, world, 0)
    ctxs = [tagc.Context(cfg, world_size=world, rank=r, device=0) for r in range(world)]
    owned = [[s for s in shards if s.owner == r] for r in range(world)]
    acc = [torch.zeros(total, device=DEV) for _ in range(world)]
    oacc = [np.zeros(total, np.float32) for _ in range(world)]
    for step in range(steps):
        grads = [lognormal(total, 1000 * step + r) for r in range(world)]
        send_f = [torch.zeros(world * Bf, device=DEV) for _ in range(world)]
        send_u = [torch.zeros(world * Bu, dtype=torch.int32, device=DEV) for _ in range(world)]
        outs = [torch.full((max(1, sum(s.size() for s in owned[r])),), float("nan"), device=DEV)
                for r in range(world)]
        sup = [torch.zeros(world * Bu * 32, dtype=torch.uint8, device=DEV) for _ in range(world)]
        for r in range(world):
            bf, bu = ctxs[r].reduce_shards_begin(shards, torch.from_numpy(grads[r]).to(DEV), acc[r], outs[r],
                                                 send_f[r], send_u[r])
            assert (bf, bu) == (Bf, Bu)
            if width == 1:  # index_lost / _spurious need the OR of the ranks' supports
                assert ctxs[r].reduce_shards_support(sup[r]) == Bu * 32
        stats = []
        for o in range(world):  # the reduce-scatter, ascending rank order
            rf = send_f[0][o * Bf:(o + 1) * Bf].clone()
            ru = send_u[0][o * Bu:(o + 1) * Bu].to(torch.int64)
            rs = sup[0][o * Bu * 32:(o + 1) * Bu * 32].clone()
            for r in range(1, world):
                rf += send_f[r][o * Bf:(o + 1) * Bf]
                ru += send_u[r][o * Bu:(o + 1) * Bu].to(torch.int64)
                rs = torch.maximum(rs, sup[r][o * Bu * 32:(o + 1) * Bu * 32])
            ru = ((ru & 0xFFFFFFFF) ^ 0x80000000).sub(0x80000000).to(torch.int32)  # wrap to u32 bits
            stats.append(ctxs[o].reduce_shards_end(rf, ru, recv_support=rs if width == 1 else None))
        torch.cuda.synchronize()
        # oracle, shard by shard (accumulators are updated in place per shard slice)
        refs, rsts = {}, {}
        for sh in shards:
            osh = O.Shard(sh.id, sh.owner, sh.begin, sh.end,
                          [O.Segment(s.kind, s.begin, s.end, s.name) for s in sh.segments])
            g = [grads[r][sh.begin:sh.end] for r in range(world)]
            a = [oacc[r][sh.begin:sh.end].copy() for r in range(world)]
            ref, rst = orc.tagc_reduce_shard(osh, g, a, ocfg)
            for r in range(world):
                oacc[r][sh.begin:sh.end] = a[r]
            refs[sh.id], rsts[sh.id] = ref.copy(), dict(rst)
        for r in range(world):
            assert np.array_equal(bits(acc[r].cpu().numpy()), bits(oacc[r])), (step, r)
        for o in range(world):
            got = outs[o].cpu().numpy()
            off = 0
            for sh in owned[o]:
                check_close(got[off:off + sh.size()], refs[sh.id])
                off += sh.size()
            for k in ("presence", "peeled", "unresolved", "index_lost", "index_spurious"):
                assert getattr(stats[o], k) == sum(rsts[s.id][k] for s in owned[o]), (k, o, stats[o])
        if width == 1:
            assert sum(st.index_lost + st.index_spurious for st in stats) > 0  # carries did happen


def test_split_exchange_without_support_flags_unavailable():
    """1-bit index, split API, no support blocks: the diagnostic cannot be
    computed and says so instead of reporting 0."""
    world, n = 2, 1 << 16
    shards = [tagc.ShardSpec(i, i, i * n, (i + 1) * n, [tagc.LayerSegment("b", "feed_forward", i * n, (i + 1) * n)])
              for i in range(world)]
    cfg = tagc.CompressionConfig(theta=98.75, ratio=10, index_width=1, policy="all_layers", seed=77)
    _, Bf, Bu = tagc.plan_exchange(cfg, shards, world, 0)
    ctxs = [tagc.Context(cfg, world_size=world, rank=r, device=0) for r in range(world)]
    sf = [torch.zeros(world * Bf, device=DEV) for _ in range(world)]
    su = [torch.zeros(world * Bu, dtype=torch.int32, device=DEV) for _ in range(world)]
    outs = [torch.empty(n, device=DEV) for _ in range(world)]
    for r in range(world):
        g = torch.from_numpy(lognormal(world * n, r)).to(DEV)
        ctxs[r].reduce_shards_begin(shards, g, torch.zeros(world * n, device=DEV), outs[r], sf[r], su[r])
    st = ctxs[0].reduce_shards_end(sf[0][:Bf] + sf[1][:Bf], su[0][:Bu] + su[1][:Bu])
    assert st.index_lost == tagc.STAT_UNAVAILABLE and st.index_spurious == tagc.STAT_UNAVAILABLE
    ctxs[1].reduce_shards_end(sf[0][Bf:] + sf[1][Bf:], su[0][Bu:] + su[1][Bu:], stats=False)
    torch.cuda.synchronize()


@pytest.mark.parametrize("world,width,steps", [(2, 4, 5), (4, 4, 2), (2, 1, 2)])
def test_peer_exchange_matches_oracle(orc, world, width, steps):
    """Pull-mode exchange over peer memory (tagc_ctx_peer_*): all ranks as
    contexts of this process on one GPU, each on its own stream so that the
    step flags are raised and awaited concurrently. Five steps at W=2 cover
    both send sets, the CUDA-graph capture (third call) and replay (fifth)."""
    specs = [tagc.LayerSpec(n, k, c) for n, k, c in SPECS]
    shards = tagc.make_shards(specs, world, world)
    total = shards[-1].end
    theta = 99.0 if width == 4 else 98.75
    cfg = tagc.CompressionConfig(theta=theta, ratio=10, index_width=width, policy="non_attention_linear",
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
    acc = [torch.zeros(total, device=DEV) for _ in range(world)]
    g_d = [torch.empty(total, device=DEV) for _ in range(world)]
    outs = [torch.empty(max(1, sum(s.size() for s in owned[r])), device=DEV) for r in range(world)]
    oacc = [np.zeros(total, np.float32) for _ in range(world)]
    torch.cuda.synchronize()
    for step in range(steps):
        grads = [lognormal(total, 7000 + 100 * step + r) for r in range(world)]
        for r in range(world):
            g_d[r].copy_(torch.from_numpy(grads[r]))
        torch.cuda.synchronize()
        # one host thread per rank, as in a real deployment (one process per
        # GPU): the 1-bit path's ordered peel synchronises its own stream
        # between generations, which must not stall the other ranks' enqueues
        errs = [None] * world

        want_stats = step == min(1, steps - 1)  # eager; the graph capture / replay steps stay stat-less
        stats = [None] * world

        def run(r):
            try:
                _, stats[r] = ctxs[r].tagc_reduce_shards(shards, g_d[r], acc[r], outs[r], stats=want_stats)
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
        refs, rsts = {}, {}
        for sh in shards:
            osh = O.Shard(sh.id, sh.owner, sh.begin, sh.end,
                          [O.Segment(s.kind, s.begin, s.end, s.name) for s in sh.segments])
            a = [oacc[r][sh.begin:sh.end].copy() for r in range(world)]
            ref, rst = orc.tagc_reduce_shard(osh, [grads[r][sh.begin:sh.end] for r in range(world)], a, ocfg)
            for r in range(world):
                oacc[r][sh.begin:sh.end] = a[r]
            refs[sh.id], rsts[sh.id] = ref.copy(), dict(rst)
        if want_stats:  # index_lost / _spurious from the peers' send blocks (hook.cpp:176-188)
            for o in range(world):
                for k in ("presence", "peeled", "unresolved", "index_lost", "index_spurious"):
                    assert getattr(stats[o], k) == sum(rsts[s.id][k] for s in owned[o]), (k, o, stats[o])
        for r in range(world):
            assert np.array_equal(bits(acc[r].cpu().numpy()), bits(oacc[r])), (step, r)
        for o in range(world):
            got = outs[o].cpu().numpy()
            off = 0
            for sh in owned[o]:
                check_close(got[off:off + sh.size()], refs[sh.id])
                off += sh.size()


@pytest.mark.parametrize("world,width,theta,steps", [(2, 4, 99.0, 2), (3, 1, 98.75, 1)])
def test_split_exchange_deferred_scatter(orc, monkeypatch, world, width, theta, steps):
    """The region-ordered sketch scatter (kDeferScatter, used for sketches
    beyond L2) forced on every segment: same parity bar against the oracle."""
    monkeypatch.setenv("TAGC_DEFER_SCATTER_BYTES", "0")
    test_split_exchange_matches_oracle(orc, world, width, theta, steps)


@pytest.mark.parametrize("world,width,theta,steps", [(2, 4, 99.0, 2), (3, 1, 98.75, 1)])
def test_split_exchange_deferred_scatter_groups(orc, monkeypatch, world, width, theta, steps):
    """The deferred scatter in several groups (every segment deferred, groups
    capped at 2^14 floats of sketch span: one launch_deferred_scatter call per
    group, each with its own bins and fill counters over the shared record
    buffers): same parity bar against the oracle."""
    monkeypatch.setenv("TAGC_DEFER_SCATTER_BYTES", "0")
    monkeypatch.setenv("TAGC_DS_GROUP_SPAN", str(1 << 14))
    test_split_exchange_matches_oracle(orc, world, width, theta, steps)


@pytest.mark.parametrize("world,width,theta,steps", [(2, 4, 99.0, 2)])
def test_split_exchange_deferred_scatter_overflow(orc, monkeypatch, world, width, theta, steps):
    """The deferred scatter's overflow path: bins capped at a quarter of their
    mean load (TAGC_DS_TIGHT), so most updates go to the overflow list and
    are added with REDs after the shared-memory apply: same parity bar."""
    monkeypatch.setenv("TAGC_DEFER_SCATTER_BYTES", "0")
    monkeypatch.setenv("TAGC_DS_TIGHT", "1")
    test_split_exchange_matches_oracle(orc, world, width, theta, steps)
