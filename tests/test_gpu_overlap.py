"""GPU parity of the overlapped exchange (tagc_overlap_begin / _ready /
_finish): segments are encoded as a producer stream writes
the gradient layer by layer (the order of a backward pass), and the results
must be those of the one-shot tagc_reduce_shards: residual accumulators bit
for bit, peel statistics exactly, decoded shards within the reference's 1e-5
tolerance (the sketch's float reductions are order-nondeterministic) and the
raw segments bit for bit."""
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
    ("h1.mlp.c_fc", "feed_forward", 131_072), ("ln_f", "norm", 512), ("lm_head", "lm_head", 120_001),
]


def lognormal(n, seed):
    rng = np.random.default_rng(seed)
    mag = np.exp(rng.standard_normal(n, dtype=np.float32))
    return np.where(rng.integers(0, 2, n, dtype=np.int8) == 1, -mag, mag).astype(np.float32)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def check_close(got, ref, tol=1e-5):
    scale = float(np.abs(ref).max())
    err = float(np.max(np.abs(got.astype(np.float64) - ref) / np.maximum(np.abs(ref), scale)))
    assert err <= tol, err


def layer_ranges():
    out, off = [], 0
    for _, _, n in SPECS:
        out.append((off, off + n))
        off += n
    return out


def produce(src, dst, ranges, stream, ctx, chunks=None):
    """Writes dst from src range by range on `stream` (reverse layer order, as
    a backward pass produces them) and hands each range to the context."""
    for lo, hi in reversed(chunks or ranges):
        with torch.cuda.stream(stream):
            torch.cuda._sleep(20_000)  # the producer takes a while per layer
            dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        ctx.overlap_ready(lo, hi, ev)


@pytest.mark.parametrize("width,split", [(4, False), (4, True), (1, False)])
def test_overlap_w1_matches_one_shot(width, split):
    specs = [tagc.LayerSpec(n, k, c) for n, k, c in SPECS]
    shards = tagc.make_shards(specs, 1, 1)
    total = shards[-1].end
    cfg = tagc.CompressionConfig(theta=99.0 if width == 4 else 98.75, ratio=10, index_width=width,
                                 policy="non_attention_linear", include_out_proj=True, seed=77)
    src = torch.from_numpy(lognormal(total, 3)).to(DEV)
    # one-shot reference run
    c1 = tagc.Context(cfg, device=0)
    acc1 = torch.zeros(total, device=DEV)
    out1, st1 = c1.tagc_reduce_shards(shards, src, acc1)
    # overlapped run: the gradient buffer starts as garbage and is produced
    # while the context encodes
    c2 = tagc.Context(cfg, device=0)
    grad = torch.full((total,), float("nan"), device=DEV)
    acc2 = torch.zeros(total, device=DEV)
    producer = torch.cuda.Stream()
    torch.cuda.synchronize()
    out2 = c2.overlap_begin(shards, grad, acc2)
    ranges = layer_ranges()
    chunks = None
    if split:  # ranges that cut through segments: each is encoded once fully covered
        cuts = sorted({0, total} | {int(x) for x in np.random.default_rng(1).integers(1, total, 9)})
        chunks = list(zip(cuts[:-1], cuts[1:]))
    produce(src, grad, ranges, producer, c2, chunks)
    if split:  # the last chunks only cover segments partly: cover everything once more
        with torch.cuda.stream(producer):
            ev = torch.cuda.Event()
            ev.record(producer)
        c2.overlap_ready(0, total, ev)
    st2 = c2.overlap_finish(stats=True)
    torch.cuda.synchronize()
    assert torch.equal(acc1.view(torch.int32), acc2.view(torch.int32))
    assert st1 == st2
    o1, o2 = out1.cpu().numpy(), out2.cpu().numpy()
    check_close(o2, o1)
    for sh in shards:
        for s in sh.segments:
            if not tagc.kind_compressible(s.kind, cfg.policy, cfg.include_out_proj):
                assert np.array_equal(bits(o2[s.begin:s.end]), bits(o1[s.begin:s.end])), s.name


def test_overlap_finish_covers_unannounced_segments():
    specs = [tagc.LayerSpec(n, k, c) for n, k, c in SPECS]
    shards = tagc.make_shards(specs, 1, 1)
    total = shards[-1].end
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="non_attention_linear", seed=77)
    g = torch.from_numpy(lognormal(total, 9)).to(DEV)
    c1, c2 = tagc.Context(cfg, device=0), tagc.Context(cfg, device=0)
    a1, a2 = torch.zeros(total, device=DEV), torch.zeros(total, device=DEV)
    o1, _ = c1.tagc_reduce_shards(shards, g, a1)
    o2 = c2.overlap_begin(shards, g, a2)
    c2.overlap_ready(0, 300_000)  # no event: the gradient is already there
    c2.overlap_finish()
    c2.sync()
    assert torch.equal(a1.view(torch.int32), a2.view(torch.int32))
    check_close(o2.cpu().numpy(), o1.cpu().numpy())
    with pytest.raises(tagc.TagcInvalidArgument):
        c2.overlap_ready(0, 10)
    with pytest.raises(tagc.TagcInvalidArgument):
        c2.overlap_finish()
    c2.overlap_begin(shards, g, a2)
    with pytest.raises(tagc.TagcInvalidArgument):
        c2.overlap_begin(shards, g, a2)
    c2.overlap_finish()
    c2.sync()


@pytest.mark.parametrize("world", [2, 3])
def test_overlap_peer_matches_oracle(orc, world):
    """W ranks as contexts of this process over the peer-memory exchange,
    one host thread and one producer stream per rank."""
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
    grads = [lognormal(total, 500 + r) for r in range(world)]
    src = [torch.from_numpy(g).to(DEV) for g in grads]
    g_d = [torch.full((total,), float("nan"), device=DEV) for _ in range(world)]
    acc = [torch.zeros(total, device=DEV) for _ in range(world)]
    producers = [torch.cuda.Stream() for _ in range(world)]
    torch.cuda.synchronize()
    outs, errs = [None] * world, [None] * world

    def run(r):
        try:
            outs[r] = ctxs[r].overlap_begin(shards, g_d[r], acc[r])
            produce(src[r], g_d[r], layer_ranges() + [(layer_ranges()[-1][1], total)], producers[r], ctxs[r])
            ctxs[r].overlap_finish()
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
    oacc = [np.zeros(total, np.float32) for _ in range(world)]
    refs = {}
    for sh in shards:
        osh = O.Shard(sh.id, sh.owner, sh.begin, sh.end,
                      [O.Segment(s.kind, s.begin, s.end, s.name) for s in sh.segments])
        a = [oacc[r][sh.begin:sh.end].copy() for r in range(world)]
        ref, _ = orc.tagc_reduce_shard(osh, [grads[r][sh.begin:sh.end] for r in range(world)], a, ocfg)
        for r in range(world):
            oacc[r][sh.begin:sh.end] = a[r]
        refs[sh.id] = ref.copy()
    for r in range(world):
        assert np.array_equal(bits(acc[r].cpu().numpy()), bits(oacc[r])), r
    for o in range(world):
        got = outs[o].cpu().numpy()
        check_close(got, np.concatenate([refs[s.id] for s in owned[o]]))
