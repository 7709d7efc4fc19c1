"""BASELINE configs 3-5 at their world sizes, on one GPU: W rank contexts run
the one-process-per-GPU code path split at its collective
(tagc_reduce_shards_begin / _end) and the test performs the reduce-scatter
the way the reference's World does (ascending-rank fp32 sums of the owner
blocks, wrapping u32 sums of the index blocks; collectives.cpp:127-166).

* C3 (Llama-3-8B, make_shards(specs, 8, 8)): sampled
  segments of every one of the 8 shards - an FFN cut by a shard boundary,
  whole FFNs, out-proj, raw attention_qkv and norm segments - re-based into a
  compact flat buffer (every quantity of the path is per segment and
  segment-relative, hook.cpp:117-166), against the CPU oracle segment by
  segment: every rank's residual bit-exact, peel statistics exact, owners'
  decoded values within 1e-5 (roundtrip.cpp:119-137). The two 525M-element
  segments (embedding, lm_head) are beyond the CPU oracle's memory at W = 8
  and are checked through the size-independent properties below. (Llama's
  8.03B parameters split into 8 equal shards exactly: there is no pad tail
  at W = 8; pad tails are covered at W = 3 in test_gpu_multirank.py.)
* C4 (one 2^28 bucket): W = 2 against the oracle; W = 8 by properties.
* C5 (one 2^30 bucket, 8 shards of 2^27): W = 8 by properties.

Properties (integer-valued gradients, so every sum is exact in fp32):
per rank, with comb = g + acc (one fp32 add) and tau the c-th smallest |comb|
(sparsify.cpp:30-37): an element is dropped iff its residual is comb bit for
bit, kept iff its residual is +0; #dropped >= c > #(|comb| < max dropped) and
every kept magnitude exceeds max dropped (so the split is exactly
|comb| > tau, kernels.cpp:95). Per owner: presence = |union of the kept
supports| (a 4-bit index is exact, index.cpp:80-93), positions outside the
union decode to +0 exactly, and at least `peeled` positions of the union
decode to the exact rank sum (a peeled value is exact on integers,
roundtrip.cpp:109-118); all of them when nothing is left unresolved.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
import paper_2504_05638_b200 as tagc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def bits_np(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def check_close(got, ref, tol=1e-5):
    scale = float(np.abs(ref).max())
    if scale == 0.0:
        assert np.array_equal(bits_np(got), bits_np(ref))
        return
    err = float(np.max(np.abs(got.astype(np.float64) - ref) / np.maximum(np.abs(ref), scale)))
    assert err <= tol, err


def int_grad(n, seed, dev=DEV):
    """Integer-valued gradient with log-normal-like magnitudes and fair signs
    (many ties at every threshold)."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    mag = torch.randn(n, device=dev, generator=g).mul_(1.5).exp_().round_().clamp_(max=4096)
    sign = torch.randint(0, 2, (n,), device=dev, generator=g, dtype=torch.int8)
    # + 0.0: the -0.0 of a zero magnitude becomes +0.0, as g + acc does with
    # a zero accumulator, so g itself is the first step's combined value
    return torch.where(sign.bool(), -mag, mag).add_(0.0)


def lognormal_np(n, seed):
    rng = np.random.default_rng(seed)
    mag = np.exp(rng.standard_normal(n, dtype=np.float32))
    return np.where(rng.integers(0, 2, n, dtype=np.int8) == 1, -mag, mag).astype(np.float32)


def run_split(cfg, shards, world, grads, accs, outs):
    """One exchange of every rank through _begin / _end, the reduce-scatter
    done here in the reference World's fold order. Returns the owners' stats."""
    _, Bf, Bu = tagc.plan_exchange(cfg, shards, world, 0)
    ctxs = [tagc.Context(cfg, world_size=world, rank=r, device=0) for r in range(world)]
    send_f = [torch.empty(world * Bf, device=DEV) for _ in range(world)]
    send_u = [torch.empty(world * Bu, dtype=torch.int32, device=DEV) for _ in range(world)]
    for r in range(world):
        ctxs[r].reduce_shards_begin(shards, grads[r], accs[r], outs[r], send_f[r], send_u[r])
    stats = []
    for o in range(world):
        rf = send_f[0][o * Bf:(o + 1) * Bf].clone()
        ru = send_u[0][o * Bu:(o + 1) * Bu].clone()
        for r in range(1, world):
            rf += send_f[r][o * Bf:(o + 1) * Bf]
            ru += send_u[r][o * Bu:(o + 1) * Bu]  # int32 add wraps like the u32 merge
        stats.append(ctxs[o].reduce_shards_end(rf, ru))
        del rf, ru
    torch.cuda.synchronize()
    for c in ctxs:
        c.close()
    del send_f, send_u
    torch.cuda.empty_cache()
    return stats


def check_rank_split(comb, acc_new, c):
    """sparsify (sparsify.cpp:18-49) from what it left behind, bit for bit."""
    cb, ab = comb.view(torch.int32), acc_new.view(torch.int32)
    dropped = ab == cb
    kept = ~dropped
    assert bool((ab[kept] == 0).all()), "kept residual must be +0"
    a = comb.abs()
    n_drop = int(dropped.sum())
    assert n_drop >= c
    tau = float(a[dropped].max()) if n_drop else 0.0
    assert int((a < tau).sum()) < c
    if int(kept.sum()):
        assert float(a[kept].min()) > tau
    return kept


def check_owner(out_seg, truth, union, st_presence, st_peeled, st_unresolved):
    zero_i = torch.zeros((), dtype=torch.int32, device=DEV)
    assert st_presence == int(union.sum())
    assert bool((out_seg.view(torch.int32)[~union] == zero_i).all()), "positions outside the union decode to +0"
    exact = int((out_seg[union] == truth[union]).sum())
    assert exact >= st_peeled, (exact, st_peeled)
    if st_unresolved == 0:
        assert torch.equal(out_seg, truth)


# --------------------------------------------------------------------- C3
def compact(shards, picks):
    """picks: {shard id: [segment names]} -> the same segments re-based into
    a compact flat layout (ids and owners kept). Returns (shards, sources)
    where sources lists (new begin, size, kind, name)."""
    out, off, src = [], 0, []
    for sh in shards:
        names = picks.get(sh.id, [])
        segs = []
        b0 = off
        for s in sh.segments:
            if s.name in names:
                segs.append(tagc.LayerSegment(s.name, s.kind, off, off + s.size()))
                src.append((off, s.size(), s.kind, s.name))
                off += s.size()
        if segs:
            out.append(tagc.ShardSpec(sh.id, sh.owner, b0, off, segs))
    return out, src


C3_PICKS = {
    0: ["layers.2.mlp.gate_proj", "layers.2.self_attn.o_proj", "layers.0.self_attn.q_proj"],
    1: ["layers.2.mlp.gate_proj"],       # the other piece of the boundary-cut FFN (58.4M)
    2: ["layers.6.input_layernorm", "layers.11.self_attn.o_proj"],
    3: ["layers.16.self_attn.q_proj", "layers.15.input_layernorm"],  # a 2048-element raw cut
    4: ["layers.16.self_attn.k_proj", "layers.20.self_attn.o_proj"],
    5: ["layers.25.mlp.gate_proj"],      # 2.6M cut piece
    6: ["layers.29.mlp.down_proj"],      # 16.5M cut piece
    7: ["norm", "layers.29.post_attention_layernorm", "layers.29.mlp.down_proj"],
}


def test_c3_llama3_8b_sampled_segments_match_oracle(orc):
    world = 8
    full = tagc.make_shards(tagc.llama3_8b_specs(), world, world)
    shards, _ = compact(full, C3_PICKS)
    assert sorted(s.owner for s in shards) == list(range(world))
    total = shards[-1].end
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="non_attention_linear",
                                 include_out_proj=True, seed=77)
    ocfg = O.Config(99.0, 10, 4, "non_attention_linear", True, 77, 3, False, 1024)
    comp = sum(s.size() for sh in shards for s in sh.segments
               if tagc.kind_compressible(s.kind, "non_attention_linear", True))
    assert comp > 100_000_000  # the sample holds >100M compressed parameters per rank
    grads_np = [lognormal_np(total, 31 + r) for r in range(world)]
    grads = [torch.from_numpy(g).to(DEV) for g in grads_np]
    accs = [torch.zeros(total, device=DEV) for _ in range(world)]
    owned = [[s for s in shards if s.owner == r] for r in range(world)]
    outs = [torch.empty(max(1, sum(s.size() for s in owned[r])), device=DEV) for r in range(world)]
    stats = run_split(cfg, shards, world, grads, accs, outs)
    oacc = [np.zeros(total, np.float32) for _ in range(world)]
    for sh in shards:
        osh = O.Shard(sh.id, sh.owner, sh.begin, sh.end,
                      [O.Segment(s.kind, s.begin, s.end, s.name) for s in sh.segments])
        a = [oacc[r][sh.begin:sh.end].copy() for r in range(world)]
        ref, rst = orc.tagc_reduce_shard(osh, [g[sh.begin:sh.end] for g in grads_np], a, ocfg)
        for r in range(world):
            assert np.array_equal(bits_np(accs[r][sh.begin:sh.end].cpu().numpy()), bits_np(a[r])), (sh.id, r)
        o = sh.owner
        off = sum(s.size() for s in owned[o] if s.id < sh.id)
        check_close(outs[o][off:off + sh.size()].cpu().numpy(), ref)
        sh_stats = stats[o]
        # one shard per owner in this sample: the owner's stats are the shard's
        for k in ("presence", "peeled", "unresolved", "index_lost", "index_spurious", "compressed_segments",
                  "baseline_segments"):
            assert getattr(sh_stats, k) == rst[k], (sh.id, k, sh_stats, rst)


@pytest.mark.parametrize("name,shard_id", [("embed_tokens", 0), ("lm_head", 7)])
def test_c3_llama3_8b_525m_segments_properties(name, shard_id):
    """The 525,336,576-element embedding / lm_head segment of its Llama-3-8B
    shard, all 8 ranks, theta 99 (union density 7.7 %, peel load 0.77)."""
    world = 8
    full = tagc.make_shards(tagc.llama3_8b_specs(), world, world)
    shards, src = compact(full, {shard_id: [name]})
    n = shards[0].size()
    assert n == 525_336_576 and shards[0].owner == shard_id
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="non_attention_linear",
                                 include_out_proj=True, seed=77)
    grads = [int_grad(n, 700 + r) for r in range(world)]
    accs = [torch.zeros(n, device=DEV) for _ in range(world)]
    outs = [torch.empty(n if r == shard_id else 1, device=DEV) for r in range(world)]
    stats = run_split(cfg, shards, world, grads, accs, outs)
    c = math.ceil(99.0 * n / 100.0)
    truth = torch.zeros(n, device=DEV)
    union = torch.zeros(n, dtype=torch.bool, device=DEV)
    for r in range(world):
        kept = check_rank_split(grads[r], accs[r], c)
        truth += torch.where(kept, grads[r], torch.zeros((), device=DEV))
        union |= kept
        grads[r] = accs[r] = None
        del kept
    st = stats[shard_id]
    assert st.compressed_segments == 1 and st.index_lost == 0 and st.index_spurious == 0
    assert st.peeled + st.unresolved == st.presence
    check_owner(outs[shard_id], truth, union, st.presence, st.peeled, st.unresolved)


# --------------------------------------------------------------------- C4 / C5
def bucket_shards(n, world):
    return tagc.make_shards([tagc.LayerSpec("bucket", "feed_forward", n)], world, world)


def test_c4_2e28_w2_matches_oracle(orc):
    n, world = 1 << 28, 2
    shards = bucket_shards(n, world)
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="all_layers", seed=77,
                                 min_compress_segment=1)
    ocfg = O.Config(99.0, 10, 4, "all_layers", True, 77, 3, False, 1)
    grads_np = [np.asarray(g) for g in orc.stream(n, 4242, count=world)]
    grads = [torch.from_numpy(g).to(DEV) for g in grads_np]
    accs = [torch.zeros(n, device=DEV) for _ in range(world)]
    outs = [torch.empty(n // world, device=DEV) for _ in range(world)]
    stats = run_split(cfg, shards, world, grads, accs, outs)
    for sh in shards:
        osh = O.Shard(sh.id, sh.owner, sh.begin, sh.end,
                      [O.Segment(s.kind, s.begin, s.end, s.name) for s in sh.segments])
        a = [np.zeros(sh.size(), np.float32) for _ in range(world)]
        ref, rst = orc.tagc_reduce_shard(osh, [g[sh.begin:sh.end] for g in grads_np], a, ocfg)
        for r in range(world):
            assert np.array_equal(bits_np(accs[r][sh.begin:sh.end].cpu().numpy()), bits_np(a[r])), (sh.id, r)
        check_close(outs[sh.owner].cpu().numpy(), ref)
        for k in ("presence", "peeled", "unresolved"):
            assert getattr(stats[sh.owner], k) == rst[k], (k, stats[sh.owner], rst)


@pytest.mark.parametrize("log2n,world,theta", [(28, 8, 99.0), (28, 4, 95.0), (30, 8, 99.9), (30, 8, 99.0)])
def test_c4_c5_multirank_properties(log2n, world, theta):
    """C4 at W = 4 / 8 (theta 95 at W = 4 is past the peel threshold: load
    0.74 at r = 4) and C5 (2^30, 8 shards of 2^27) at W = 8, two
    error-feedback steps for C4."""
    n = 1 << log2n
    ratio = 10 if theta >= 98.75 else 4
    shards = bucket_shards(n, world)
    L = shards[0].size()
    cfg = tagc.CompressionConfig(theta=theta, ratio=ratio, index_width=4, policy="all_layers", seed=77,
                                 min_compress_segment=1)
    accs = [torch.zeros(n, device=DEV) for _ in range(world)]
    steps = 2 if log2n <= 28 else 1
    for step in range(steps):
        grads = [int_grad(n, 100 * step + r) for r in range(world)]
        # comb = g + acc, formed before the call overwrites acc (one fp32 add)
        combs = [g + a for g, a in zip(grads, accs)] if step else grads
        outs = [torch.empty(L, device=DEV) for _ in range(world)]
        stats = run_split(cfg, shards, world, grads, accs, outs)
        c = math.ceil(theta * L / 100.0)
        kept = [[None] * world for _ in range(world)]  # per shard, per rank
        for r in range(world):
            for sh in shards:
                kept[sh.id][r] = check_rank_split(combs[r][sh.begin:sh.end], accs[r][sh.begin:sh.end], c)
        for sh in shards:
            truth = torch.zeros(L, device=DEV)
            union = torch.zeros(L, dtype=torch.bool, device=DEV)
            for r in range(world):
                truth += torch.where(kept[sh.id][r], combs[r][sh.begin:sh.end], torch.zeros((), device=DEV))
                union |= kept[sh.id][r]
            st = stats[sh.owner]
            check_owner(outs[sh.owner], truth, union, st.presence, st.peeled, st.unresolved)
        del grads, combs, outs, kept, truth, union
        torch.cuda.empty_cache()
