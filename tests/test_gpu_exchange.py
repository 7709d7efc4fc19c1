"""GPU parity of the fused exchange (tagc_reduce_shard, simulated W-rank
world on one GPU) against the CPU oracle: sparsification mask (residual
accumulators) bit-exact, recovered/unresolved counts and index diagnostics
exact, decoded values within the reference's 1e-5 tolerance (roundtrip.cpp:
119-137) and bit-exact on integer-valued inputs (roundtrip.cpp:109-118)."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2504_05638_b200 as tagc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32).copy()).to(DEV)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def to_oracle(shard):
    return O.Shard(shard.id, shard.owner, shard.begin, shard.end,
                   [O.Segment(s.kind, s.begin, s.end, s.name) for s in shard.segments])


def ocfg(c):
    return O.Config(c.theta, c.ratio, c.index_width, c.policy, c.include_out_proj, c.seed,
                    c.sketch_rows, c.allow_low_theta, c.min_compress_segment)


def run_both(orc, cfg, shard, grads, accs=None, steps=1):
    """Runs `steps` exchanges on both paths; returns final outputs."""
    world = len(grads)
    n = shard.size()
    accs = accs or [np.zeros(n, np.float32) for _ in range(world)]
    o_acc = [a.copy() for a in accs]
    g_d = [d(g) for g in grads]
    a_d = [d(a) for a in accs]
    ctx = tagc.Context(cfg, device=0)
    for _ in range(steps):
        out, st = ctx.tagc_reduce_shard_sim(shard, g_d, a_d)
        ref, rst = orc.tagc_reduce_shard(to_oracle(shard), grads, o_acc, ocfg(cfg))
    torch.cuda.synchronize()
    return out.cpu().numpy(), st, ref, rst, [a.cpu().numpy() for a in a_d], o_acc, ctx


def check_close(got, ref, tol=1e-5):
    scale = float(np.abs(ref).max()) if ref.size else 0.0
    if scale == 0.0:
        assert np.array_equal(bits(got), bits(ref))
        return 0.0
    err = float(np.max(np.abs(got.astype(np.float64) - ref) / np.maximum(np.abs(ref), scale)))
    assert err <= tol, err
    return err


def single(n, kind="feed_forward"):
    return tagc.ShardSpec(0, 0, 0, n, [tagc.LayerSegment("seg", kind, 0, n)])


@pytest.mark.parametrize("n,world,width,theta,ratio", [
    (1 << 20, 2, 4, 99.0, 10), (1 << 20, 2, 1, 98.75, 10), (1 << 20, 4, 4, 99.5, 10),
    (1 << 20, 8, 4, 99.9, 10), (1_000_003, 2, 4, 90.0, 4), (1 << 20, 2, 4, 80.0, 2),
    (1 << 24, 2, 4, 99.0, 10),  # BASELINE config 1 (C1)
    (1 << 24, 2, 1, 99.0, 10),
])
def test_reduce_shard_lognormal_vs_oracle(orc, n, world, width, theta, ratio):
    cfg = tagc.CompressionConfig(theta=theta, ratio=ratio, index_width=width, policy="all_layers",
                                 seed=77, min_compress_segment=1)
    grads = list(orc.stream(n, 100, count=world))
    out, st, ref, rst, acc, oacc, _ = run_both(orc, cfg, single(n), grads)
    for r in range(world):
        assert np.array_equal(bits(acc[r]), bits(oacc[r])), r  # mask bit-exact
    for k in ("presence", "peeled", "unresolved", "index_lost", "index_spurious",
              "compressed_segments", "baseline_segments"):
        assert getattr(st, k) == rst[k], (k, st, rst)
    check_close(out, ref)


def test_reduce_shard_error_feedback_steps(orc):
    # three steps with the residual carried in the accumulators (train loop shape)
    n = 1 << 19
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="all_layers", seed=5,
                                 min_compress_segment=1)
    grads = list(orc.stream(n, 7, count=2))
    out, st, ref, rst, acc, oacc, _ = run_both(orc, cfg, single(n), grads, steps=3)
    for r in range(2):
        assert np.array_equal(bits(acc[r]), bits(oacc[r]))
    assert st.presence == rst["presence"] and st.unresolved == rst["unresolved"]
    check_close(out, ref)


def roundtrip_grads(n, world, theta, seed, integer):
    """reference roundtrip.cpp:65-87 generator (numpy restatement, same shape)."""
    rng = np.random.default_rng(seed)
    zeros = int(np.ceil(theta * n / 100.0))
    support = np.sort(rng.choice(n, n - min(zeros, n), replace=False))
    grads = [np.zeros(n, np.float32) for _ in range(world)]
    for p in support:
        mask = int(rng.integers(1, 2 ** world))
        for r in range(world):
            if mask >> r & 1:
                if integer:
                    v = float(rng.integers(1, 17)) * (1 if rng.random() < 0.5 else -1)
                else:
                    v = 0.0
                    while v == 0.0:
                        v = float(np.float32(rng.random() * 2 - 1))
                grads[r][p] = v
    return grads


@pytest.mark.parametrize("theta,ratio,world", [(80.0, 2, 2), (90.0, 4, 4), (98.75, 10, 8)])
def test_roundtrip_integer_bit_exact(orc, theta, ratio, world):
    # acceptance criterion 1 operating points: integer trials decode bit-exactly
    n = 10000
    for t in range(6):
        grads = roundtrip_grads(n, world, theta, 1000 * t + world, integer=(t % 2 == 0))
        cfg = tagc.CompressionConfig(theta=theta, ratio=ratio, index_width=4, policy="all_layers",
                                     seed=20250808 + t, min_compress_segment=1)
        out, st, ref, rst, acc, oacc, _ = run_both(orc, cfg, single(n), grads)
        assert st.unresolved == rst["unresolved"] and st.presence == rst["presence"]
        truth = np.sum(np.stack(grads), axis=0, dtype=np.float32)
        if t % 2 == 0 and st.unresolved == 0:
            assert np.array_equal(bits(out), bits(ref))
            assert np.array_equal(bits(out), bits(truth))
        else:
            check_close(out, ref)


def test_gpt2_small_shards_layer_selective(orc):
    # BASELINE config 2: GPT-2 small (tied, 124M), make_shards(specs, 2, 2),
    # non_attention_linear, theta 98.75 / ratio 10 / 1-bit index (paper setting).
    specs = tagc.gpt2_specs()
    shards = tagc.make_shards(specs, 2, 2)
    total = sum(s.size() for s in shards)
    grads = list(orc.stream(total, 2024, count=2))
    cfg = tagc.CompressionConfig(theta=98.75, ratio=10, index_width=1, policy="non_attention_linear",
                                 seed=77)
    ctx = tagc.Context(cfg, device=0)
    for sh in shards:
        g = [x[sh.begin:sh.end] for x in grads]
        g_d = [d(x) for x in g]
        a_d = [torch.zeros(sh.size(), device=DEV) for _ in g]
        out, st = ctx.tagc_reduce_shard_sim(sh, g_d, a_d)
        oacc = [np.zeros(sh.size(), np.float32) for _ in g]
        ref, rst = orc.tagc_reduce_shard(to_oracle(sh), g, oacc, ocfg(cfg))
        for r in range(2):
            assert np.array_equal(bits(a_d[r].cpu().numpy()), bits(oacc[r]))
        for k in rst:
            assert getattr(st, k) == rst[k], (k, st, rst)
        check_close(out.cpu().numpy(), ref)


def test_raw_and_bypass_paths_bit_exact(orc):
    # hook.cpp:125-135 raw segments; test_hook.cpp:203-217 bypass == baseline
    rng = np.random.default_rng(41)
    n, world = 7000, 3
    grads = [(rng.random(n) * 2 - 1).astype(np.float32) for _ in range(world)]
    shard = tagc.ShardSpec(0, 1, 0, n, [tagc.LayerSegment("ln", "norm", 0, 128),
                                        tagc.LayerSegment("ffn", "feed_forward", 128, 5000),
                                        tagc.LayerSegment("small", "feed_forward", 5000, 5500),
                                        tagc.LayerSegment("qkv", "attention_qkv", 5500, n)])
    cfg = tagc.CompressionConfig(theta=80.0, ratio=2, index_width=4, policy="non_attention_linear",
                                 seed=9, min_compress_segment=1024)
    out, st, ref, rst, acc, oacc, ctx = run_both(orc, cfg, shard, grads)
    assert st.compressed_segments == 1 and st.baseline_segments == 3
    raw = np.r_[0:128, 5000:n]
    assert np.array_equal(bits(out[raw]), bits(ref[raw]))
    for r in range(world):
        assert np.array_equal(bits(acc[r]), bits(oacc[r]))
        assert not acc[r][raw].any()  # raw segments leave the accumulator untouched
    check_close(out, ref)
    csv = ctx.ledger_csv()
    assert "reduce_scatter,grad/shard0/ln," in csv and "reduce,sketch/shard0/ffn," in csv
    bypass = tagc.CompressionConfig(theta=0.0, ratio=1, index_width=4, policy="all_layers")
    c2 = tagc.Context(bypass, device=0)
    g_d = [d(g) for g in grads]
    o1, _ = c2.tagc_reduce_shard_sim(shard, g_d, [torch.zeros(n, device=DEV) for _ in g_d])
    o2 = c2.baseline_reduce_shard_sim(shard, g_d)
    assert torch.equal(o1.view(torch.int32), o2.view(torch.int32))
    want = orc.baseline_reduce_shard(to_oracle(shard), grads)
    assert np.array_equal(bits(o2.cpu().numpy()), bits(want))


def test_one_bit_carry_loses_and_fabricates(orc):
    # test_hook.cpp:152-169 / acceptance criterion 7
    n = 2048
    grads = [np.zeros(n, np.float32), np.zeros(n, np.float32)]
    grads[0][0], grads[1][0] = 5.0, 3.0
    cfg = tagc.CompressionConfig(theta=80.0, ratio=2, index_width=1, policy="all_layers",
                                 min_compress_segment=1)
    out, st, ref, rst, acc, oacc, _ = run_both(orc, cfg, single(n), grads)
    assert st.index_lost == 1 and st.index_spurious == 1
    assert out[0] == 0.0 and not acc[0].any() and not acc[1].any()


def test_theta_100_moves_everything_to_accumulators(orc):
    n = 1500
    rng = np.random.default_rng(51)
    grads = [(rng.random(n) * 2 - 1).astype(np.float32) for _ in range(2)]
    cfg = tagc.CompressionConfig(theta=100.0, ratio=2, index_width=4, policy="all_layers",
                                 min_compress_segment=1)
    out, st, ref, rst, acc, oacc, _ = run_both(orc, cfg, single(n), grads)
    assert not out.any() and st.presence == 0
    for r in range(2):
        assert np.array_equal(bits(acc[r]), bits(grads[r]))


def test_nan_is_rejected(orc):
    # sparsify.cpp:26 throws std::invalid_argument; as in the reference (which
    # has already updated the accumulators of segments/ranks processed before
    # the throw), accumulator contents after the error are unspecified.
    n = 1 << 18
    g = np.ones(n, np.float32)
    g[100] = np.nan
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="all_layers",
                                 min_compress_segment=1)
    ctx = tagc.Context(cfg, device=0)
    acc = [torch.full((n,), 0.25, device=DEV) for _ in range(2)]
    with pytest.raises(tagc.TagcInvalidArgument):
        ctx.tagc_reduce_shard_sim(single(n), [d(g), d(np.ones(n))], acc)
    # the context stays usable after the error
    out, st = ctx.tagc_reduce_shard_sim(single(n), [d(np.ones(n)), d(np.ones(n))],
                                        [torch.zeros(n, device=DEV) for _ in range(2)])
    assert st.compressed_segments == 1


def test_validation_errors():
    n = 64
    ctx = tagc.Context(tagc.CompressionConfig(), device=0)
    with pytest.raises(tagc.TagcInvalidArgument):  # low theta for ratio 10 (test_hook.cpp:340-351)
        ctx.set_config(tagc.CompressionConfig(theta=50.0, ratio=10))
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, policy="all_layers", min_compress_segment=1)
    ctx.set_config(cfg)
    g = [torch.ones(20, device=DEV)] * 2
    a = [torch.zeros(20, device=DEV) for _ in range(2)]
    with pytest.raises(tagc.TagcInvalidArgument):  # m == 0 (sketch.cpp:16-20)
        ctx.tagc_reduce_shard_sim(single(20), g, a)
    with pytest.raises(tagc.TagcInvalidArgument):  # 4-bit index beyond 15 ranks
        ctx.tagc_reduce_shard_sim(single(n), [torch.ones(n, device=DEV)] * 16,
                                  [torch.zeros(n, device=DEV) for _ in range(16)])


@pytest.mark.parametrize("world,theta,ratio,width", [(2, 80.0, 2, 4), (4, 99.0, 10, 4), (3, 98.75, 10, 1)])
def test_ledger_matches_volume_model(orc, world, theta, ratio, width):
    """test_hook.cpp:262-278: after an exchange the context's ledger charges
    exactly comm_volume_model's index / sketch bits per parameter, and the
    JSON dump agrees with the CSV rows."""
    import json
    n = 10_000
    rng = np.random.default_rng(world)
    grads = [(rng.random(n) * 2 - 1).astype(np.float32) for _ in range(world)]
    cfg = tagc.CompressionConfig(theta=theta, ratio=ratio, index_width=width, policy="all_layers",
                                 min_compress_segment=1)
    _, _, _, _, _, _, ctx = run_both(orc, cfg, single(n), grads)
    model = tagc.comm_volume_model(cfg, world, n)
    led = ctx.ledger()
    assert led.bits_per_param_per_rank("index/") == model["index_bits"]
    assert led.bits_per_param_per_rank("sketch/") == model["sketch_bits"]
    rows = json.loads(led.to_json())
    csv_rows = ctx.ledger_csv().strip().split("\n")[1:]
    assert [f"{r['op']},{r['tag']},{r['calls']},{r['payload_bits']},{r['charged_bits']}" for r in rows] == \
        [",".join(c.split(",")[:5]) for c in csv_rows]
