"""GPU parity of the per-layer codec entry points (C-ABI) against the CPU
oracle. Integer/index work is bit-exact; fp32 sums use the reference's own
tolerances (test_sketch.cpp:92-117: 1e-6 of the sketch scale;
roundtrip.cpp:119-137: 1e-5 of the vector scale)."""
import numpy as np
import pytest
import torch

import paper_2504_05638_b200 as tagc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def d(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    elif a.dtype.kind == "f":
        a = a.astype(np.float32)
    return torch.from_numpy(a.copy()).to(DEV)


def h(t, u32=False):
    a = t.detach().cpu().numpy()
    return a.view(np.uint32) if u32 else a


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ------------------------------------------------------------------ hash
def test_bucket_and_sign_bit_exact_dense_integers(ctx, orc):
    # Every position nonzero with a small integer value: the fp32 sums are
    # exact in any order, so equality proves bucket(p) and sign(p) for all p.
    rng = np.random.default_rng(1)
    for n, ratio, rows, seed in [(60000, 2, 3, 0x1234), (100003, 4, 3, 77), (30000, 10, 2, 2**64 - 5),
                                 (4096, 2, 5, 9)]:
        v = rng.integers(1, 8, n).astype(np.float32) * rng.choice([-1, 1], n)
        got = h(ctx.sketch_compress(d(v), ratio, seed, rows))
        want = orc.sketch_compress(v, ratio, seed, rows)
        assert np.array_equal(bits(got), bits(want)), (n, ratio, rows)


def test_sketch_golden_dump(ctx):
    # test_sketch.cpp:144-154: n=12, ratio 2, rows 2, seed 1, v[3]=2
    v = np.zeros(12, np.float32)
    v[3] = 2.0
    got = h(ctx.sketch_compress(d(v), 2, 1, 2)).reshape(2, 3)
    assert got.tolist() == [[-2.0, 0.0, 0.0], [0.0, 0.0, 2.0]]
    words = h(ctx.index_create(d(v), 4), True)
    assert words.tolist() == [4096, 0]


def test_sketch_float_within_tolerance(ctx, orc):
    rng = np.random.default_rng(2)
    n = 1 << 20
    v = np.where(rng.random(n) < 0.05, rng.standard_normal(n), 0).astype(np.float32)
    got = h(ctx.sketch_compress(d(v), 10, 5))
    want = orc.sketch_compress(v, 10, 5)
    scale = np.abs(want).max()
    assert np.max(np.abs(got - want)) <= 1e-6 * scale


# ------------------------------------------------------------------ sparsify
def test_sparsify_hand_example(ctx):
    # test_sparsify.cpp:40-47
    sp, res, tau, zc = ctx.sparsify(d(np.array([4.0, -1.0, 0.0, 3.0], np.float32)), 50.0)
    assert tau == 1.0 and zc == 2
    assert h(sp).tolist() == [4.0, 0.0, 0.0, 3.0]
    assert h(res).tolist() == [0.0, -1.0, 0.0, 0.0]


def test_sparsify_threshold_equals_oracle_randomized(ctx, orc):
    # test_sparsify.cpp:63-81 / acceptance criterion 3: ties, zeros, +-1.
    rng = np.random.default_rng(11)
    for trial in range(120):
        n = int(rng.integers(1, 258)) if trial % 10 else int(rng.integers(60000, 300000))
        theta = float(rng.integers(0, 10001)) / 100.0
        g = (rng.random(n) * 20 - 10).astype(np.float32)
        g[rng.random(n) < 0.25] = 0.0
        g[rng.random(n) < 1 / 16] = 1.0
        g[rng.random(n) < 1 / 32] = -0.0
        sp, res, tau, zc = ctx.sparsify(d(g), theta)
        osp, ores, otau, ozc = orc.sparsify(g, theta)
        assert np.float32(tau).view(np.uint32) == np.float32(otau).view(np.uint32), (trial, n, theta)
        assert zc == ozc
        assert np.array_equal(bits(h(sp)), bits(osp))
        assert np.array_equal(bits(h(res)), bits(ores))


@pytest.mark.parametrize("n,theta", [(10000, 98.75), (1 << 20, 99.0), (1 << 24, 99.0), (3_000_001, 90.0),
                                     (1 << 22, 100.0), (1 << 21, 0.0)])
def test_sparsify_lognormal_matches_oracle(ctx, orc, n, theta):
    g = orc.stream(n, 404)[0]
    sp, res, tau, zc = ctx.sparsify(d(g), theta)
    osp, ores, otau, ozc = orc.sparsify(g, theta)
    assert np.float32(tau) == otau and zc == ozc
    assert np.array_equal(bits(h(sp)), bits(osp))
    assert np.array_equal(bits(h(res)), bits(ores))


def test_sparsify_massive_ties_fallback(ctx, orc):
    # 95% zeros plus a block of identical values: exercises tau = 0 and the
    # full radix fallback when the sample bracket overflows.
    n = 1 << 21
    rng = np.random.default_rng(3)
    g = np.zeros(n, np.float32)
    idx = rng.random(n) < 0.05
    g[idx] = rng.standard_normal(idx.sum()).astype(np.float32)
    g[: n // 4] = 0.5
    for theta in (50.0, 80.0, 96.0, 99.9):
        _, _, tau, zc = ctx.sparsify(d(g), theta)
        _, _, otau, ozc = orc.sparsify(g, theta)
        assert tau == otau and zc == ozc, theta


def test_sparsify_rejects_nan_and_bad_theta(ctx):
    with pytest.raises(tagc.TagcInvalidArgument):
        ctx.sparsify(d(np.array([1.0, np.nan], np.float32)), 50.0)
    with pytest.raises(tagc.TagcInvalidArgument):
        ctx.sparsify(d(np.array([1.0], np.float32)), 100.5)


# ------------------------------------------------------------------ index
@pytest.mark.parametrize("width", [1, 4])
def test_index_create_and_presence_bit_exact(ctx, orc, width):
    rng = np.random.default_rng(4)
    for n in (1, 31, 32, 33, 100, 4099, 1 << 20):
        v = np.where(rng.random(n) < 0.3, rng.standard_normal(n), 0).astype(np.float32)
        v[rng.random(n) < 0.1] = -0.0
        w = h(ctx.index_create(d(v), width), True)
        ow = orc.index_create(v, width)
        assert np.array_equal(w[: ow.size], ow), n
        pres = h(ctx.index_presence(d(ow), n, width), True)
        assert np.array_equal(pres, orc.presence(ow, n, width))


def test_index_nibble_layout_and_one_bit_carry(ctx, orc):
    # test_index.cpp:11-22 and :69-80
    w = h(ctx.index_create(d(np.array([0.0, 1.5, 0.0, -2.0], np.float32)), 4), True)
    assert w[0] == 0x1010
    a = np.zeros(8, np.float32)
    a[0] = 1.0
    b = a.copy()
    b[0] = 2.0
    m = h(ctx.merge_indices([ctx.index_create(d(a), 1), ctx.index_create(d(b), 1)]), True)
    assert m[0] == 2
    assert h(ctx.index_presence(d(m), 8, 1), True).tolist() == [1]


def test_merge_sixteen_ranks_overflows_nibble(ctx):
    # test_index.cpp:94-108
    v = np.zeros(8, np.float32)
    v[2] = 1.0
    words = [ctx.index_create(d(v), 4) for _ in range(16)]
    m15 = h(ctx.merge_indices(words[:15]), True)
    assert (m15[0] >> 8) & 0xF == 15
    m16 = h(ctx.merge_indices(words), True)
    assert (m16[0] >> 8) & 0xF == 0 and (m16[0] >> 12) & 0xF == 1


# ------------------------------------------------------------------ decode
def test_peel_empty_presence(ctx):
    vals, unres, pf = ctx.peeling_decompress(torch.zeros(0, dtype=torch.int32, device=DEV),
                                             torch.zeros(30, device=DEV), 60, 2, 1)
    assert pf == 1.0 and unres.numel() == 0 and float(h(vals).max()) == 0.0


def test_peel_disjoint_integer_exact(ctx, orc):
    # test_decode.cpp:40-60
    n = 40
    a = np.zeros(n, np.float32)
    b = np.zeros(n, np.float32)
    a[1], a[20], b[5], b[33] = 3.0, -7.0, 11.0, 2.0
    sk = h(ctx.sketch_add(ctx.sketch_compress(d(a), 2, 5), ctx.sketch_compress(d(b), 2, 5)))
    pres = np.array([1, 5, 20, 33], np.uint32)
    vals, unres, pf = ctx.peeling_decompress(d(pres), d(sk), n, 2, 5)
    assert pf == 1.0 and unres.numel() == 0
    assert np.array_equal(bits(h(vals)), bits(a + b))


@pytest.mark.parametrize("n,density,ratio,seed", [
    (1 << 16, 0.02, 10, 1), (1 << 20, 0.025, 10, 2), (1 << 20, 0.075, 10, 3),  # near threshold
    (1 << 20, 0.30, 2, 4), (300000, 0.12, 4, 5), (1 << 20, 0.5, 2, 6),         # estimation-heavy
])
def test_peel_sets_match_oracle(ctx, orc, n, density, ratio, seed):
    rng = np.random.default_rng(seed)
    pres = np.sort(rng.choice(n, int(n * density), replace=False)).astype(np.uint32)
    v = np.zeros(n, np.float32)
    v[pres] = rng.integers(-50, 51, pres.size).astype(np.float32)
    v[pres[v[pres] == 0]] = 1.0
    sk = orc.sketch_compress(v, ratio, seed * 7919)
    ovals, ounres, opf = orc.peeling_decompress(pres, sk, n, ratio, seed * 7919)
    vals, unres, pf = ctx.peeling_decompress(d(pres), d(sk), n, ratio, seed * 7919)
    assert np.array_equal(h(unres, True), ounres)  # recovered/unresolved sets bit-exact
    assert pf == opf
    got = h(vals)
    peeled = np.setdiff1d(pres, ounres)
    # integer values: peeled positions are exact regardless of order
    assert np.array_equal(bits(got[peeled]), bits(ovals[peeled]))
    assert np.array_equal(bits(np.delete(got, pres)), bits(np.delete(ovals, pres)))
    if ounres.size:
        scale = max(1.0, float(np.abs(ovals).max()))
        assert np.max(np.abs(got[ounres] - ovals[ounres])) <= 1e-5 * scale


def test_peel_rejects_oob_and_duplicates(ctx):
    sk = torch.zeros(30, device=DEV)
    with pytest.raises(tagc.TagcInvalidArgument):
        ctx.peeling_decompress(d(np.array([60], np.uint32)), sk, 60, 2, 1)
    with pytest.raises(tagc.TagcInvalidArgument):
        ctx.peeling_decompress(d(np.array([1, 1], np.uint32)), sk, 60, 2, 1)


def test_estimation_matches_oracle(ctx, orc):
    rng = np.random.default_rng(8)
    n = 300
    v = (rng.random(n) + 0.5).astype(np.float32)
    allp = np.arange(n, dtype=np.uint32)
    sk = orc.sketch_compress(v, 2, 17)
    got = h(ctx.estimation_decompress(d(allp), d(sk), d(allp), n, 2, 17))
    want = orc.estimation_decompress(allp, sk, allp, n, 2, 17)
    assert np.array_equal(bits(got), bits(want))
    with pytest.raises(tagc.TagcInvalidArgument):
        ctx.estimation_decompress(d(allp[:2]), d(sk), d(np.array([3], np.uint32)), n, 2, 17)


@pytest.mark.parametrize("width", [1, 4])
def test_wire_bytes_match_reference(ctx, ref, width):
    """Index::to_bytes / CountSketch::to_bytes (index.cpp:59-69,
    sketch.cpp:77-89): the device buffers' little-endian word layout is the
    reference's wire format byte for byte. Integer-valued sparse values keep
    the sketch sums exact, so its bytes are order-independent."""
    rng = np.random.default_rng(21 + width)
    n = 300_007
    v = np.zeros(n, np.float32)
    idx = rng.choice(n, 3000, replace=False)
    v[idx] = rng.integers(-50, 51, idx.size).astype(np.float32)
    vd = torch.from_numpy(v).to(DEV)
    words = ctx.index_create(vd, width)
    assert ctx.to_bytes(words) == ref.index_to_bytes(v, width)
    sk = ctx.sketch_compress(vd, 10, 77)
    assert ctx.to_bytes(sk) == ref.sketch_to_bytes(v, 10, 77)


_EPOCH_WRAP_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2504_05638_b200 as tagc
from oracle import Oracle
orc = Oracle()
ctx = tagc.Context(tagc.CompressionConfig(theta=99.0, ratio=10, index_width=1, seed=5), device=0)
for call in range(4):
    rng = np.random.default_rng(100 + call)
    n, ratio, seed = 1 << 18, 4, 4242 + call
    pres = np.sort(rng.choice(n, int(n * 0.2), replace=False)).astype(np.uint32)
    v = np.zeros(n, np.float32)
    v[pres] = rng.integers(-50, 51, pres.size).astype(np.float32)
    v[pres[v[pres] == 0]] = 1.0
    sk = orc.sketch_compress(v, ratio, seed)
    ovals, ounres, opf = orc.peeling_decompress(pres, sk, n, ratio, seed)
    vals, unres, pf = ctx.peeling_decompress(torch.from_numpy(pres.view(np.int32).copy()).cuda(),
                                             torch.from_numpy(sk.copy()).cuda(), n, ratio, seed)
    got = vals.cpu().numpy()
    assert np.array_equal(unres.cpu().numpy().view(np.uint32), ounres), call
    peeled = np.setdiff1d(pres, ounres)
    assert np.array_equal(got[peeled].view(np.uint32), ovals[peeled].view(np.uint32)), call
print("epoch wrap ok", ctx.last_peel_rounds())
"""


def test_ordered_peel_across_epoch_wrap():
    """The ordered peel's epoch tags (slot keys, claims) restart from zero once
    the persistent device epoch passes 0xF0000000: start it one below the wrap
    point (TAGC_ORD_EPOCH_START; every call advances it at least once, so the
    second call restarts the tags) and check four FIFO-exact decodes against
    the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TAGC_ORD_EPOCH_START=str(0xF0000000 - 1))
    r = subprocess.run([sys.executable, "-c", _EPOCH_WRAP_SCRIPT, root], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "epoch wrap ok" in r.stdout
