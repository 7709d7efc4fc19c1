"""Full-size GPU cases of BASELINE configs 4 and 5, checked
through size-independent properties instead of the CPU oracle (which cannot
hold them): one rank (W = 1), so the exchange must return exactly the
sparsified gradient.

* tau is the c-th smallest |g| (sparsify.cpp:30-37): #(|g| < tau) < c <= #(|g| <= tau),
  with tau recovered as the largest residual magnitude;
* mask: an element is kept iff |g| > tau (kernels.cpp:95), the residual of a
  kept element is +0 and of a dropped one the element itself, bit for bit;
* decode: every position of a compressed segment decodes to the kept value
  (within the reference's 1e-5 relative tolerance, roundtrip.cpp:119-137) or
  to exactly +0, and the peel resolves every present position at these loads.
"""
import math

import pytest
import torch

import paper_2504_05638_b200 as tagc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def lognormal(n, seed):
    g = torch.Generator(device=DEV)
    g.manual_seed(seed)
    mag = torch.randn(n, device=DEV, generator=g).exp_()
    sign = torch.randint(0, 2, (n,), device=DEV, generator=g, dtype=torch.int8)
    return torch.where(sign.bool(), -mag, mag)


def check_exchange(n, theta, ratio, seed=5):
    cfg = tagc.CompressionConfig(theta=theta, ratio=ratio, index_width=4, policy="all_layers", seed=77,
                                 min_compress_segment=1)
    shards = [tagc.ShardSpec(0, 0, 0, n, [tagc.LayerSegment("bucket", "feed_forward", 0, n)])]
    ctx = tagc.Context(cfg, device=0)
    grad = lognormal(n, seed)
    acc = torch.zeros(n, device=DEV)
    out = torch.empty(n, device=DEV)
    _, st = ctx.tagc_reduce_shards(shards, grad, acc, out, stats=True)
    c = min(n, math.ceil(theta * float(n) / 100.0))  # sparsify.cpp:30
    a = grad.abs()
    tau = float(acc.abs().max())
    assert int((a < tau).sum()) < c <= int((a <= tau).sum())
    kept = a > tau
    n_kept = int(kept.sum())
    assert st.presence == n_kept and st.unresolved == 0 and st.peeled == n_kept, st
    # residual: bit-exact split
    zero = torch.zeros((), device=DEV)
    assert torch.equal(acc.view(torch.int32), torch.where(kept, zero, grad).view(torch.int32))
    # decode: the kept values, zeros elsewhere
    ref = torch.where(kept, grad, zero)
    assert torch.equal(out[~kept].view(torch.int32), torch.zeros_like(out[~kept]).view(torch.int32))
    scale = float(ref.abs().max())
    err = float(((out - ref).abs() / torch.clamp(ref.abs(), min=scale)).max())
    assert err <= 1e-5, err
    del grad, acc, out, a, kept, ref
    torch.cuda.empty_cache()


@pytest.mark.parametrize("theta,ratio", [(99.9, 10), (99.5, 10), (99.0, 10), (98.0, 4), (95.0, 4)])
def test_density_sweep_256m(theta, ratio):
    # BASELINE config 4: 256M-element bucket, density 0.1 % - 5 % (W = 1)
    check_exchange(1 << 28, theta, ratio)


def test_one_billion_single_bucket():
    # BASELINE config 5: 2^30-element single bucket, theta 99.9, ratio 10
    check_exchange(1 << 30, 99.9, 10)


def test_grouped_decode_many_segments():
    """Bucket states beyond 128 MB in total (here 3 x 80M-element segments,
    192 MB of state) are decoded in groups (Engine::run_decode_grouped); the
    result must be the same property-exact exchange, per segment."""
    seg = 80 << 20
    n = 3 * seg
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4, policy="all_layers", seed=77,
                                 min_compress_segment=1)
    shards = [tagc.ShardSpec(0, 0, 0, n, [tagc.LayerSegment(f"s{i}", "feed_forward", i * seg, (i + 1) * seg)
                                         for i in range(3)])]
    ctx = tagc.Context(cfg, device=0)
    grad = lognormal(n, 17)
    acc = torch.zeros(n, device=DEV)
    out = torch.empty(n, device=DEV)
    _, st = ctx.tagc_reduce_shards(shards, grad, acc, out, stats=True)
    zero = torch.zeros((), device=DEV)
    n_kept = 0
    for i in range(3):
        g, a, o = grad[i * seg:(i + 1) * seg], acc[i * seg:(i + 1) * seg], out[i * seg:(i + 1) * seg]
        c = math.ceil(99.0 * seg / 100.0)  # sparsify.cpp:30
        tau = float(a.abs().max())
        assert int((g.abs() < tau).sum()) < c <= int((g.abs() <= tau).sum())
        kept = g.abs() > tau
        assert torch.equal(a.view(torch.int32), torch.where(kept, zero, g).view(torch.int32))
        ref = torch.where(kept, g, zero)
        assert torch.equal(o[~kept].view(torch.int32), torch.zeros_like(o[~kept]).view(torch.int32))
        scale = float(ref.abs().max())
        assert float(((o - ref).abs() / torch.clamp(ref.abs(), min=scale)).max()) <= 1e-5
        n_kept += int(kept.sum())
    assert st.presence == n_kept and st.peeled == n_kept and st.unresolved == 0, st
    assert st.compressed_segments == 3
    del grad, acc, out
    torch.cuda.empty_cache()
