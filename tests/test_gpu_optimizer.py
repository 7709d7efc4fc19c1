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
