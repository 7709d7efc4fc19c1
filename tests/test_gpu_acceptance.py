"""Acceptance criterion 1 (reference tests/acceptance.cpp:68-97) through the
CUDA path at the reference's own parameters: n = 10000, 500 trials, the three
Table-1 operating points (80 %/2x, 90 %/4x, 98.75 %/10x), W in {2, 4, 8},
4-bit index, seed 20250808 + W + ratio. Every trial's inputs come from the
reference's own roundtrip_experiment generator (oracle/_ref
ref_roundtrip_trial, pinned in tests/test_oracle.py) and run through
tagc_reduce_shard_sim on the GPU; the report is compared with the
reference's roundtrip_experiment report for the same point: identical peel
statistics (presence, unresolved, fully peeled trials, lost/spurious),
integer trials bit-exact when resolved, float trials within 1e-5
(roundtrip.cpp:109-142), and the criterion's own pass rule."""
import numpy as np
import pytest
import torch

import paper_2504_05638_b200 as tagc
from roundtrip_util import ACCEPTANCE_POINTS, ACCEPTANCE_WORLDS, acceptance_seed, roundtrip_report

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
N, TRIALS = 10000, 500


@pytest.mark.parametrize("theta,ratio", ACCEPTANCE_POINTS)
@pytest.mark.parametrize("world", ACCEPTANCE_WORLDS)
def test_acceptance_criterion_1(ref, theta, ratio, world):
    seed = acceptance_seed(world, ratio)
    shard = tagc.ShardSpec(0, 0, 0, N, [tagc.LayerSegment("block", "feed_forward", 0, N)])
    base = dict(theta=theta, ratio=ratio, index_width=4, policy="all_layers", min_compress_segment=1)
    ctx = tagc.Context(tagc.CompressionConfig(seed=0, **base), device=0)
    g_d = [torch.empty(N, device=DEV) for _ in range(world)]
    a_d = [torch.empty(N, device=DEV) for _ in range(world)]
    out = torch.empty(N, device=DEV)

    def run(t, grads, tseed):
        ctx.set_config(tagc.CompressionConfig(seed=tseed, **base))  # trial_config.seed (roundtrip.cpp:95)
        for r in range(world):
            g_d[r].copy_(torch.from_numpy(grads[r]))
            a_d[r].zero_()
        _, st = ctx.tagc_reduce_shard_sim(shard, g_d, a_d, out)
        return out.cpu().numpy(), st.__dict__

    got = roundtrip_report(ref, N, TRIALS, theta, world, seed, run)
    live = ref.roundtrip(N, TRIALS, theta, ratio, 4, world, seed=seed)
    for k in ("trials_fully_peeled", "presence_total", "unresolved_total", "index_lost", "index_spurious",
              "integer_exact_when_resolved"):
        assert got[k] == live[k], (k, got[k], live[k])
    assert got["mean_peeled_fraction"] == pytest.approx(live["mean_peeled_fraction"], abs=1e-12)
    assert got["min_peeled_fraction"] == pytest.approx(live["min_peeled_fraction"], abs=1e-12)
    assert got["max_rel_error_resolved"] <= 1e-5
    # acceptance.cpp:88-90
    assert got["pass"] == 1 and got["index_lost"] == 0 and got["index_spurious"] == 0
