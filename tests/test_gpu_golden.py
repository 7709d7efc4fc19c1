"""GPU: the CUDA path against fixtures produced by the compiled reference
(tests/golden/make_golden.py) — no oracle in the loop."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2504_05638_b200 as tagc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))
with open(os.path.join(HERE, "golden", "golden.json")) as f:
    M = json.load(f)


def d(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    elif a.dtype.kind == "f":
        a = a.astype(np.float32)
    return torch.from_numpy(a.copy()).to(DEV)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_sparsify_fixtures_bit_exact(ctx):
    for c in M["sparsify"]:
        i = c["i"]
        sp, res, tau, zc = ctx.sparsify(d(G[f"sp{i}_g"]), c["theta"])
        assert tau == c["tau"] and zc == c["zero_count"], c
        assert np.array_equal(bits(sp.cpu().numpy()), bits(G[f"sp{i}_sparse"]))
        assert np.array_equal(bits(res.cpu().numpy()), bits(G[f"sp{i}_residual"]))
    sp, _, tau, zc = ctx.sparsify(d(G["sp_lognormal_g"]), 98.75)
    assert tau == M["sp_lognormal"]["tau"] and zc == M["sp_lognormal"]["zero_count"]
    assert np.array_equal(bits(sp.cpu().numpy()), bits(G["sp_lognormal_sparse"]))


def test_index_fixtures_bit_exact(ctx):
    for c in M["index"]:
        w = ctx.index_create(d(G[f"ix{c['i']}_v"]), c["width"]).cpu().numpy().view(np.uint32)
        want = G[f"ix{c['i']}_words"]
        assert np.array_equal(w[: want.size], want)


def test_sketch_fixtures(ctx):
    for c in M["sketch"]:
        got = ctx.sketch_compress(d(G[f"sk{c['i']}_v"]), c["ratio"], c["seed"], c["rows"]).cpu().numpy()
        want = G[f"sk{c['i']}_sketch"]
        scale = max(float(np.abs(want).max()), 1e-30)
        assert np.max(np.abs(got - want)) <= 1e-6 * scale  # test_sketch.cpp:92-117


def test_peel_fixtures(ctx):
    for c in M["peel"]:
        i = c["i"]
        vals, unres, pf = ctx.peeling_decompress(d(G[f"pe{i}_presence"]), d(G[f"pe{i}_sketch"]), c["n"],
                                                 c["ratio"], c["seed"])
        assert pf == c["pf"]
        assert np.array_equal(unres.cpu().numpy().view(np.uint32), G[f"pe{i}_unresolved"])
        want = G[f"pe{i}_values"]
        scale = max(float(np.abs(want).max()), 1e-30)
        assert np.max(np.abs(vals.cpu().numpy() - want)) <= 1e-5 * scale


@pytest.mark.parametrize("case", [c["name"] for c in M["hook"]])
def test_reduce_shard_fixtures(case):
    c = next(x for x in M["hook"] if x["name"] == case)
    n = c["segments"][-1][2]
    shard = tagc.ShardSpec(0, c["owner"], 0, n, [tagc.LayerSegment(f"seg{j}", k, b, e)
                                                   for j, (k, b, e) in enumerate(c["segments"])])
    grads = O.Oracle().stream(n, 31 + c["world"], count=c["world"])  # pinned to the reference stream
    cfg = tagc.CompressionConfig(theta=c["theta"], ratio=c["ratio"], index_width=c["width"],
                                 policy=c["policy"], seed=77, min_compress_segment=c["min_compress_segment"])
    ctx = tagc.Context(cfg, device=0)
    accs = [torch.zeros(n, device=DEV) for _ in range(c["world"])]
    out, st = ctx.tagc_reduce_shard_sim(shard, [d(g) for g in grads], accs)
    assert {k: getattr(st, k) for k in c["stats"]} == c["stats"]
    assert np.array_equal(bits(torch.stack(accs).cpu().numpy()), bits(G[f"hk_{case}_accs"]))
    want = G[f"hk_{case}_decoded"]
    scale = float(np.abs(want).max())
    err = np.abs(out.cpu().numpy().astype(np.float64) - want) / np.maximum(np.abs(want), scale)
    assert err.max() <= 1e-5, err.max()
    assert ctx.ledger_csv() == c["ledger_csv"]
