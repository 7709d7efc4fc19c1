"""CPU: the C-ABI library loads, exports every symbol include/tagc_b200.h
declares, and its host-only entry points (config validation, layer policy,
sketch geometry, volume model, make_shards, exchange planning) agree with the
reference. Compute entry points need a GPU and must fail loudly without one."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

import paper_2504_05638_b200 as tagc
from paper_2504_05638_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
    M = json.load(f)


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tagc_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tagc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 40
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)
    assert _lib.lib.tagc_abi_version() == 1


def test_no_cpu_fallback_without_gpu():
    if tagc.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(tagc.TagcError) as ei:
        tagc.Context(tagc.CompressionConfig(), stream=0)
    assert ei.value.status == 1 and "no CUDA device" in str(ei.value)


def test_config_validation_mirrors_reference():
    # config.cpp:27-59
    assert [tagc.theta_floor(r) for r in (1, 2, 4, 10)] == [0.0, 80.0, 90.0, 98.75]
    with pytest.raises(tagc.TagcInvalidArgument):
        tagc.theta_floor(3)
    tagc.CompressionConfig(theta=98.75, ratio=10).validate()
    for bad in (dict(theta=50.0, ratio=10), dict(theta=101.0), dict(index_width=2),
                dict(sketch_rows=0), dict(ratio=3, theta=99.0)):
        with pytest.raises(tagc.TagcInvalidArgument):
            tagc.CompressionConfig(**bad).validate()
    tagc.CompressionConfig(theta=50.0, ratio=10, allow_low_theta=True).validate()
    tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4).validate_for_world(15)
    with pytest.raises(tagc.TagcInvalidArgument):
        tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4).validate_for_world(16)
    tagc.CompressionConfig(theta=99.0, ratio=10, index_width=1).validate_for_world(64)


def test_layer_policy_mirrors_reference():
    # layers.cpp:42-65 and test_hook.cpp:203-214
    nal = "non_attention_linear"
    for k in ("embedding", "positional_embedding", "feed_forward", "lm_head"):
        assert tagc.kind_compressible(k, nal)
    assert tagc.kind_compressible("attention_out_proj", nal, True)
    assert not tagc.kind_compressible("attention_out_proj", nal, False)
    for k in ("attention_qkv", "norm", "bias", "other"):
        assert not tagc.kind_compressible(k, nal)
    assert all(tagc.kind_compressible(k, "all_layers") for k in tagc.api.KIND)
    assert not any(tagc.kind_compressible(k, "none") for k in tagc.api.KIND)


def test_sketch_geometry_and_words():
    assert tagc.sketch_geometry(3000, 10)["buckets_per_row"] == 100
    assert tagc.sketch_geometry(3000, 2)["buckets_per_row"] == 500
    for bad in ((20, 10), (100, 3)):
        with pytest.raises(tagc.TagcInvalidArgument):
            tagc.sketch_geometry(*bad)
    for n in (1, 31, 32, 33, 100):
        for w in (1, 4):
            assert tagc.words_needed(n, w) == (n * w + 31) // 32


def test_volume_model_matches_reference():
    # hook.cpp:202-236, test_hook.cpp:94-124, test_collectives.cpp:171-203
    for c in M["volume"]:
        cfg = tagc.CompressionConfig(theta=c["theta"], ratio=c["ratio"], index_width=c["width"],
                                     policy="all_layers")
        fn = tagc.lhc_comm_volume_model if c["lhc"] else tagc.comm_volume_model
        v = fn(cfg, c["world"], c["n"] or None)
        assert [v["index_bits"], v["sketch_bits"], v["total_bits"], v["factor"]] == c["out"]
    v = tagc.comm_volume_model(tagc.CompressionConfig(theta=98.75, ratio=10, index_width=1), 2)
    assert v["total_bits"] == 5.2 and abs(v["factor"] - 6.15) <= 0.005


def test_make_shards_matches_reference():
    G = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
    specs = tagc.gpt2_specs()
    assert [s.param_count for s in specs] == [int(x) for x in G["gpt2_counts"]]
    assert [tagc.api.KIND[s.kind] for s in specs] == [int(x) for x in G["gpt2_kinds"]]
    shards = tagc.make_shards(specs, 2, 2)
    got = [(sh.id, tagc.api.KIND[s.kind], s.begin, s.end) for sh in shards for s in sh.segments]
    assert got == [tuple(int(x) for x in r) for r in G["gpt2_w2_segments"]]
    # padding tail and round-robin owners (test_hook.cpp:312-338)
    toy = tagc.make_shards([tagc.LayerSpec("a", "embedding", 181)], 4, 2)
    assert [s.owner for s in toy] == [0, 1, 0, 1]
    assert toy[3].segments[-1].name == "pad" and toy[3].segments[-1].size() == 4 * 46 - 181
    with pytest.raises(tagc.TagcInvalidArgument):
        tagc.make_shards([], 2, 2)


def test_llama3_8b_layout():
    # 8,030,261,248 params, 298 segments / 136 compressed at W=8
    specs = tagc.llama3_8b_specs()
    assert sum(s.param_count for s in specs) == 8_030_261_248
    shards = tagc.make_shards(specs, 8, 8)
    segs = [s for sh in shards for s in sh.segments]
    comp = [s for s in segs if tagc.kind_compressible(s.kind, "non_attention_linear") and s.size() >= 1024]
    assert len(segs) == 298 and len(comp) == 136
    assert sum(s.size() for s in comp) == 7_224_688_640


def test_exchange_plan_covers_every_segment_once():
    cfg = tagc.CompressionConfig(theta=99.0, ratio=10, index_width=4)
    shards = tagc.make_shards(tagc.gpt2_specs(), 4, 4)
    for rank in range(4):
        plan, bf, bu = tagc.plan_exchange(cfg, shards, 4, rank)
        assert len(plan) == sum(len(s.segments) for s in shards)
        for owner in range(4):
            f_iv, u_iv = [], []
            for p in plan:
                if p["owner"] != owner:
                    continue
                if p["compressed"]:
                    f_iv.append((p["sk_off"], p["sk_off"] + 3 * p["buckets_per_row"]))
                    u_iv.append((p["word_off"], p["word_off"] + p["n_words"]))
                else:
                    f_iv.append((p["raw_off"], p["raw_off"] + p["len"]))
            for iv, cap in ((sorted(f_iv), bf), (sorted(u_iv), bu)):
                for (a0, a1), (b0, _) in zip(iv, iv[1:]):
                    assert a1 <= b0  # disjoint
                assert not iv or iv[-1][1] <= cap
        owned = [p for p in plan if p["owner"] == rank]
        assert all(p["out_off"] != 2**64 - 1 for p in owned)


def test_ledger_csv_json_match_reference(ref):
    """TrafficLedger (collectives.cpp:37-93) on the host: CSV, JSON dump text
    and bits/param aggregates identical to the compiled reference's for the
    same records (cost factors, row order, nlohmann number formatting)."""
    import random

    rnd = random.Random(4)
    ops = ["all_reduce", "reduce", "reduce_scatter", "all_gather"]
    records = []
    for i in range(60):
        op = rnd.randrange(4)
        tag = rnd.choice(["index/", "sketch/", "grad/", "params/"]) + f"shard{rnd.randrange(3)}/l{rnd.randrange(5)}"
        bits = rnd.choice([0, 1, 7, 32 * 768, 3 * 559240 * 32, rnd.randrange(1 << 40), 10 ** 18])
        params = rnd.choice([0, 1, 3, 768, 16_777_216, rnd.randrange(1 << 30), 10 ** 13])
        records.append((op, tag, bits, params))
    records.append((3, "params/allgather", 62_219_904 * 2 * 32, 62_219_904 * 2))
    led = tagc.TrafficLedger()
    for op, tag, bits, params in records:
        led.record(ops[op], tag, bits, params)
    for prefix in ("", "index/", "grad/shard1", "nope"):
        csv, js, bpp = ref.ledger_dump(records, prefix)
        assert led.to_csv() == csv
        assert led.to_json() == js
        assert led.bits_per_param_per_rank(prefix) == bpp
    rows = led.rows()  # TrafficLedger::rows(): (op, tag) order, one row per distinct key
    assert [(r["op"], r["tag"]) for r in rows] == sorted({(ops[o], t) for o, t, _, _ in records},
                                                          key=lambda k: (ops.index(k[0]), k[1]))
    for r in rows:
        mine = [(b, p) for o, t, b, p in records if ops[o] == r["op"] and t == r["tag"]]
        factor = 2 if r["op"] == "all_reduce" else 1
        assert r["calls"] == len(mine) and r["params"] == sum(p for _, p in mine) % 2**64
        assert r["payload_bits"] == sum(b for b, _ in mine) % 2**64
        assert r["charged_bits"] == factor * sum(b for b, _ in mine) % 2**64
    with pytest.raises(tagc.TagcInvalidArgument):
        led.record("broadcast", "x", 1, 1)
    led.clear()
    assert led.to_json() == "[]"


def test_ledger_json_number_format(ref):
    """Doubles across the nlohmann formatting regimes: integral ("4.0"),
    fixed, small ("0.0001"), exponent ("1e-05", "1.5e+17")."""
    cases = [(0, 8, 2), (1, 32, 10), (2, 1, 10_000), (2, 1, 100_000), (2, 3, 7), (1, 15 * 10 ** 16, 1),
             (2, 10 ** 17, 3), (3, 0, 5), (1, 2 ** 60, 3), (2, 1, 3 * 10 ** 9)]
    for op, bits, params in cases:
        led = tagc.TrafficLedger()
        led.record(["all_reduce", "reduce", "reduce_scatter", "all_gather"][op], "t", bits, params)
        _, js, _ = ref.ledger_dump([(op, "t", bits, params)])
        assert led.to_json() == js, (bits, params, led.to_json(), js)
