"""CPU: pin the oracle (oracle/tagc_oracle.c, the C restatement) to the
reference — the golden values in the reference's own unit tests and the
fixtures in tests/golden generated from the compiled reference
(tests/golden/make_golden.py). Runs without a GPU."""
import json
import os

import numpy as np
import pytest

from oracle import Config, Segment, Shard

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))
with open(os.path.join(HERE, "golden", "golden.json")) as f:
    M = json.load(f)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ------------------------------------------------------------ reference KATs
def test_hash_golden_values(orc):
    # test_hash.cpp:54-63
    assert orc.splitmix64(0) == 0xE220A8397B1DCDAF
    assert orc.splitmix64(1) == 0x910A2DEC89025CC1
    assert [orc.bucket(0x1234, 0, p, 1000) for p in (0, 1, 12345)] == [289, 536, 285]
    assert orc.sign(0x1234, 0, 0) == 1.0 and orc.sign(0x1234, 0, 1) == -1.0


def test_hash_table_matches_reference(orc):
    for k, v in M["splitmix64"].items():
        assert orc.splitmix64(int(k)) == v
    for s, r, p, m, b, sg in zip(G["hash_seed"], G["hash_row"], G["hash_pos"], G["hash_m"],
                                 G["hash_bucket"], G["hash_sign"]):
        assert orc.bucket(int(s), int(r), int(p), int(m)) == b
        assert orc.sign(int(s), int(r), int(p)) == sg


def test_synthetic_stream_matches_reference(orc):
    assert np.array_equal(bits(orc.stream(1000, 5, count=2)), bits(G["stream_n1000_seed5_x2"]))


def test_sparsify_hand_example_and_theta_edges(orc):
    # test_sparsify.cpp:32-47, :106-111
    sp, res, tau, zc = orc.sparsify(np.array([4.0, -1.0, 0.0, 3.0]), 50.0)
    assert tau == 1.0 and zc == 2 and sp.tolist() == [4, 0, 0, 3] and res.tolist() == [0, -1, 0, 0]
    g = np.array([0.5, -1.0, 3.0, 0.0], np.float32)
    sp, res, tau, zc = orc.sparsify(g, 0.0)
    assert np.array_equal(sp, g) and not res.any()
    sp, res, _, _ = orc.sparsify(np.array([1.0, -2.0, 3.0]), 100.0)
    assert not sp.any() and res.tolist() == [1.0, -2.0, 3.0]


def test_sparsify_rejects_bad_input(orc):
    from oracle import InvalidArgument

    for args in ((np.array([1.0]), -1.0), (np.array([1.0]), 100.5), (np.array([1.0, np.nan]), 50.0)):
        with pytest.raises(InvalidArgument):
            orc.sparsify(*args)


def test_sparsify_matches_reference_fixtures(orc):
    for c in M["sparsify"]:
        i = c["i"]
        sp, res, tau, zc = orc.sparsify(G[f"sp{i}_g"], c["theta"])
        assert float(tau) == c["tau"] and zc == c["zero_count"]
        assert np.array_equal(bits(sp), bits(G[f"sp{i}_sparse"]))
        assert np.array_equal(bits(res), bits(G[f"sp{i}_residual"]))
    sp, _, tau, zc = orc.sparsify(G["sp_lognormal_g"], 98.75)
    assert float(tau) == M["sp_lognormal"]["tau"] and zc == M["sp_lognormal"]["zero_count"]
    assert np.array_equal(bits(sp), bits(G["sp_lognormal_sparse"]))


def test_index_layout_and_carries(orc):
    # test_index.cpp:11-22, :31-37, :69-80, :94-108
    assert orc.index_create(np.array([0.0, 1.5, 0.0, -2.0]), 4)[0] == 0x1010
    assert orc.index_create(np.array([-0.0, 3.0]), 1)[0] == 0b10
    c = M["one_bit_carry"]
    a = np.zeros(8, np.float32)
    a[0] = 1.0
    m = orc.merge_indices([orc.index_create(a, 1), orc.index_create(a * 2, 1)])
    assert m[0] == c["merged_word0"] == 2
    assert orc.presence(m, 8, 1).tolist() == c["presence"] == [1]
    v = np.zeros(8, np.float32)
    v[2] = 1.0
    m15 = orc.merge_indices([orc.index_create(v, 4)] * 15)
    assert (m15[0] >> 8) & 15 == 15 and (m15[0] >> 4) & 15 == 0 and (m15[0] >> 12) & 15 == 0
    m16 = orc.merge_indices([orc.index_create(v, 4)] * 16)
    assert (m16[0] >> 8) & 15 == 0 and (m16[0] >> 12) & 15 == 1


def test_index_matches_reference_fixtures(orc):
    for c in M["index"]:
        w = orc.index_create(G[f"ix{c['i']}_v"], c["width"])
        assert np.array_equal(w, G[f"ix{c['i']}_words"])


def test_sketch_matches_reference(orc):
    for c in M["sketch"]:
        got = orc.sketch_compress(G[f"sk{c['i']}_v"], c["ratio"], c["seed"], c["rows"])
        assert np.array_equal(bits(got), bits(G[f"sk{c['i']}_sketch"]))
    # test_sketch.cpp:144-154 golden dump
    v = np.zeros(12, np.float32)
    v[3] = 2.0
    assert orc.sketch_compress(v, 2, 1, 2).reshape(2, 3).tolist() == [[-2.0, 0.0, 0.0], [0.0, 0.0, 2.0]]
    assert '"buckets":[[-2.0,0.0,0.0],[0.0,0.0,2.0]]' in M["sketch_debug_json"]
    assert orc.sketch_geometry(3000, 10) == 100 and orc.sketch_geometry(3000, 2) == 500


def test_peel_matches_reference(orc):
    for c in M["peel"]:
        i = c["i"]
        vals, unres, pf = orc.peeling_decompress(G[f"pe{i}_presence"], G[f"pe{i}_sketch"], c["n"],
                                                 c["ratio"], c["seed"])
        assert pf == c["pf"]
        assert np.array_equal(unres, G[f"pe{i}_unresolved"])
        assert np.array_equal(bits(vals), bits(G[f"pe{i}_values"]))


def test_peel_rejects_duplicates_and_oob(orc):
    from oracle import InvalidArgument

    sk = np.zeros(30, np.float32)
    for pres in ([60], [1, 1]):
        with pytest.raises(InvalidArgument):
            orc.peeling_decompress(np.array(pres, np.uint32), sk, 60, 2, 1)


@pytest.mark.parametrize("case", [c["name"] for c in M["hook"]])
def test_reduce_shard_matches_reference(orc, case):
    c = next(x for x in M["hook"] if x["name"] == case)
    n = c["segments"][-1][2]
    shard = Shard(0, c["owner"], 0, n, [Segment(k, b, e, f"s{j}") for j, (k, b, e) in enumerate(c["segments"])])
    grads = list(orc.stream(n, 31 + c["world"], count=c["world"]))
    accs = [np.zeros(n, np.float32) for _ in range(c["world"])]
    cfg = Config(c["theta"], c["ratio"], c["width"], c["policy"], True, 77, 3, False,
                 c["min_compress_segment"])
    dec, st = orc.tagc_reduce_shard(shard, grads, accs, cfg)
    assert st == c["stats"]
    assert np.array_equal(bits(dec), bits(G[f"hk_{case}_decoded"]))
    assert np.array_equal(bits(np.stack(accs)), bits(G[f"hk_{case}_accs"]))


def test_make_shards_matches_reference(orc):
    from oracle import KIND

    names = {v: k for k, v in KIND.items()}
    layers = [(f"l{i}", names[int(k)], int(c)) for i, (c, k) in enumerate(zip(G["gpt2_counts"], G["gpt2_kinds"]))]
    assert sum(c for _, _, c in layers) == 124_439_808
    shards = orc.make_shards(layers, 2, 2)
    assert shards[0].size == M["gpt2_w2_shard_len"]
    got = [(sh.id, KIND[s.kind], s.begin, s.end) for sh in shards for s in sh.segments]
    assert got == [tuple(int(x) for x in r) for r in G["gpt2_w2_segments"]]


def test_roundtrip_reference_reports_pass():
    # acceptance criterion 1 operating points (reduced trials): the reference
    # itself passes. tests/test_gpu_acceptance.py drives the same generator's
    # trials through the CUDA path at acceptance.cpp's full parameters.
    for r in M["roundtrip"]:
        rep = r["report"]
        assert rep["pass"] == 1 and rep["index_lost"] == 0 and rep["index_spurious"] == 0


def test_oracle_vs_live_reference(orc, ref):
    """When the compiled reference is present, cross-check on fresh seeds."""
    rng = np.random.default_rng(99)
    for t in range(4):
        n = int(rng.integers(5000, 60000))
        world = int(rng.integers(2, 5))
        width = int(rng.choice([1, 4]))
        shard = Shard(0, world - 1, 0, n, [Segment("feed_forward", 0, n)])
        grads = list(orc.stream(n, 1000 + t, count=world))
        cfg = Config(99.0, 10, width, "all_layers", True, int(rng.integers(0, 2**63)), 3, False, 1)
        a1 = [np.zeros(n, np.float32) for _ in range(world)]
        a2 = [np.zeros(n, np.float32) for _ in range(world)]
        d1, s1 = orc.tagc_reduce_shard(shard, grads, a1, cfg)
        d2, s2, _ = ref.tagc_reduce_shard(shard, grads, a2, cfg)
        assert s1 == s2
        assert np.array_equal(bits(d1), bits(d2))
        assert all(np.array_equal(bits(x), bits(y)) for x, y in zip(a1, a2))


def _adamw_nm_f32(params, g, v, lr, wd, step):
    """numpy float32 restatement of apply_optimizer's adamw_nm loop
    (train.cpp:209-219): every operation rounded to fp32, in source order."""
    f = np.float32
    b2, eps = f(0.999), f(1e-8)
    bias_fix = f(1.0) - np.power(b2, f(step), dtype=np.float32)
    v[:] = b2 * v + ((f(1.0) - b2) * g) * g
    vhat = v / bias_fix
    params[:] = params - f(lr) * (g / (np.sqrt(vhat) + eps) + f(wd) * params)


def test_oracle_optimizer(orc):
    """Owner-side consumer (train.cpp:355-359): SGD pinned to the reference's
    own scale_sub_inplace when oracle/_ref is present, adamw_nm to an
    independent fp32 restatement; both bit-exact over several steps."""
    from oracle import Ref

    rng = np.random.default_rng(3)
    n, world = 10_007, 3
    p0 = rng.standard_normal(n).astype(np.float32)
    # sgd
    p_o, p_r = p0.copy(), p0.copy()
    for step in range(1, 4):
        dec = (rng.standard_normal(n) * world).astype(np.float32)
        orc.apply_optimizer(0, 0.01, 0.0, world, step, p_o, dec.copy(), None)
        if Ref.available():
            mean = dec * np.float32(1.0 / np.float32(world))
            Ref().scale_sub_inplace(p_r, mean, np.float32(0.01))
            assert np.array_equal(bits(p_o), bits(p_r)), step
    # adamw_nm (momentum-free: only the second moment is kept)
    p_o, p_n = p0.copy(), p0.copy()
    v_o, v_n = np.zeros(n, np.float32), np.zeros(n, np.float32)
    for step in range(1, 6):
        dec = (rng.standard_normal(n) * world).astype(np.float32)
        dec[rng.integers(0, n, 500)] = 0.0  # unselected positions decode to zero
        orc.apply_optimizer(1, 0.01, 0.1, world, step, p_o, dec.copy(), v_o)
        _adamw_nm_f32(p_n, dec * np.float32(1.0 / np.float32(world)), v_n, 0.01, 0.1, step)
        assert np.array_equal(bits(v_o), bits(v_n)), step
        assert np.array_equal(bits(p_o), bits(p_n)), step


def audit_identity(shard, grads, accs_before, accs_after, cfg_policy="all_layers"):
    """audit_exchanged_sum restated from what the exchange leaves behind: a
    rank's exchanged sparse value is its combined g + acc where sparsify left
    a +0.0 residual (kept, or a +0.0 that was dropped), else +0.0
    (sparsify.cpp:43, kernels.cpp:95); summed over ranks in ascending order."""
    n = shard.size
    out = np.zeros(n, np.float32)
    for s in shard.segments:
        lo, hi = s.begin - shard.begin, s.end - shard.begin
        acc = np.zeros(hi - lo, np.float32)
        for g, a0, a1 in zip(grads, accs_before, accs_after):
            comb = (g[lo:hi] + a0[lo:hi]).astype(np.float32)
            acc = (acc + np.where(bits(a1[lo:hi]) == 0, comb, np.float32(0))).astype(np.float32)
        out[lo:hi] = acc
    return out


def test_audit_identity_matches_reference(orc, ref):
    """collect_audit (hook.cpp:191-195): the reference's own
    audit_exchanged_sum equals the identity the GPU audit kernel computes,
    bit for bit, over error-feedback steps (ties, zeros, 1- and 4-bit)."""
    rng = np.random.default_rng(7)
    for t in range(4):
        n = int(rng.integers(20000, 80000))
        world = int(rng.integers(2, 5))
        width = int(rng.choice([1, 4]))
        shard = Shard(0, 0, 0, n, [Segment("feed_forward", 0, n)])
        cfg = Config(99.0, 10, width, "all_layers", True, 77 + t, 3, False, 1)
        accs = [np.zeros(n, np.float32) for _ in range(world)]
        for step in range(2):
            grads = [g.copy() for g in orc.stream(n, 100 * t + step, count=world)]
            grads[0][:500] = 0.0  # dropped +0.0 elements
            grads[1][500:900] = np.float32(1.5)  # ties at the threshold
            before = [a.copy() for a in accs]
            _, audit = ref.tagc_reduce_shard_audit(shard, grads, accs, cfg)
            assert np.array_equal(bits(audit), bits(audit_identity(shard, grads, before, accs))), (t, step)


def test_roundtrip_generator_pinned_to_reference(orc, ref):
    """oracle/_ref's ref_roundtrip_trial (roundtrip.cpp:65-95, with the
    file-static sample_support restated) fed through the reference's own
    tagc_reduce_shard reproduces roundtrip_experiment's report exactly: the
    generator the GPU acceptance test uses is the reference's."""
    from roundtrip_util import roundtrip_report

    n, trials = 10000, 24
    for theta, ratio, world in ((98.75, 10, 4), (80.0, 2, 2), (90.0, 4, 8)):
        seed = 20250808 + world + ratio
        live = ref.roundtrip(n, trials, theta, ratio, 4, world, seed=seed)

        def run(t, grads, tseed):
            shard = Shard(0, 0, 0, n, [Segment("feed_forward", 0, n)])
            cfg = Config(theta, ratio, 4, "all_layers", True, tseed, 3, False, 1)
            accs = [np.zeros(n, np.float32) for _ in range(world)]
            dec, st, _ = ref.tagc_reduce_shard(shard, list(grads), accs, cfg)
            return dec, st

        rep = roundtrip_report(ref, n, trials, theta, world, seed, run)
        for k in ("trials_fully_peeled", "presence_total", "unresolved_total", "index_lost", "index_spurious",
                  "integer_exact_when_resolved", "pass"):
            assert rep[k] == live[k], (k, rep[k], live[k])
        assert rep["mean_peeled_fraction"] == live["mean_peeled_fraction"]
        assert rep["max_rel_error_resolved"] == live["max_rel_error_resolved"]
