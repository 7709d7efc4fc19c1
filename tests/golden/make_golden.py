"""Generates tests/golden/*.npz|json from the UNMODIFIED reference library
(oracle/_ref/libtagc_ref.so, built by oracle/Makefile from
/root/reference/proj/src). Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin the C restatement (oracle/tagc_oracle.c) and the CUDA path
to the reference's own outputs; they are small so they travel with the repo.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import KIND, Config, Ref, Segment, Shard  # noqa: E402


def main():
    ref = Ref()
    out = {}
    meta = {}
    rng = np.random.default_rng(20251017)

    # ---- hash family (test_hash.cpp golden values + a wider table)
    seeds = [0, 1, 0x1234, 77, 0xDEADBEEF, 2**64 - 1, 20250808]
    hp = []
    for seed in seeds:
        for row in range(4):
            for p in [0, 1, 2, 12345, 65535, 1 << 20, 2**32 - 1]:
                for m in [1, 13, 1000, 559240, 35791394]:
                    hp.append((seed, row, p, m, ref.bucket(seed, row, p, m), ref.sign(seed, row, p)))
    a = np.array(hp, dtype=object)
    out["hash_seed"] = np.array([h[0] for h in hp], np.uint64)
    out["hash_row"] = np.array([h[1] for h in hp], np.uint32)
    out["hash_pos"] = np.array([h[2] for h in hp], np.uint32)
    out["hash_m"] = np.array([h[3] for h in hp], np.uint32)
    out["hash_bucket"] = np.array([h[4] for h in hp], np.uint32)
    out["hash_sign"] = np.array([h[5] for h in hp], np.float32)
    meta["splitmix64"] = {str(x): ref.splitmix64(x) for x in [0, 1, 2, 12345, 2**64 - 1]}

    # ---- SyntheticStream (train.cpp:445-459)
    out["stream_n1000_seed5_x2"] = ref.stream(1000, 5, count=2)

    # ---- sparsify (sparsify.cpp:18-49)
    sp_cases = []
    for i in range(40):
        n = int(rng.integers(1, 3000))
        theta = float(rng.integers(0, 10001)) / 100.0
        g = (rng.random(n) * 20 - 10).astype(np.float32)
        g[rng.random(n) < 0.25] = 0.0
        g[rng.random(n) < 1 / 16] = 1.0
        g[rng.random(n) < 1 / 32] = -0.0
        sparse, residual, tau, zc = ref.sparsify(g, theta)
        out[f"sp{i}_g"] = g
        out[f"sp{i}_sparse"] = sparse
        out[f"sp{i}_residual"] = residual
        sp_cases.append({"i": i, "theta": theta, "tau": float(tau), "zero_count": zc})
    ln = ref.stream(100000, 404)[0]
    sparse, residual, tau, zc = ref.sparsify(ln, 98.75)
    out["sp_lognormal_g"] = ln
    out["sp_lognormal_sparse"] = sparse
    meta["sp_lognormal"] = {"theta": 98.75, "tau": float(tau), "zero_count": zc}
    meta["sparsify"] = sp_cases

    # ---- index (index.cpp)
    idx_cases = []
    for i, (n, w) in enumerate([(1, 1), (31, 4), (32, 1), (33, 4), (100, 1), (4099, 4), (4099, 1)]):
        v = np.where(rng.random(n) < 0.3, rng.standard_normal(n), 0).astype(np.float32)
        out[f"ix{i}_v"] = v
        out[f"ix{i}_words"] = ref.index_create(v, w)
        idx_cases.append({"i": i, "n": n, "width": w})
    meta["index"] = idx_cases
    a1 = np.zeros(8, np.float32)
    a1[0] = 1.0
    b1 = a1.copy()
    b1[0] = 2.0
    merged = ref.merge_indices([ref.index_create(a1, 1), ref.index_create(b1, 1)], 8, 1)
    meta["one_bit_carry"] = {"merged_word0": int(merged[0]),
                             "presence": ref.presence(merged, 8, 1).tolist()}

    # ---- sketch (sketch.cpp)
    sk_cases = []
    for i, (n, ratio, rows, seed) in enumerate([(60, 2, 3, 7), (3000, 10, 3, 99), (120, 4, 2, 3),
                                                  (10000, 10, 3, 2**64 - 5), (4096, 2, 5, 9)]):
        v = np.where(rng.random(n) < 0.2, rng.standard_normal(n), 0).astype(np.float32)
        out[f"sk{i}_v"] = v
        out[f"sk{i}_sketch"] = ref.sketch_compress(v, ratio, seed, rows)
        sk_cases.append({"i": i, "n": n, "ratio": ratio, "rows": rows, "seed": seed})
    meta["sketch"] = sk_cases
    v = np.zeros(12, np.float32)
    v[3] = 2.0
    meta["sketch_debug_json"] = ref.sketch_debug_json(v, 2, 2, 1)

    # ---- decode (decode.cpp)
    pe_cases = []
    for i, (n, dens, ratio, seed) in enumerate([(2000, 0.02, 10, 1), (5000, 0.075, 10, 2),
                                                 (3000, 0.3, 2, 3), (300, 1.0, 2, 17),
                                                 (8000, 0.12, 4, 5)]):
        pres = np.sort(rng.choice(n, max(1, int(n * dens)), replace=False)).astype(np.uint32)
        vv = np.zeros(n, np.float32)
        vv[pres] = rng.standard_normal(pres.size).astype(np.float32)
        sk = ref.sketch_compress(vv, ratio, seed)
        vals, unres, pf = ref.peeling_decompress(pres, sk, n, ratio, seed)
        out[f"pe{i}_presence"] = pres
        out[f"pe{i}_sketch"] = sk
        out[f"pe{i}_values"] = vals
        out[f"pe{i}_unresolved"] = unres
        pe_cases.append({"i": i, "n": n, "ratio": ratio, "seed": seed, "pf": pf})
    meta["peel"] = pe_cases

    # ---- hook (hook.cpp:98-200): small shards through tagc_reduce_shard
    hk_cases = []
    specs = [
        ("ffn_w4", 2, 4, 99.0, 10, "all_layers", [("feed_forward", 0, 20000)], 1),
        ("ffn_w1", 2, 1, 98.75, 10, "all_layers", [("feed_forward", 0, 20000)], 1),
        ("w4_8ranks", 8, 4, 99.9, 10, "all_layers", [("feed_forward", 0, 30000)], 1),
        ("mixed", 3, 4, 80.0, 2, "non_attention_linear",
         [("norm", 0, 128), ("feed_forward", 128, 5000), ("feed_forward", 5000, 5500),
          ("attention_qkv", 5500, 7000)], 1024),
        ("r4", 4, 4, 90.0, 4, "all_layers", [("embedding", 0, 12000)], 1),
    ]
    for name, world, width, theta, ratio, policy, segs, minseg in specs:
        n = segs[-1][2]
        shard = Shard(0, world - 1, 0, n, [Segment(k, b, e, f"s{j}") for j, (k, b, e) in enumerate(segs)])
        grads = list(ref.stream(n, 31 + world, count=world))
        accs = [np.zeros(n, np.float32) for _ in range(world)]
        cfg = Config(theta, ratio, width, policy, True, 77, 3, False, minseg)
        dec, st, csv = ref.tagc_reduce_shard(shard, grads, accs, cfg)
        # grads are regenerated by the tests with the (separately pinned) stream
        out[f"hk_{name}_decoded"] = dec
        out[f"hk_{name}_accs"] = np.stack(accs)
        hk_cases.append({"name": name, "world": world, "width": width, "theta": theta, "ratio": ratio,
                         "policy": policy, "segments": segs, "min_compress_segment": minseg,
                         "owner": world - 1, "stats": st, "ledger_csv": csv})
    meta["hook"] = hk_cases

    # ---- comm volume model (hook.cpp:202-236)
    vol = []
    for width, ratio, theta, world, n, lhc in [(1, 10, 98.75, 2, 0, 0), (4, 2, 80.0, 2, 0, 0),
                                                (4, 2, 80.0, 2, 0, 1), (4, 10, 98.75, 2, 0, 0),
                                                (4, 10, 98.75, 2, 10000, 0), (4, 1, 0.0, 2, 0, 0)]:
        cfg = Config(theta, ratio, width, "all_layers", True, 7, 3, False, 1)
        vol.append({"width": width, "ratio": ratio, "theta": theta, "world": world, "n": n,
                    "lhc": lhc, "out": ref.comm_volume(cfg, world, n, bool(lhc))})
    meta["volume"] = vol

    # ---- make_shards (hook.cpp:30-61) for GPT-2 small (tied) and the test_hook toy
    counts, kinds = ref.model_layer_specs(12, 768, 12, 4, 50257, 1024, False)
    out["gpt2_counts"] = counts
    out["gpt2_kinds"] = kinds
    sl, segs = ref.make_shards(counts, kinds, 2, 2)
    out["gpt2_w2_segments"] = np.array(segs, np.uint64)
    meta["gpt2_w2_shard_len"] = sl

    # ---- roundtrip_experiment (roundtrip.cpp:31-144), reduced trial counts
    rt = []
    for theta, ratio, world in [(80.0, 2, 2), (90.0, 4, 4), (98.75, 10, 8)]:
        rep = ref.roundtrip(10000, 40, theta, ratio, 4, world, 3, 20250808 + world + ratio)
        rt.append({"theta": theta, "ratio": ratio, "world": world, "report": rep})
    meta["roundtrip"] = rt

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
