"""roundtrip_experiment's per-trial bookkeeping (reference roundtrip.cpp:31-144),
restated for the tests that drive its generator's trials through another
implementation (the CUDA path, or the reference's own tagc_reduce_shard to
pin the generator). `run_trial(t, grads, seed)` returns (decoded, stats dict)."""
import math

import numpy as np

ACCEPTANCE_POINTS = [(80.0, 2), (90.0, 4), (98.75, 10)]  # acceptance.cpp:74
ACCEPTANCE_WORLDS = (2, 4, 8)                            # acceptance.cpp:79


def acceptance_seed(world, ratio):
    return 20250808 + world + ratio  # acceptance.cpp:87


def rank_sum(grads):
    out = np.zeros(grads.shape[1], np.float32)
    for g in grads:  # kernels::rank_sum, ascending rank order
        out = (out + g).astype(np.float32)
    return out


def roundtrip_report(ref, n, trials, theta, world, seed, run_trial):
    rep = dict(trials_fully_peeled=0, presence_total=0, unresolved_total=0, index_lost=0, index_spurious=0,
               integer_exact_when_resolved=1, max_rel_error_resolved=0.0, max_rel_error_any=0.0,
               min_peeled_fraction=1.0)
    peel_sum = 0.0
    for t in range(trials):
        grads, tseed = ref.roundtrip_trial(n, theta, world, seed, t)
        reference = rank_sum(grads)
        decoded, st = run_trial(t, grads, tseed)
        pf = 1.0 if st["presence"] == 0 else st["peeled"] / st["presence"]
        peel_sum += pf
        rep["min_peeled_fraction"] = min(rep["min_peeled_fraction"], pf)
        for k in ("presence", "unresolved", "index_lost", "index_spurious"):
            rep[k if k.startswith("index") else k + "_total"] += st[k]
        fully = st["unresolved"] == 0
        rep["trials_fully_peeled"] += int(fully)
        clean = fully and st["index_lost"] == 0 and st["index_spurious"] == 0
        if t % 2 == 0:  # integer trial: bit-exact when resolved (roundtrip.cpp:109-118)
            if clean and not np.array_equal(decoded, reference):
                rep["integer_exact_when_resolved"] = 0
        else:  # float trial (roundtrip.cpp:119-137)
            ref64 = reference.astype(np.float64)
            scale = float(np.abs(ref64).max())
            err = np.abs(decoded.astype(np.float64) - ref64)
            nz = err != 0.0
            max_rel = float(np.max(err[nz] / np.maximum(np.abs(ref64[nz]), scale))) if nz.any() else 0.0
            rep["max_rel_error_any"] = max(rep["max_rel_error_any"], max_rel)
            if clean:
                rep["max_rel_error_resolved"] = max(rep["max_rel_error_resolved"], max_rel)
    rep["mean_peeled_fraction"] = peel_sum / trials
    rep["pass"] = int(rep["mean_peeled_fraction"] >= 0.99 and rep["integer_exact_when_resolved"] == 1
                      and rep["max_rel_error_resolved"] <= 1e-5)
    return rep


def zeros_for(theta, n):
    return min(n, math.ceil(theta * n / 100.0))
