"""GPU parity of the one-process-per-GPU entry points at the bench workload
(BASELINE config 2: GPT-2 small, tied head, 124M fp32, make_shards(specs, 1, 1),
non_attention_linear + out-proj, theta 99, ratio 10, 4-bit index, seed 77):

* tagc_reduce_shards (device buffers, the NCCL-world path bench.py times), and
* tagc_reduce_shards_host (host buffers, the e2e path; asynchronous and
  pipelined across calls with double-buffered device copies),

both against the CPU oracle's tagc_reduce_shard (reference hook.cpp:98-200)
over three error-feedback steps with distinct gradients: residual
accumulators bit-exact (sparsification mask), peel statistics exact, decoded
values within the reference's 1e-5 tolerance (roundtrip.cpp:119-137)."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2504_05638_b200 as tagc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
STEPS = 3
CFG = dict(theta=99.0, ratio=10, index_width=4, policy="non_attention_linear", include_out_proj=True,
           seed=77)


def lognormal(n, seed):
    """SyntheticStream's distribution (log-normal magnitude, fair sign), numpy-fast."""
    rng = np.random.default_rng(seed)
    mag = np.exp(rng.standard_normal(n, dtype=np.float32))
    return np.where(rng.integers(0, 2, n, dtype=np.int8) == 1, -mag, mag).astype(np.float32)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def check_close(got, ref, tol=1e-5):
    scale = float(np.abs(ref).max())
    err = float(np.max(np.abs(got.astype(np.float64) - ref) / np.maximum(np.abs(ref), scale)))
    assert err <= tol, err
    return err


@pytest.fixture(scope="module")
def world1(orc):
    specs = tagc.gpt2_specs()
    shards = tagc.make_shards(specs, 1, 1)
    sh = shards[0]
    osh = O.Shard(sh.id, sh.owner, sh.begin, sh.end,
                  [O.Segment(s.kind, s.begin, s.end, s.name) for s in sh.segments])
    c = tagc.CompressionConfig(**CFG)
    ocfg = O.Config(c.theta, c.ratio, c.index_width, c.policy, c.include_out_proj, c.seed,
                    c.sketch_rows, c.allow_low_theta, c.min_compress_segment)
    grads = [lognormal(sh.end, 31 + k) for k in range(STEPS)]
    oacc = [np.zeros(sh.size(), np.float32)]
    refs = []
    for g in grads:
        ref, rst = orc.tagc_reduce_shard(osh, [g], oacc, ocfg)
        refs.append((ref.copy(), dict(rst), oacc[0].copy()))
    return shards, grads, refs


def test_reduce_shards_world1_matches_oracle(world1):
    shards, grads, refs = world1
    n = shards[0].size()
    ctx = tagc.Context(tagc.CompressionConfig(**CFG), device=0)
    acc = torch.zeros(n, device=DEV)
    out = torch.empty(n, device=DEV)
    for g, (ref, rst, oacc) in zip(grads, refs):
        _, st = ctx.tagc_reduce_shards(shards, torch.from_numpy(g).to(DEV), acc, out, stats=True)
        assert np.array_equal(bits(acc.cpu().numpy()), bits(oacc))  # mask bit-exact
        for k in ("presence", "peeled", "unresolved", "compressed_segments", "baseline_segments"):
            assert getattr(st, k) == rst[k], (k, st, rst)
        check_close(out.cpu().numpy(), ref)


def test_reduce_shards_host_pipelined_matches_oracle(world1):
    """Back-to-back asynchronous host-buffer calls (no sync in between): each
    call's host output must be its own step's result, so the double-buffered
    device copies and the copy-stream ordering are exercised."""
    shards, grads, refs = world1
    n = shards[0].size()
    ctx = tagc.Context(tagc.CompressionConfig(**CFG), device=0)
    acc = torch.zeros(n, device=DEV)
    hg = [torch.from_numpy(g).pin_memory() for g in grads]
    ho = [torch.full((n,), float("nan"), dtype=torch.float32).pin_memory() for _ in grads]
    for k in range(STEPS):
        ctx.tagc_reduce_shards_host(shards, hg[k], acc, ho[k])
    ctx.sync()
    for k, (ref, _, _) in enumerate(refs):
        check_close(ho[k].numpy(), ref)
    assert np.array_equal(bits(acc.cpu().numpy()), bits(refs[-1][2]))
    # a synchronous call with stats reports the same peel statistics
    acc.zero_()
    _, st = ctx.tagc_reduce_shards_host(shards, hg[0], acc, ho[0], stats=True)
    for k in ("presence", "peeled", "unresolved"):
        assert getattr(st, k) == refs[0][1][k]
    check_close(ho[0].numpy(), refs[0][0])


def test_host_entry_rejects_device_buffers():
    ctx = tagc.Context(tagc.CompressionConfig(**CFG), device=0)
    sh = tagc.make_shards(tagc.gpt2_specs()[:4], 1, 1)
    n = sh[0].size()
    with pytest.raises(tagc.TagcInvalidArgument):
        ctx.tagc_reduce_shards_host(sh, torch.zeros(n, device=DEV), torch.zeros(n, device=DEV))


def test_graph_replay_matches_oracle(world1):
    """Same buffers every step (new gradient copied in): call 1 runs eagerly,
    call 2 is captured into a CUDA graph, call 3 replays it."""
    shards, grads, refs = world1
    n = shards[0].size()
    ctx = tagc.Context(tagc.CompressionConfig(**CFG), device=0)
    ctx.set_graphs(True)
    acc = torch.zeros(n, device=DEV)
    out = torch.empty(n, device=DEV)
    g_d = torch.empty(n, device=DEV)
    for g, (ref, _, oacc) in zip(grads, refs):
        g_d.copy_(torch.from_numpy(g))
        ctx.tagc_reduce_shards(shards, g_d, acc, out, stats=False)
        ctx.sync()
        assert np.array_equal(bits(acc.cpu().numpy()), bits(oacc))
        check_close(out.cpu().numpy(), ref)
    assert ctx.last_launches() > 10


@pytest.mark.parametrize("width", [4, 1])
def test_nccl_collective_one_rank_matches_oracle(world1, monkeypatch, width):
    """The NCCL data path on one GPU: a one-rank communicator
    (tagc_nccl_unique_id + tagc_ctx_init_nccl) with TAGC_FORCE_COLLECTIVE=1
    runs the grouped ncclReduceScatter of the f32 and u32 owner blocks (and,
    for a 1-bit index with stats, the ncclMax support reduce-scatter), and the
    owner decodes the RECEIVED blocks. Against the oracle over three
    error-feedback steps, and the uncompressed comparator through
    ncclReduceScatter equal to the gradient bit for bit."""
    shards, grads, refs = world1
    monkeypatch.setenv("TAGC_FORCE_COLLECTIVE", "1")
    cfg = dict(CFG, index_width=width)
    ctx = tagc.Context(tagc.CompressionConfig(**cfg), device=0)
    ctx.init_nccl(tagc.Context.nccl_unique_id())
    n = shards[0].size()
    acc = torch.zeros(n, device=DEV)
    out = torch.empty(n, device=DEV)
    if width == 4:
        for g, (ref, rst, oacc) in zip(grads, refs):
            _, st = ctx.tagc_reduce_shards(shards, torch.from_numpy(g).to(DEV), acc, out, stats=True)
            assert np.array_equal(bits(acc.cpu().numpy()), bits(oacc))
            for k in ("presence", "peeled", "unresolved", "compressed_segments", "baseline_segments"):
                assert getattr(st, k) == rst[k], (k, st, rst)
            check_close(out.cpu().numpy(), ref)
    else:  # 1-bit: the in-place W=1 path of a context without the collective as the reference
        ref_ctx = tagc.Context(tagc.CompressionConfig(**cfg), device=0)
        ref_acc = torch.zeros(n, device=DEV)
        ref_out = torch.empty(n, device=DEV)
        for g in grads:
            gd = torch.from_numpy(g).to(DEV)
            _, st = ctx.tagc_reduce_shards(shards, gd, acc, out, stats=True)
            _, rst = ref_ctx.tagc_reduce_shards(shards, gd, ref_acc, ref_out, stats=True)
            assert np.array_equal(bits(acc.cpu().numpy()), bits(ref_acc.cpu().numpy()))
            # values: the same tolerance as against the oracle (peel rounds
            # subtract with float REDs, whose order differs run to run)
            check_close(out.cpu().numpy(), ref_out.cpu().numpy().astype(np.float64))
            assert (st.presence, st.peeled, st.unresolved, st.index_lost, st.index_spurious) == \
                (rst.presence, rst.peeled, rst.unresolved, rst.index_lost, rst.index_spurious)
    g = torch.from_numpy(grads[0]).to(DEV)
    base = torch.empty(n, device=DEV)
    ctx.baseline_reduce_shards(shards, g, base)
    torch.cuda.synchronize()
    assert np.array_equal(bits(base.cpu().numpy()), bits(grads[0]))
