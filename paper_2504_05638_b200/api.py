"""Python mirror of the reference compressor API for the exchange path, over the
C-ABI (libtagc_b200.so). Names, argument meaning and error behaviour follow
the reference (tagc::CompressionConfig, make_shards, tagc_reduce_shard, ...);
device buffers are torch CUDA tensors used as plain memory (torch is plumbing,
every computation runs in the library's sm_100a kernels).

u32 buffers (index words, positions) are carried in torch.int32 tensors and
reinterpreted bit-for-bit.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _lib
from ._lib import TagcError, TagcInvalidArgument, check, lib

POLICY = {"all_layers": 0, "non_attention_linear": 1, "none": 2}
KIND = {
    "embedding": 0,
    "positional_embedding": 1,
    "attention_qkv": 2,
    "attention_out_proj": 3,
    "feed_forward": 4,
    "lm_head": 5,
    "norm": 6,
    "bias": 7,
    "other": 8,
}
KIND_NAME = {v: k for k, v in KIND.items()}

__all__ = [
    "CompressionConfig", "LayerSpec", "LayerSegment", "ShardSpec", "PeelStats", "Context",
    "make_shards", "kind_compressible", "sketch_geometry", "words_needed", "theta_floor",
    "comm_volume_model", "lhc_comm_volume_model", "TagcError", "TagcInvalidArgument",
    "device_count", "plan_exchange", "TrafficLedger", "STAT_UNAVAILABLE",
]


@dataclass
class CompressionConfig:
    """reference config.hpp:16-35"""

    theta: float = 0.0
    ratio: int = 1
    index_width: int = 4
    policy: str = "non_attention_linear"
    include_out_proj: bool = True
    seed: int = 0
    sketch_rows: int = 3
    allow_low_theta: bool = False
    min_compress_segment: int = 1024

    def c(self) -> _lib.Config:
        if self.policy not in POLICY:
            raise TagcInvalidArgument(2, f"unknown policy: {self.policy}")
        return _lib.Config(float(self.theta), int(self.ratio), int(self.index_width),
                           POLICY[self.policy], int(bool(self.include_out_proj)),
                           int(self.seed) & (2**64 - 1), int(self.sketch_rows),
                           int(bool(self.allow_low_theta)), int(self.min_compress_segment))

    def validate_for_world(self, world_size: int) -> None:
        check(lib.tagc_config_validate(C.byref(self.c()), world_size), "validate_for_world")

    def validate(self) -> None:
        self.validate_for_world(1)


@dataclass
class LayerSpec:
    """reference layers.hpp:27-31"""

    name: str
    kind: str
    param_count: int


@dataclass
class LayerSegment:
    """reference hook.hpp:21-28"""

    name: str
    kind: str
    begin: int
    end: int

    def size(self) -> int:
        return self.end - self.begin


@dataclass
class ShardSpec:
    """reference hook.hpp:30-38"""

    id: int
    owner: int
    begin: int
    end: int
    segments: List[LayerSegment] = field(default_factory=list)

    def size(self) -> int:
        return self.end - self.begin


@dataclass
class PeelStats:
    """reference hook.hpp:45-59"""

    presence: int = 0
    peeled: int = 0
    unresolved: int = 0
    index_lost: int = 0
    index_spurious: int = 0
    compressed_segments: int = 0
    baseline_segments: int = 0

    def peel_success(self) -> float:
        return 1.0 if self.presence == 0 else self.peeled / self.presence

    def index_collision_rate(self) -> float:
        truth = self.presence + self.index_lost - self.index_spurious
        return 0.0 if truth == 0 else (self.index_lost + self.index_spurious) / truth


class _ShardC:
    def __init__(self, shard: ShardSpec):
        self.names = [s.name.encode() for s in shard.segments]
        n = max(1, len(shard.segments))
        self.segs = (_lib.Segment * n)(*[
            _lib.Segment(KIND[s.kind], s.begin, s.end, nm)
            for s, nm in zip(shard.segments, self.names)])
        self.c = _lib.Shard(shard.id, shard.owner, shard.begin, shard.end, self.segs,
                            len(shard.segments))


def device_count() -> int:
    return int(lib.tagc_device_count())


def theta_floor(ratio: int) -> float:
    out = C.c_double()
    check(lib.tagc_theta_floor(ratio, C.byref(out)), "theta_floor")
    return out.value


def kind_compressible(kind: str, policy: str, include_out_proj: bool = True) -> bool:
    """reference layers.cpp:42-65"""
    r = lib.tagc_kind_compressible(KIND[kind], POLICY[policy], int(include_out_proj))
    if r < 0:
        raise TagcInvalidArgument(2, "bad kind/policy")
    return bool(r)


def sketch_geometry(n: int, ratio: int, rows: int = 3) -> dict:
    g = _lib.SketchGeom()
    check(lib.tagc_sketch_geometry(n, ratio, rows, C.byref(g)), "sketch_geometry")
    return {"n": g.n, "ratio": g.ratio, "rows": g.rows, "buckets_per_row": g.buckets_per_row}


def words_needed(n: int, width: int) -> int:
    return int(lib.tagc_index_words(n, width))


def _volume(fn, cfg, world, n):
    v = _lib.CommVolume()
    check(fn(C.byref(cfg.c()), world, int(n or 0), C.byref(v)), "comm_volume_model")
    return {"index_bits": v.index_bits, "sketch_bits": v.sketch_bits,
            "total_bits": v.total_bits, "factor": v.factor}


def comm_volume_model(cfg: CompressionConfig, world_size: int, n: Optional[int] = None) -> dict:
    """reference hook.cpp:202-226"""
    return _volume(lib.tagc_comm_volume_model, cfg, world_size, n)


def lhc_comm_volume_model(cfg: CompressionConfig, world_size: int, n: Optional[int] = None) -> dict:
    """reference hook.cpp:228-236"""
    return _volume(lib.tagc_lhc_comm_volume_model, cfg, world_size, n)


def make_shards(layers: Sequence[LayerSpec], shard_count: int, world_size: int) -> List[ShardSpec]:
    """reference hook.cpp:30-61"""
    names = [l.name.encode() for l in layers]
    arr = (_lib.LayerSpecC * max(1, len(layers)))(*[
        _lib.LayerSpecC(nm, KIND[l.kind], int(l.param_count)) for l, nm in zip(layers, names)])
    h = C.c_void_p()
    check(lib.tagc_make_shards(arr, len(layers), shard_count, world_size, C.byref(h)), "make_shards")
    try:
        out = []
        for i in range(lib.tagc_shard_set_count(h)):
            s = _lib.Shard()
            check(lib.tagc_shard_set_get(h, i, C.byref(s)))
            segs = [LayerSegment(s.segments[j].name.decode(), KIND_NAME[s.segments[j].kind],
                                 int(s.segments[j].begin), int(s.segments[j].end))
                    for j in range(s.num_segments)]
            out.append(ShardSpec(int(s.id), int(s.owner), int(s.begin), int(s.end), segs))
        return out
    finally:
        lib.tagc_shard_set_destroy(h)


def plan_exchange(cfg: CompressionConfig, shards: Sequence[ShardSpec], world_size: int, rank: int):
    """Owner-major exchange layout of tagc_reduce_shards on `rank`:
    (list of per-segment dicts, f32 block size, u32 block size)."""
    scs = [_ShardC(s) for s in shards]
    arr = (_lib.Shard * len(scs))(*[s.c for s in scs])
    n = C.c_uint32()
    bf, bu = C.c_uint64(), C.c_uint64()
    check(lib.tagc_plan_exchange(C.byref(cfg.c()), arr, len(scs), world_size, rank, None, C.byref(n),
                                 C.byref(bf), C.byref(bu)), "plan_exchange")
    segs = (_lib.SegPlan * max(1, n.value))()
    check(lib.tagc_plan_exchange(C.byref(cfg.c()), arr, len(scs), world_size, rank, segs, C.byref(n),
                                 C.byref(bf), C.byref(bu)), "plan_exchange")
    out = [{k: int(getattr(segs[i], k)) for k, _ in _lib.SegPlan._fields_} for i in range(n.value)]
    return out, int(bf.value), int(bu.value)


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


STAT_UNAVAILABLE = 2**64 - 1  # index_lost / index_spurious without the ranks' supports


def _dev_f32(t, n: int, name: str, device: int):
    """The kernels take raw pointers and trust the sizes: check a device
    buffer before its pointer crosses the C-ABI (float32, contiguous, on the
    context's device, at least n elements)."""
    if t is None:
        raise TagcInvalidArgument(2, f"{name}: missing buffer")
    if not t.is_cuda or t.device.index != device:
        raise TagcInvalidArgument(2, f"{name}: must be a CUDA tensor on cuda:{device}")
    if str(t.dtype) != "torch.float32":
        raise TagcInvalidArgument(2, f"{name}: must be float32")
    if not t.is_contiguous():
        raise TagcInvalidArgument(2, f"{name}: must be contiguous")
    if t.numel() < n:
        raise TagcInvalidArgument(2, f"{name}: {t.numel()} elements, needs {n}")


def _ptr_array(ts):
    return (C.c_void_p * len(ts))(*[_ptr(t) for t in ts])


def _text(fn, *args) -> str:
    need = C.c_size_t()
    check(fn(*args, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check(fn(*args, buf, len(buf), None))
    return buf.value.decode()


class TrafficLedger:
    """tagc::TrafficLedger (collectives.hpp:60-81): record(op, tag, payload_bits,
    params), to_csv(), to_json() (the reference's dump() text),
    bits_per_param_per_rank(prefix). Context.ledger() returns the context's
    own ledger (borrowed: valid while the context lives)."""

    OPS = {"all_reduce": 0, "reduce": 1, "reduce_scatter": 2, "all_gather": 3}

    def __init__(self, _handle=None, _owner=None):
        self._own = _handle is None
        self.h = lib.tagc_ledger_create() if _handle is None else _handle
        self._owner = _owner  # keeps a borrowing context alive
        if not self.h:
            raise TagcError(1, "tagc_ledger_create failed")

    def __del__(self):
        if getattr(self, "_own", False) and self.h:
            lib.tagc_ledger_destroy(self.h)
            self.h = None

    def record(self, op: str, tag: str, payload_bits: int, params: int):
        if op not in self.OPS:
            raise TagcInvalidArgument(2, f"unknown collective op: {op}")
        check(lib.tagc_ledger_record(self.h, self.OPS[op], tag.encode(), int(payload_bits), int(params)))

    def to_csv(self) -> str:
        return _text(lib.tagc_ledger_csv, self.h)

    def to_json(self) -> str:
        return _text(lib.tagc_ledger_json, self.h)

    def bits_per_param_per_rank(self, prefix: str = "") -> float:
        out = C.c_double()
        check(lib.tagc_ledger_bits_per_param(self.h, prefix.encode(), C.byref(out)))
        return out.value

    def clear(self):
        check(lib.tagc_ledger_clear(self.h))

    def rows(self):
        """TrafficLedger::rows() (collectives.hpp:67): dicts in (op, tag) order."""
        n = C.c_uint32()
        check(lib.tagc_ledger_row_count(self.h, C.byref(n)))
        names = {v: k for k, v in self.OPS.items()}
        out = []
        for i in range(n.value):
            op = C.c_int32()
            tag = C.create_string_buffer(512)
            calls, pb, cb, pr = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
            check(lib.tagc_ledger_row(self.h, i, C.byref(op), tag, len(tag), C.byref(calls), C.byref(pb),
                                      C.byref(cb), C.byref(pr)))
            out.append({"op": names[op.value], "tag": tag.value.decode(), "calls": calls.value,
                        "payload_bits": pb.value, "charged_bits": cb.value, "params": pr.value})
        return out


class Context:
    """Owns a tagc_ctx (one CUDA stream, workspaces, ledger, optional NCCL comm).

    By default the context enqueues on torch's current CUDA stream so torch
    allocations and library kernels are ordered without extra syncs.
    """

    def __init__(self, cfg: CompressionConfig, world_size: int = 1, rank: int = 0, device: int = 0,
                 nccl_comm: int = 0, stream: Optional[int] = None):
        import torch

        self.torch = torch
        self.cfg = cfg
        self.device = device
        self.world_size = world_size
        self.rank = rank
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
            if stream == 0:
                stream = 1  # cudaStreamLegacy: torch's default stream
        h = C.c_void_p()
        check(lib.tagc_ctx_create(C.byref(cfg.c()), world_size, rank, device, nccl_comm or None,
                                  stream or None, C.byref(h)), "ctx_create")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib.tagc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ misc
    def set_config(self, cfg: CompressionConfig):
        check(lib.tagc_ctx_set_config(self.h, C.byref(cfg.c())), "set_config")
        self.cfg = cfg

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib.tagc_nccl_unique_id(buf), "nccl_unique_id")
        return bytes(buf)

    def init_nccl(self, uid: bytes):
        buf = (C.c_uint8 * 128)(*uid)
        check(lib.tagc_ctx_init_nccl(self.h, buf), "init_nccl")

    def ledger_csv(self) -> str:
        need = C.c_size_t()
        check(lib.tagc_ctx_ledger_csv(self.h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        check(lib.tagc_ctx_ledger_csv(self.h, buf, len(buf), None))
        return buf.value.decode()

    def ledger(self) -> TrafficLedger:
        return TrafficLedger(_handle=lib.tagc_ctx_ledger(self.h), _owner=self)

    def ledger_json(self) -> str:
        return self.ledger().to_json()

    def wire_bytes(self) -> int:
        out = C.c_uint64()
        check(lib.tagc_ctx_wire_bytes(self.h, C.byref(out)), "wire_bytes")
        return out.value

    def to_bytes(self, words) -> bytes:
        """Index::to_bytes / CountSketch::to_bytes of a device u32 / f32 buffer
        (index.cpp:59-69, sketch.cpp:77-89): its little-endian word layout."""
        n = words.numel()
        buf = (C.c_uint8 * max(1, 4 * n))()
        check(lib.tagc_wire_bytes_from_device(self.h, _ptr(words), n, buf), "to_bytes")
        return bytes(buf)[:4 * n]

    def ledger_reset(self):
        check(lib.tagc_ctx_ledger_reset(self.h))

    def workspace_bytes(self) -> int:
        return int(lib.tagc_ctx_workspace_bytes(self.h))

    def set_timing(self, on: bool):
        check(lib.tagc_ctx_set_timing(self.h, int(on)))

    def last_timing(self):
        out = (C.c_float * 5)()
        check(lib.tagc_ctx_last_timing(self.h, out))
        return list(out)

    def set_graphs(self, on: bool):
        """CUDA-graph replay of repeated tagc_reduce_shards calls (default on)."""
        check(lib.tagc_ctx_set_graphs(self.h, int(on)), "set_graphs")

    def last_kernel_spans(self):
        """(select+fused pass, decode) device execution spans in ms (timing mode)."""
        out = (C.c_float * 2)()
        check(lib.tagc_ctx_last_kernel_spans(self.h, out))
        return list(out)

    def last_launches(self) -> int:
        return int(lib.tagc_ctx_last_launches(self.h))

    def last_peel_rounds(self):
        out = (C.c_uint32 * 2)()
        check(lib.tagc_ctx_last_peel_rounds(self.h, out))
        return list(out)

    def sync(self):
        check(lib.tagc_ctx_sync(self.h), "sync")

    def _empty(self, n, dtype=None):
        t = self.torch
        return t.empty(int(n), dtype=dtype or t.float32, device=f"cuda:{self.device}")

    # ------------------------------------------------------------ fused exchange
    def tagc_reduce_shard_sim(self, shard: ShardSpec, grads, accs, out=None, stats=True):
        """reference tagc_reduce_shard (hook.cpp:98-200) with len(grads) simulated ranks."""
        w = len(grads)
        if len(accs) != w:
            raise TagcInvalidArgument(2, "need one accumulator per rank")
        for g, a in zip(grads, accs):
            if g.numel() != shard.size() or a.numel() != shard.size():
                raise TagcInvalidArgument(2, "gradient slice length does not match the shard")
        out = self._empty(shard.size()) if out is None else out
        for i, (g, a) in enumerate(zip(grads, accs)):
            _dev_f32(g, shard.size(), f"grads[{i}]", self.device)
            _dev_f32(a, shard.size(), f"accs[{i}]", self.device)
        _dev_f32(out, shard.size(), "out", self.device)
        sc = _ShardC(shard)
        st = _lib.PeelStats()
        check(lib.tagc_reduce_shard_sim(self.h, C.byref(sc.c), w, _ptr_array(grads), _ptr_array(accs),
                                        _ptr(out), C.byref(st) if stats else None), "tagc_reduce_shard")
        return out, (PeelStats(**st.as_dict()) if stats else None)

    def tagc_reduce_shard_sim_audit(self, shard: ShardSpec, grads, accs, out=None, stats=True):
        """tagc_reduce_shard(..., collect_audit=true): (out, stats, audit),
        audit = audit_exchanged_sum (hook.cpp:191-195)."""
        w = len(grads)
        if len(accs) != w:
            raise TagcInvalidArgument(2, "need one accumulator per rank")
        out = self._empty(shard.size()) if out is None else out
        for i, (g, a) in enumerate(zip(grads, accs)):
            _dev_f32(g, shard.size(), f"grads[{i}]", self.device)
            _dev_f32(a, shard.size(), f"accs[{i}]", self.device)
        _dev_f32(out, shard.size(), "out", self.device)
        audit = self._empty(max(1, shard.size()))
        sc = _ShardC(shard)
        st = _lib.PeelStats()
        check(lib.tagc_reduce_shard_sim_audit(self.h, C.byref(sc.c), w, _ptr_array(grads), _ptr_array(accs),
                                              _ptr(out), C.byref(st) if stats else None, _ptr(audit)),
              "tagc_reduce_shard")
        return out, (PeelStats(**st.as_dict()) if stats else None), audit

    def baseline_reduce_shard_sim(self, shard: ShardSpec, grads, out=None):
        for g in grads:
            if g.numel() != shard.size():
                raise TagcInvalidArgument(2, "gradient slice length does not match the shard")
        out = self._empty(shard.size()) if out is None else out
        sc = _ShardC(shard)
        check(lib.tagc_baseline_reduce_shard_sim(self.h, C.byref(sc.c), len(grads), _ptr_array(grads),
                                                 _ptr(out)), "baseline_reduce_shard")
        return out

    def _check_exchange(self, shards, grad, acc, out, owned):
        end = max((s.end for s in shards), default=0)
        if grad is not None:
            _dev_f32(grad, end, "grad", self.device)
        _dev_f32(acc, end, "acc", self.device)
        if out is not None:
            _dev_f32(out, owned, "out", self.device)

    def tagc_reduce_shards(self, shards: Sequence[ShardSpec], grad, acc, out=None, stats=True):
        """One process per GPU: exchange every shard, decode the owned ones."""
        owned = sum(s.size() for s in shards if s.owner == self.rank)
        out = self._empty(max(owned, 1)) if out is None else out
        self._check_exchange(shards, grad, acc, out, owned)
        scs = [_ShardC(s) for s in shards]
        arr = (_lib.Shard * len(scs))(*[s.c for s in scs])
        st = _lib.PeelStats()
        check(lib.tagc_reduce_shards(self.h, arr, len(scs), _ptr(grad), _ptr(acc), _ptr(out),
                                     C.byref(st) if stats else None), "tagc_reduce_shards")
        return out, (PeelStats(**st.as_dict()) if stats else None)

    def tagc_reduce_shards_host(self, shards: Sequence[ShardSpec], host_grad, acc, host_out=None,
                                stats=False):
        """Host-buffer form (the end-to-end call): host_grad / host_out are CPU
        tensors (pinned for copy/compute overlap), acc stays on the device.
        Asynchronous unless stats: host_out is complete after sync(), or on the
        context stream after host_join()."""
        owned = sum(s.size() for s in shards if s.owner == self.rank)
        if host_out is None:
            host_out = self.torch.empty(max(owned, 1), dtype=self.torch.float32, pin_memory=True)
        for t in (host_grad, host_out):
            if t.is_cuda:
                raise TagcInvalidArgument(2, "host buffers must be CPU tensors")
            if t.dtype != self.torch.float32 or not t.is_contiguous():
                raise TagcInvalidArgument(2, "host buffers must be contiguous float32")
        if host_grad.numel() < max((s.end for s in shards), default=0) or host_out.numel() < owned:
            raise TagcInvalidArgument(2, "host buffer too short for the shard layout")
        self._check_exchange(shards, None, acc, None, owned)
        scs = [_ShardC(s) for s in shards]
        arr = (_lib.Shard * len(scs))(*[s.c for s in scs])
        st = _lib.PeelStats()
        check(lib.tagc_reduce_shards_host(self.h, arr, len(scs), _ptr(host_grad), _ptr(acc), _ptr(host_out),
                                          C.byref(st) if stats else None), "tagc_reduce_shards_host")
        return host_out, (PeelStats(**st.as_dict()) if stats else None)

    def reduce_shards_begin(self, shards: Sequence[ShardSpec], grad, acc, out, send_f, send_u):
        """First half of tagc_reduce_shards for a caller-provided transport:
        encodes into the caller's owner-major send blocks (send_f: world *
        block_f32 floats, send_u: world * block_u32 int32 words, sizes from
        plan_exchange). Returns (block_f32, block_u32)."""
        owned = sum(s.size() for s in shards if s.owner == self.rank)
        self._check_exchange(shards, grad, acc, out, owned)
        scs = [_ShardC(s) for s in shards]
        arr = (_lib.Shard * len(scs))(*[s.c for s in scs])
        pf, pu = C.c_void_p(_ptr(send_f)), C.c_void_p(_ptr(send_u))
        bf, bu = C.c_uint64(), C.c_uint64()
        check(lib.tagc_reduce_shards_begin(self.h, arr, len(scs), _ptr(grad), _ptr(acc), _ptr(out), C.byref(pf),
                                           C.byref(pu), C.byref(bf), C.byref(bu)), "reduce_shards_begin")
        return int(bf.value), int(bu.value)

    def reduce_shards_end(self, recv_f, recv_u, stats=True, recv_support=None):
        """Second half: decode this rank's reduced blocks into the `out` given
        to begin. recv_support (1-bit index): this rank's max-reduced support
        block (reduce_shards_support), so that stats carry index_lost /
        index_spurious; without it they read STAT_UNAVAILABLE."""
        st = _lib.PeelStats()
        if recv_support is not None:
            check(lib.tagc_reduce_shards_end_support(self.h, _ptr(recv_f), _ptr(recv_u), _ptr(recv_support),
                                                     C.byref(st) if stats else None), "reduce_shards_end")
        else:
            check(lib.tagc_reduce_shards_end(self.h, _ptr(recv_f), _ptr(recv_u), C.byref(st) if stats else None),
                  "reduce_shards_end")
        return PeelStats(**st.as_dict()) if stats else None

    def reduce_shards_support(self, send_support):
        """1-bit index, after reduce_shards_begin: this rank's support bytes
        (0/1 per position, owner-major) into send_support (uint8 CUDA tensor
        of world_size * block_bytes); returns block_bytes (= 32 * block_u32)."""
        bb = C.c_uint64()
        p = C.c_void_p(_ptr(send_support))
        check(lib.tagc_reduce_shards_support(self.h, C.byref(p), C.byref(bb)), "reduce_shards_support")
        return int(bb.value)

    def tagc_reduce_shards_audit(self, shards: Sequence[ShardSpec], grad, acc, out=None, stats=True):
        """tagc_reduce_shards with collect_audit (hook.cpp:191-195): returns
        (out, stats, audit), audit laid out like out (zeros over raw segments)."""
        owned = sum(s.size() for s in shards if s.owner == self.rank)
        out = self._empty(max(owned, 1)) if out is None else out
        audit = self._empty(max(owned, 1))
        self._check_exchange(shards, grad, acc, out, owned)
        scs = [_ShardC(s) for s in shards]
        arr = (_lib.Shard * len(scs))(*[s.c for s in scs])
        st = _lib.PeelStats()
        check(lib.tagc_reduce_shards_audit(self.h, arr, len(scs), _ptr(grad), _ptr(acc), _ptr(out),
                                           C.byref(st) if stats else None, _ptr(audit)), "tagc_reduce_shards_audit")
        return out, (PeelStats(**st.as_dict()) if stats else None), audit

    def peer_prepare(self, shards: Sequence[ShardSpec]) -> bytes:
        """Allocate this rank's peer-exchange region for the shard layout and
        return its 64-byte CUDA IPC handle (all-gather it across ranks)."""
        scs = [_ShardC(s) for s in shards]
        arr = (_lib.Shard * len(scs))(*[s.c for s in scs])
        buf = C.create_string_buffer(64)
        check(lib.tagc_ctx_peer_prepare(self.h, arr, len(scs), buf), "peer_prepare")
        return buf.raw

    def peer_open(self, handles: Sequence[bytes]):
        """Map every rank's region (handles in rank order); reduce_shards then
        reduces over peer memory instead of NCCL."""
        blob = b"".join(handles)
        check(lib.tagc_ctx_peer_open(self.h, blob), "peer_open")

    def peer_attach_local(self, ranks: Sequence["Context"]):
        """All ranks' contexts in this process (one GPU): attach their regions."""
        arr = (C.c_void_p * len(ranks))(*[r.h for r in ranks])
        check(lib.tagc_ctx_peer_attach_local(self.h, arr, len(ranks)), "peer_attach_local")

    def host_join(self):
        check(lib.tagc_ctx_host_join(self.h), "host_join")

    def baseline_reduce_shards(self, shards: Sequence[ShardSpec], grad, out=None):
        L = shards[0].size()
        out = self._empty(L) if out is None else out
        scs = [_ShardC(s) for s in shards]
        arr = (_lib.Shard * len(scs))(*[s.c for s in scs])
        check(lib.tagc_baseline_reduce_shards(self.h, arr, len(scs), _ptr(grad), _ptr(out)),
              "baseline_reduce_shards")
        return out

    # ------------------------------------------------------------ per-layer codec
    def apply_accumulator(self, g, acc):
        out = self._empty(g.numel())
        check(lib.tagc_apply_accumulator(self.h, _ptr(g), _ptr(acc), _ptr(out), g.numel()))
        return out

    def sparsify(self, g, theta: float):
        """reference sparsify (sparsify.cpp:18-49): (sparse, residual, tau, zero_count)"""
        n = g.numel()
        sparse, residual = self._empty(n), self._empty(n)
        tau = C.c_float()
        zc = C.c_uint64()
        check(lib.tagc_sparsify(self.h, _ptr(g), n, float(theta), _ptr(sparse), _ptr(residual),
                                C.byref(tau), C.byref(zc)), "sparsify")
        return sparse, residual, tau.value, int(zc.value)

    def index_create(self, values, width: int):
        words = self._empty(max(1, words_needed(values.numel(), width)), self.torch.int32)
        check(lib.tagc_index_create(self.h, _ptr(values), values.numel(), width, _ptr(words)),
              "index_create")
        return words

    def merge_indices(self, words_list):
        out = self._empty(words_list[0].numel(), self.torch.int32)
        check(lib.tagc_merge_indices(self.h, _ptr_array(words_list), len(words_list),
                                     words_list[0].numel(), _ptr(out)), "merge_indices")
        return out

    def index_presence(self, words, n: int, width: int):
        pos = self._empty(max(1, n), self.torch.int32)
        cnt = C.c_uint32()
        check(lib.tagc_index_presence(self.h, _ptr(words), n, width, _ptr(pos), C.byref(cnt)),
              "presence")
        return pos[: cnt.value]

    def sketch_compress(self, values, ratio: int, seed: int, rows: int = 3):
        g = sketch_geometry(values.numel(), ratio, rows)
        out = self._empty(rows * g["buckets_per_row"])
        check(lib.tagc_sketch_compress(self.h, _ptr(values), values.numel(), ratio, rows,
                                       int(seed) & (2**64 - 1), _ptr(out)), "compress")
        return out

    def sketch_add(self, a, b):
        out = self._empty(a.numel())
        check(lib.tagc_sketch_add(self.h, _ptr(a), _ptr(b), _ptr(out), a.numel()), "sketch_add")
        return out

    def apply_optimizer(self, optimizer: str, lr: float, params, decoded, world: int, step: int,
                        adam_v=None, weight_decay: float = 0.0):
        """Owner-side consumer (reference train.cpp:355-359, apply_optimizer
        :202-220): params -= update(decoded / world) in place; adam_v (zeros
        before step 1) is the adamw_nm second moment, updated in place."""
        kinds = {"sgd": 0, "adamw_nm": 1}
        if optimizer not in kinds:
            raise TagcInvalidArgument(2, f"unknown optimizer: {optimizer}")
        n = params.numel()
        if decoded.numel() != n or (adam_v is not None and adam_v.numel() != n):
            raise TagcInvalidArgument(2, "params, decoded and adam_v must have equal length")
        check(lib.tagc_apply_optimizer(self.h, kinds[optimizer], float(lr), float(weight_decay), int(world),
                                       int(step), _ptr(params), _ptr(decoded),
                                       _ptr(adam_v) if adam_v is not None else None, n), "apply_optimizer")
        return params

    def tagc_reduce_shards_step(self, shards: Sequence[ShardSpec], grad, acc, params, optimizer: str, lr: float,
                                step: int, adam_v=None, weight_decay: float = 0.0, out=None, stats=False):
        """tagc_reduce_shards + the owner's optimizer step, fused into the decode
        (SURVEY §8f row 2): params / adam_v / out are laid out like
        tagc_reduce_shards' out; out=None skips storing the decoded values."""
        kinds = {"sgd": 0, "adamw_nm": 1}
        if optimizer not in kinds:
            raise TagcInvalidArgument(2, f"unknown optimizer: {optimizer}")
        owned = sum(s.size() for s in shards if s.owner == self.rank)
        self._check_exchange(shards, grad, acc, out, owned)
        _dev_f32(params, owned, "params", self.device)
        if adam_v is not None:
            _dev_f32(adam_v, owned, "adam_v", self.device)
        scs = [_ShardC(s) for s in shards]
        arr = (_lib.Shard * len(scs))(*[s.c for s in scs])
        st = _lib.PeelStats()
        check(lib.tagc_reduce_shards_step(self.h, arr, len(scs), _ptr(grad), _ptr(acc),
                                          _ptr(out) if out is not None else None, kinds[optimizer], float(lr),
                                          float(weight_decay), int(step), _ptr(params),
                                          _ptr(adam_v) if adam_v is not None else None,
                                          C.byref(st) if stats else None), "tagc_reduce_shards_step")
        return PeelStats(**st.as_dict()) if stats else None

    def overlap_begin(self, shards: Sequence[ShardSpec], grad, acc, out=None):
        """Open an exchange before the gradient exists (tagc_overlap_begin);
        returns out (this rank's decoded shards, complete after finish)."""
        owned = sum(s.size() for s in shards if s.owner == self.rank)
        out = self._empty(max(owned, 1)) if out is None else out
        self._check_exchange(shards, grad, acc, out, owned)
        scs = [_ShardC(s) for s in shards]
        self._overlap_keep = (scs, grad, acc, out)
        arr = (_lib.Shard * len(scs))(*[s.c for s in scs])
        check(lib.tagc_overlap_begin(self.h, arr, len(scs), _ptr(grad), _ptr(acc), _ptr(out)), "overlap_begin")
        return out

    def overlap_ready(self, begin: int, end: int, event=None):
        """The gradient range [begin, end) is written once `event` (a
        torch.cuda.Event recorded on the producer's stream) completes."""
        ev = C.c_void_p(event.cuda_event) if event is not None else None
        check(lib.tagc_overlap_ready(self.h, int(begin), int(end), ev), "overlap_ready")

    def overlap_finish(self, stats=False):
        st = _lib.PeelStats()
        check(lib.tagc_overlap_finish(self.h, C.byref(st) if stats else None), "overlap_finish")
        self._overlap_keep = None
        return PeelStats(**st.as_dict()) if stats else None

    def allgather_params(self, params):
        """World::all_gather of the owners' slices (train.cpp:364) over NCCL,
        in place: params is the padded flat space, this rank's slice is
        params[rank*L:(rank+1)*L]."""
        check(lib.tagc_allgather_params(self.h, _ptr(params), params.numel()), "allgather_params")
        return params

    def peeling_decompress(self, presence, sketch, n: int, ratio: int, seed: int, rows: int = 3):
        """reference peeling_decompress (decode.cpp:53-140): (values, unresolved, peeled_fraction)"""
        cnt = presence.numel()
        vals = self._empty(n)
        unres = self._empty(max(1, cnt), self.torch.int32)
        nu = C.c_uint32()
        pf = C.c_double()
        check(lib.tagc_peeling_decompress(self.h, _ptr(presence) if cnt else None, cnt, n, ratio, rows,
                                          int(seed) & (2**64 - 1), _ptr(sketch), _ptr(vals),
                                          _ptr(unres), C.byref(nu), C.byref(pf)), "peeling_decompress")
        return vals, unres[: nu.value], pf.value

    def estimation_decompress(self, presence, sketch, targets, n: int, ratio: int, seed: int,
                              rows: int = 3):
        out = self._empty(max(1, targets.numel()))
        check(lib.tagc_estimation_decompress(self.h, _ptr(presence), presence.numel(), n, ratio, rows,
                                             int(seed) & (2**64 - 1), _ptr(sketch), _ptr(targets),
                                             targets.numel(), _ptr(out)), "estimation_decompress")
        self.sync()
        return out[: targets.numel()]
