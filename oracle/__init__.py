"""Parity oracles for the TAGC exchange path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package. The product package
(``paper_2504_05638_b200``) never imports it: it is the checker, not the
thing measured or shipped.

Two CPU implementations are wrapped with ctypes + numpy:

* ``Oracle`` — ``liboracle.so``, the plain-C restatement in ``tagc_oracle.c``
  (every function cites the reference file:line it follows);
* ``Ref`` — ``_ref/libtagc_ref.so``, the UNMODIFIED reference library
  compiled from /root/reference/proj/src by ``oracle/Makefile`` plus the
  extern "C" shim ``ref_shim.cpp``. It pins the restatement (tests compare the
  two on seeded inputs) and generates ``tests/golden`` fixtures.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

OK, RUNTIME, INVALID = 0, 1, 2

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


class OracleError(Exception):
    def __init__(self, status, what):
        super().__init__(f"{what}: status {status}")
        self.status = status


class InvalidArgument(OracleError, ValueError):
    pass


def _check(status, what):
    if status == OK:
        return
    if status == INVALID:
        raise InvalidArgument(status, what)
    raise OracleError(status, what)


class CConfig(C.Structure):
    _fields_ = [
        ("theta", C.c_double),
        ("ratio", C.c_uint32),
        ("index_width", C.c_uint32),
        ("policy", C.c_int32),
        ("include_out_proj", C.c_int32),
        ("seed", C.c_uint64),
        ("sketch_rows", C.c_uint32),
        ("allow_low_theta", C.c_int32),
        ("min_compress_segment", C.c_uint64),
    ]


class CSegment(C.Structure):
    _fields_ = [("kind", C.c_int32), ("begin", C.c_uint64), ("end", C.c_uint64)]


class CShard(C.Structure):
    _fields_ = [
        ("id", C.c_uint32),
        ("owner", C.c_uint32),
        ("begin", C.c_uint64),
        ("end", C.c_uint64),
        ("segments", C.POINTER(CSegment)),
        ("num_segments", C.c_uint32),
    ]


class CPeelStats(C.Structure):
    _fields_ = [
        ("presence", C.c_uint64),
        ("peeled", C.c_uint64),
        ("unresolved", C.c_uint64),
        ("index_lost", C.c_uint64),
        ("index_spurious", C.c_uint64),
        ("compressed_segments", C.c_uint64),
        ("baseline_segments", C.c_uint64),
    ]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


@dataclass
class Config:
    """Mirror of tagc::CompressionConfig (config.hpp:16-35)."""

    theta: float = 0.0
    ratio: int = 1
    index_width: int = 4
    policy: str = "non_attention_linear"
    include_out_proj: bool = True
    seed: int = 0
    sketch_rows: int = 3
    allow_low_theta: bool = False
    min_compress_segment: int = 1024

    def c(self) -> CConfig:
        return CConfig(
            float(self.theta), self.ratio, self.index_width, POLICY[self.policy],
            int(self.include_out_proj), self.seed & (2**64 - 1), self.sketch_rows,
            int(self.allow_low_theta), self.min_compress_segment,
        )


@dataclass
class Segment:
    kind: str
    begin: int
    end: int
    name: str = "seg"

    @property
    def size(self):
        return self.end - self.begin


@dataclass
class Shard:
    id: int
    owner: int
    begin: int
    end: int
    segments: list

    @property
    def size(self):
        return self.end - self.begin


class _ShardC:
    """Keeps the ctypes arrays alive for one shard."""

    def __init__(self, shard: Shard):
        self.segs = (CSegment * max(1, len(shard.segments)))(
            *[CSegment(KIND[s.kind], s.begin, s.end) for s in shard.segments]
        )
        self.c = CShard(shard.id, shard.owner, shard.begin, shard.end, self.segs,
                        len(shard.segments))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _ptr_array(arrays, t):
    arr = (C.POINTER(t) * len(arrays))(*[_p(a, t) for a in arrays])
    return arr


def ensure_built():
    so = os.path.join(HERE, "liboracle.so")
    if not os.path.exists(so):
        subprocess.check_call(["make", "-s", "liboracle.so"], cwd=HERE)
    return so


class Oracle:
    """The C restatement (tagc_oracle.c)."""

    def __init__(self, path=None):
        self.lib = C.CDLL(path or ensure_built())
        L = self.lib
        L.or_splitmix64.restype = C.c_uint64
        L.or_splitmix64.argtypes = [C.c_uint64]
        L.or_bucket.restype = C.c_uint32
        L.or_sign.restype = C.c_float
        L.or_words_needed.restype = C.c_uint32
        L.or_index_presence.restype = C.c_uint32
        L.or_index_field.restype = C.c_uint32

    # -- hash
    def splitmix64(self, x):
        return int(self.lib.or_splitmix64(C.c_uint64(x & (2**64 - 1))))

    def rowhash(self, seed, row):
        class RH(C.Structure):
            _fields_ = [("a", C.c_uint64), ("b", C.c_uint64), ("c", C.c_uint64), ("d", C.c_uint64)]
        h = RH()
        self.lib.or_rowhash_init(C.byref(h), C.c_uint64(seed & (2**64 - 1)), C.c_uint32(row))
        return h

    def bucket(self, seed, row, p, m):
        h = self.rowhash(seed, row)
        return int(self.lib.or_bucket(C.byref(h), C.c_uint32(p), C.c_uint32(m)))

    def sign(self, seed, row, p):
        h = self.rowhash(seed, row)
        return float(self.lib.or_sign(C.byref(h), C.c_uint32(p)))

    # -- synthetic gradients
    def stream(self, n, seed, count=1, mu=0.0, sigma=1.0):
        class S(C.Structure):
            _fields_ = [("n", C.c_uint64), ("mu", C.c_double), ("sigma", C.c_double),
                        ("state", C.c_uint64)]
        s = S()
        _check(self.lib.or_stream_init(C.byref(s), C.c_uint64(n), C.c_double(mu),
                                       C.c_double(sigma), C.c_uint64(seed)), "stream")
        out = np.empty((count, n), np.float32)
        for i in range(count):
            self.lib.or_stream_next(C.byref(s), _p(out[i], C.c_float))
        return out

    # -- codec
    def sparsify(self, g, theta):
        g = _f32(g)
        n = g.size
        sparse = np.empty(n, np.float32)
        residual = np.empty(n, np.float32)
        tau = C.c_float()
        zc = C.c_uint64()
        _check(self.lib.or_sparsify(_p(g, C.c_float), C.c_size_t(n), C.c_double(theta),
                                    _p(sparse, C.c_float), _p(residual, C.c_float),
                                    C.byref(tau), C.byref(zc)), "sparsify")
        return sparse, residual, np.float32(tau.value), int(zc.value)

    def words_needed(self, n, w):
        return int(self.lib.or_words_needed(C.c_uint32(n), C.c_uint32(w)))

    def index_create(self, values, width):
        v = _f32(values)
        words = np.zeros(max(1, self.words_needed(v.size, width)), np.uint32)
        _check(self.lib.or_index_create(_p(v, C.c_float), C.c_uint32(v.size), C.c_uint32(width),
                                        _p(words, C.c_uint32)), "index_create")
        return words

    def merge_indices(self, words_list):
        ws = [_u32(w) for w in words_list]
        out = np.empty_like(ws[0])
        self.lib.or_rank_sum_words(_p(out, C.c_uint32), _ptr_array(ws, C.c_uint32),
                                   C.c_uint32(len(ws)), C.c_size_t(out.size))
        return out

    def presence(self, words, n, width):
        words = _u32(words)
        out = np.empty(max(1, n), np.uint32)
        k = self.lib.or_index_presence(_p(words, C.c_uint32), C.c_uint32(n), C.c_uint32(width),
                                       _p(out, C.c_uint32))
        return out[:k].copy()

    def sketch_geometry(self, n, ratio, rows=3):
        m = C.c_uint32()
        _check(self.lib.or_sketch_geometry(C.c_uint32(n), C.c_uint32(ratio), C.c_uint32(rows),
                                           C.byref(m)), "sketch_geometry")
        return int(m.value)

    def sketch_compress(self, values, ratio, seed, rows=3):
        v = _f32(values)
        m = self.sketch_geometry(v.size, ratio, rows)
        out = np.empty(rows * m, np.float32)
        _check(self.lib.or_sketch_compress(_p(v, C.c_float), C.c_uint32(v.size), C.c_uint32(ratio),
                                           C.c_uint32(rows), C.c_uint64(seed & (2**64 - 1)),
                                           _p(out, C.c_float)), "sketch_compress")
        return out

    def apply_optimizer(self, kind, lr, weight_decay, world, step, params, decoded, adam_v):
        """train.cpp:355-359 + apply_optimizer (train.cpp:202-220); updates in place."""
        n = params.size
        self.lib.or_apply_optimizer(C.c_int32(kind), C.c_float(lr), C.c_float(weight_decay), C.c_uint32(world),
                                    C.c_uint32(step), _p(params, C.c_float), _p(decoded, C.c_float),
                                    _p(adam_v, C.c_float) if adam_v is not None else None, C.c_size_t(n))

    def rank_sum(self, arrays):
        arrs = [_f32(a) for a in arrays]
        out = np.empty_like(arrs[0])
        self.lib.or_rank_sum(_p(out, C.c_float), _ptr_array(arrs, C.c_float), C.c_uint32(len(arrs)),
                             C.c_size_t(out.size))
        return out

    def peeling_decompress(self, presence, sketch, n, ratio, seed, rows=3):
        pres = _u32(presence) if len(presence) else np.zeros(1, np.uint32)
        sk = _f32(sketch)
        vals = np.empty(n, np.float32)
        unres = np.empty(max(1, len(presence)), np.uint32)
        nu = C.c_uint32()
        pf = C.c_double()
        _check(self.lib.or_peeling_decompress(_p(pres, C.c_uint32), C.c_uint32(len(presence)),
                                              C.c_uint32(n), C.c_uint32(ratio), C.c_uint32(rows),
                                              C.c_uint64(seed & (2**64 - 1)), _p(sk, C.c_float),
                                              _p(vals, C.c_float), _p(unres, C.c_uint32),
                                              C.byref(nu), C.byref(pf)), "peeling_decompress")
        return vals, unres[: nu.value].copy(), float(pf.value)

    def estimation_decompress(self, presence, sketch, targets, n, ratio, seed, rows=3):
        pres = _u32(presence) if len(presence) else np.zeros(1, np.uint32)
        tg = _u32(targets) if len(targets) else np.zeros(1, np.uint32)
        sk = _f32(sketch)
        out = np.empty(max(1, len(targets)), np.float32)
        _check(self.lib.or_estimation_decompress(
            _p(pres, C.c_uint32), C.c_uint32(len(presence)), C.c_uint32(n), C.c_uint32(ratio),
            C.c_uint32(rows), C.c_uint64(seed & (2**64 - 1)), _p(sk, C.c_float),
            _p(tg, C.c_uint32), C.c_uint32(len(targets)), _p(out, C.c_float)),
            "estimation_decompress")
        return out[: len(targets)]

    def config_validate(self, cfg: Config, world):
        return int(self.lib.or_config_validate(C.byref(cfg.c()), C.c_uint32(world)))

    # -- hook
    def tagc_reduce_shard(self, shard: Shard, grads, accs, cfg: Config):
        """Returns (decoded, stats dict); accs (list of float32 arrays) mutated in place."""
        world = len(grads)
        gs = [_f32(g) for g in grads]
        for a in accs:
            assert a.dtype == np.float32 and a.flags.c_contiguous
        sc = _ShardC(shard)
        out = np.empty(shard.size, np.float32)
        st = CPeelStats()
        _check(self.lib.or_tagc_reduce_shard(C.byref(sc.c), _ptr_array(gs, C.c_float),
                                             _ptr_array(accs, C.c_float), C.c_uint32(world),
                                             C.byref(cfg.c()), _p(out, C.c_float), C.byref(st)),
               "tagc_reduce_shard")
        return out, st.as_dict()

    def baseline_reduce_shard(self, shard: Shard, grads):
        gs = [_f32(g) for g in grads]
        sc = _ShardC(shard)
        out = np.empty(shard.size, np.float32)
        _check(self.lib.or_baseline_reduce_shard(C.byref(sc.c), _ptr_array(gs, C.c_float),
                                                 C.c_uint32(len(gs)), _p(out, C.c_float)),
               "baseline_reduce_shard")
        return out

    def make_shards(self, layers, shard_count, world):
        """layers: list of (name, kind, count). Returns list[Shard]."""
        counts = np.array([c for _, _, c in layers], np.uint64)
        kinds = np.array([KIND[k] for _, k, _ in layers], np.int32)
        ns = C.c_uint32()
        slen = C.c_uint64()
        _check(self.lib.or_make_shards(_p(counts, C.c_uint64), _p(kinds, C.c_int32),
                                       C.c_uint32(len(layers)), C.c_uint32(shard_count),
                                       C.c_uint32(world), C.byref(slen), None, None, None,
                                       C.byref(ns)), "make_shards")
        segs = (CSegment * ns.value)()
        sh = np.empty(ns.value, np.uint32)
        ly = np.empty(ns.value, np.int32)
        _check(self.lib.or_make_shards(_p(counts, C.c_uint64), _p(kinds, C.c_int32),
                                       C.c_uint32(len(layers)), C.c_uint32(shard_count),
                                       C.c_uint32(world), C.byref(slen), segs,
                                       _p(sh, C.c_uint32), _p(ly, C.c_int32), C.byref(ns)),
               "make_shards")
        L = slen.value
        kind_names = {v: k for k, v in KIND.items()}
        shards = [Shard(s, s % world, s * L, (s + 1) * L, []) for s in range(shard_count)]
        for i in range(ns.value):
            name = layers[ly[i]][0] if ly[i] >= 0 else "pad"
            shards[sh[i]].segments.append(
                Segment(kind_names[segs[i].kind], segs[i].begin, segs[i].end, name))
        return shards


class Ref:
    """The unmodified reference library (oracle/_ref/libtagc_ref.so)."""

    PATH = os.path.join(HERE, "_ref", "libtagc_ref.so")

    @classmethod
    def available(cls):
        return os.path.exists(cls.PATH)

    def __init__(self):
        self.lib = C.CDLL(self.PATH)
        L = self.lib
        L.ref_splitmix64.restype = C.c_uint64
        L.ref_splitmix64.argtypes = [C.c_uint64]
        L.ref_bucket.restype = C.c_uint32
        L.ref_bucket.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.ref_sign.restype = C.c_float
        L.ref_sign.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]

    def splitmix64(self, x):
        return int(self.lib.ref_splitmix64(x & (2**64 - 1)))

    def bucket(self, seed, row, p, m):
        return int(self.lib.ref_bucket(seed & (2**64 - 1), row, p, m))

    def sign(self, seed, row, p):
        return float(self.lib.ref_sign(seed & (2**64 - 1), row, p))

    def stream(self, n, seed, count=1, mu=0.0, sigma=1.0):
        out = np.empty((count, n), np.float32)
        _check(self.lib.ref_stream(C.c_uint64(n), C.c_double(mu), C.c_double(sigma),
                                   C.c_uint64(seed), C.c_uint32(count), _p(out, C.c_float)),
               "ref_stream")
        return out

    def sparsify(self, g, theta):
        g = _f32(g)
        n = g.size
        sparse = np.empty(n, np.float32)
        residual = np.empty(n, np.float32)
        tau = C.c_float()
        zc = C.c_uint64()
        _check(self.lib.ref_sparsify(_p(g, C.c_float), C.c_size_t(n), C.c_double(theta),
                                     _p(sparse, C.c_float), _p(residual, C.c_float),
                                     C.byref(tau), C.byref(zc)), "ref_sparsify")
        return sparse, residual, np.float32(tau.value), int(zc.value)

    def index_create(self, values, width):
        v = _f32(values)
        nw = (v.size * width + 31) // 32
        words = np.zeros(max(1, nw), np.uint32)
        _check(self.lib.ref_index_create(_p(v, C.c_float), C.c_uint32(v.size), C.c_uint32(width),
                                         _p(words, C.c_uint32)), "ref_index_create")
        return words

    def merge_indices(self, words_list, n, width):
        ws = [_u32(w) for w in words_list]
        out = np.empty_like(ws[0])
        _check(self.lib.ref_merge_indices(_ptr_array(ws, C.c_uint32), C.c_uint32(len(ws)),
                                          C.c_uint32(n), C.c_uint32(width), _p(out, C.c_uint32)),
               "ref_merge_indices")
        return out

    def presence(self, words, n, width):
        words = _u32(words)
        out = np.empty(max(1, n), np.uint32)
        cnt = C.c_uint32()
        _check(self.lib.ref_index_presence(_p(words, C.c_uint32), C.c_uint32(n), C.c_uint32(width),
                                           _p(out, C.c_uint32), C.byref(cnt)), "ref_presence")
        return out[: cnt.value].copy()

    def ledger_dump(self, records, prefix=""):
        """records: [(op, tag, payload_bits, params)] -> (csv, json, bits_per_param(prefix))."""
        n = len(records)
        ops = (C.c_int32 * max(1, n))(*[r[0] for r in records])
        tags = (C.c_char_p * max(1, n))(*[r[1].encode() for r in records])
        bits = (C.c_uint64 * max(1, n))(*[r[2] for r in records])
        params = (C.c_uint64 * max(1, n))(*[r[3] for r in records])
        csv = C.create_string_buffer(1 << 16)
        js = C.create_string_buffer(1 << 16)
        bpp = C.c_double()
        _check(self.lib.ref_ledger_dump(ops, tags, bits, params, C.c_uint32(n), prefix.encode(), csv,
                                        C.c_size_t(len(csv)), js, C.c_size_t(len(js)), C.byref(bpp)),
               "ref_ledger_dump")
        return csv.value.decode(), js.value.decode(), bpp.value

    def index_to_bytes(self, values, width):
        v = _f32(values)
        out = (C.c_uint8 * max(1, 4 * ((v.size * width + 31) // 32)))()
        _check(self.lib.ref_index_to_bytes(_p(v, C.c_float), C.c_uint32(v.size), C.c_uint32(width), out),
               "ref_index_to_bytes")
        return bytes(out)[:4 * ((v.size * width + 31) // 32)]

    def sketch_to_bytes(self, values, ratio, seed, rows=3):
        v = _f32(values)
        m = v.size // (ratio * rows)
        out = (C.c_uint8 * max(1, 4 * rows * m))()
        _check(self.lib.ref_sketch_to_bytes(_p(v, C.c_float), C.c_uint32(v.size), C.c_uint32(ratio),
                                            C.c_uint32(rows), C.c_uint64(seed & (2**64 - 1)), out),
               "ref_sketch_to_bytes")
        return bytes(out)[:4 * rows * m]

    def scale_sub_inplace(self, dst, src, scale):
        """kernels::scale_sub_inplace (kernels.cpp:32-41), dst updated in place."""
        _check(self.lib.ref_scale_sub_inplace(_p(dst, C.c_float), _p(_f32(src), C.c_float), C.c_size_t(dst.size),
                                              C.c_float(scale)), "ref_scale_sub_inplace")

    def sketch_compress(self, values, ratio, seed, rows=3):
        v = _f32(values)
        m = v.size // (ratio * rows)
        out = np.empty(max(1, rows * m), np.float32)
        _check(self.lib.ref_sketch_compress(_p(v, C.c_float), C.c_uint32(v.size), C.c_uint32(ratio),
                                            C.c_uint32(rows), C.c_uint64(seed & (2**64 - 1)),
                                            _p(out, C.c_float)), "ref_sketch_compress")
        return out

    def sketch_debug_json(self, values, ratio, rows, seed):
        v = _f32(values)
        buf = C.create_string_buffer(1 << 16)
        _check(self.lib.ref_sketch_debug_json(_p(v, C.c_float), C.c_uint32(v.size), C.c_uint32(ratio),
                                              C.c_uint32(rows), C.c_uint64(seed), buf,
                                              C.c_size_t(len(buf))), "ref_sketch_debug_json")
        return buf.value.decode()

    def peeling_decompress(self, presence, sketch, n, ratio, seed, rows=3):
        pres = _u32(presence) if len(presence) else np.zeros(1, np.uint32)
        sk = _f32(sketch)
        vals = np.empty(n, np.float32)
        unres = np.empty(max(1, len(presence)), np.uint32)
        nu = C.c_uint32()
        pf = C.c_double()
        _check(self.lib.ref_peeling_decompress(_p(pres, C.c_uint32), C.c_uint32(len(presence)),
                                               C.c_uint32(n), C.c_uint32(ratio), C.c_uint32(rows),
                                               C.c_uint64(seed & (2**64 - 1)), _p(sk, C.c_float),
                                               _p(vals, C.c_float), _p(unres, C.c_uint32),
                                               C.byref(nu), C.byref(pf)), "ref_peel")
        return vals, unres[: nu.value].copy(), float(pf.value)

    def tagc_reduce_shard(self, shard: Shard, grads, accs, cfg: Config, mode=0):
        world = len(grads)
        gs = [_f32(g) for g in grads]
        sc = _ShardC(shard)
        out = np.empty(shard.size, np.float32)
        st = CPeelStats()
        csv = C.create_string_buffer(1 << 20)
        _check(self.lib.ref_tagc_reduce_shard(C.byref(sc.c), _ptr_array(gs, C.c_float),
                                              _ptr_array(accs, C.c_float), C.c_uint32(world),
                                              C.byref(cfg.c()), C.c_int(mode), _p(out, C.c_float),
                                              C.byref(st), csv, C.c_size_t(len(csv))),
               "ref_tagc_reduce_shard")
        return out, st.as_dict(), csv.value.decode()

    def tagc_reduce_shard_audit(self, shard: Shard, grads, accs, cfg: Config):
        """tagc_reduce_shard(..., collect_audit=true): (decoded, audit_exchanged_sum)."""
        gs = [_f32(g) for g in grads]
        sc = _ShardC(shard)
        out = np.empty(shard.size, np.float32)
        audit = np.empty(shard.size, np.float32)
        _check(self.lib.ref_tagc_reduce_shard_audit(C.byref(sc.c), _ptr_array(gs, C.c_float),
                                                    _ptr_array(accs, C.c_float), C.c_uint32(len(gs)),
                                                    C.byref(cfg.c()), _p(out, C.c_float), _p(audit, C.c_float)),
               "ref_tagc_reduce_shard_audit")
        return out, audit

    def time_reduce_shards(self, shards, grads, cfg: Config, reps=1):
        """Times tagc_reduce_shard over every shard with World(W, parallel);
        returns per-rep seconds (conversion to reference containers untimed)."""
        world = len(grads)
        gs = [_f32(g) for g in grads]
        scs = [_ShardC(s) for s in shards]
        arr = (CShard * len(shards))(*[s.c for s in scs])
        secs = np.zeros(reps, np.float64)
        _check(self.lib.ref_time_reduce_shards(arr, C.c_uint32(len(shards)),
                                               _ptr_array(gs, C.c_float), C.c_uint32(world),
                                               C.byref(cfg.c()), C.c_int(reps),
                                               _p(secs, C.c_double)), "ref_time")
        return secs

    def baseline_reduce_shard(self, shard: Shard, grads):
        gs = [_f32(g) for g in grads]
        sc = _ShardC(shard)
        out = np.empty(shard.size, np.float32)
        _check(self.lib.ref_baseline_reduce_shard(C.byref(sc.c), _ptr_array(gs, C.c_float),
                                                  C.c_uint32(len(gs)), _p(out, C.c_float)),
               "ref_baseline")
        return out

    def config_validate(self, cfg: Config, world):
        return int(self.lib.ref_config_validate(C.byref(cfg.c()), C.c_uint32(world)))

    def comm_volume(self, cfg: Config, world, n=0, lhc=False):
        out = np.zeros(4, np.float64)
        _check(self.lib.ref_comm_volume(C.byref(cfg.c()), C.c_uint32(world), C.c_uint64(n),
                                        C.c_int(int(lhc)), _p(out, C.c_double)), "ref_comm_volume")
        return tuple(float(x) for x in out)

    def model_layer_specs(self, layers, d_model, heads, ffn_mult, vocab, ctx, untied):
        cap = 4096
        counts = np.zeros(cap, np.uint64)
        kinds = np.zeros(cap, np.int32)
        n = C.c_uint32()
        _check(self.lib.ref_model_layer_specs(layers, d_model, heads, ffn_mult, vocab, ctx,
                                              int(untied), _p(counts, C.c_uint64),
                                              _p(kinds, C.c_int32), cap, C.byref(n)), "ref_specs")
        return counts[: n.value].copy(), kinds[: n.value].copy()

    def make_shards(self, counts, kinds, shard_count, world):
        counts = np.ascontiguousarray(counts, np.uint64)
        kinds = np.ascontiguousarray(kinds, np.int32)
        cap = 1 << 16
        segs = (CSegment * cap)()
        sh = np.empty(cap, np.uint32)
        slen = C.c_uint64()
        ns = C.c_uint32()
        _check(self.lib.ref_make_shards(_p(counts, C.c_uint64), _p(kinds, C.c_int32),
                                        C.c_uint32(counts.size), C.c_uint32(shard_count),
                                        C.c_uint32(world), C.byref(slen), segs, _p(sh, C.c_uint32),
                                        C.c_uint32(cap), C.byref(ns)), "ref_make_shards")
        return int(slen.value), [(int(sh[i]), int(segs[i].kind), int(segs[i].begin), int(segs[i].end))
                                 for i in range(ns.value)]

    def roundtrip_trial(self, n, theta, world, seed, t):
        """Trial t of roundtrip_experiment's generator (roundtrip.cpp:65-95):
        (grads [world x n] float32, the trial's compression seed)."""
        g = np.empty((world, n), np.float32)
        ts = C.c_uint64()
        _check(self.lib.ref_roundtrip_trial(C.c_uint32(n), C.c_double(theta), C.c_uint32(world),
                                            C.c_uint64(seed), C.c_uint32(t), _p(g, C.c_float), C.byref(ts)),
               "ref_roundtrip_trial")
        return g, int(ts.value)

    def roundtrip(self, n, trials, theta, ratio, width, world, rows=3, seed=1):
        out = np.zeros(4, np.float64)
        cnt = np.zeros(7, np.uint64)
        _check(self.lib.ref_roundtrip(C.c_uint32(n), C.c_uint32(trials), C.c_double(theta),
                                      C.c_uint32(ratio), C.c_uint32(width), C.c_uint32(world),
                                      C.c_uint32(rows), C.c_uint64(seed), _p(out, C.c_double),
                                      _p(cnt, C.c_uint64)), "ref_roundtrip")
        keys = ["trials_fully_peeled", "presence_total", "unresolved_total", "index_lost",
                "index_spurious", "integer_exact_when_resolved", "pass"]
        d = {k: int(v) for k, v in zip(keys, cnt)}
        d.update(mean_peeled_fraction=out[0], min_peeled_fraction=out[1],
                 max_rel_error_resolved=out[2], max_rel_error_any=out[3])
        return d
