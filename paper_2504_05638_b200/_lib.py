"""ctypes binding of libtagc_b200.so (the C-ABI declared in include/tagc_b200.h).

The library is built in-tree (``__graft_entry__.build()`` / ``make -C
paper_2504_05638_b200/csrc``). Importing this module never falls back to
anything: if the shared library is missing or cannot be loaded the import
fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TAGC_LIB_PATH", os.path.join(HERE, "libtagc_b200.so"))  # override: A/B experiments

OK, RUNTIME, INVALID = 0, 1, 2


class TagcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


class TagcInvalidArgument(TagcError, ValueError):
    """Raised where the reference throws std::invalid_argument (status 2)."""


class Config(C.Structure):
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


class Segment(C.Structure):
    _fields_ = [("kind", C.c_int32), ("begin", C.c_uint64), ("end", C.c_uint64),
                ("name", C.c_char_p)]


class Shard(C.Structure):
    _fields_ = [
        ("id", C.c_uint32),
        ("owner", C.c_uint32),
        ("begin", C.c_uint64),
        ("end", C.c_uint64),
        ("segments", C.POINTER(Segment)),
        ("num_segments", C.c_uint32),
    ]


class PeelStats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in (
        "presence", "peeled", "unresolved", "index_lost", "index_spurious",
        "compressed_segments", "baseline_segments")]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class SketchGeom(C.Structure):
    _fields_ = [("n", C.c_uint32), ("ratio", C.c_uint32), ("rows", C.c_uint32),
                ("buckets_per_row", C.c_uint32)]


class CommVolume(C.Structure):
    _fields_ = [("index_bits", C.c_double), ("sketch_bits", C.c_double),
                ("total_bits", C.c_double), ("factor", C.c_double)]


class SegPlan(C.Structure):
    _fields_ = [(k, C.c_uint32) for k in ("shard", "seg", "compressed", "buckets_per_row", "n_words",
                                          "owner")] + \
               [(k, C.c_uint64) for k in ("lo", "len", "word_off", "sk_off", "raw_off", "out_off")]


class LayerSpecC(C.Structure):
    _fields_ = [("name", C.c_char_p), ("kind", C.c_int32), ("param_count", C.c_uint64)]


VP = C.c_void_p
U32, U64, I32 = C.c_uint32, C.c_uint64, C.c_int32

# name -> (restype, argtypes)
SIGNATURES = {
    "tagc_last_error": (C.c_char_p, []),
    "tagc_abi_version": (C.c_int, []),
    "tagc_device_count": (C.c_int, []),
    "tagc_config_default": (None, [C.POINTER(Config)]),
    "tagc_config_validate": (C.c_int, [C.POINTER(Config), U32]),
    "tagc_theta_floor": (C.c_int, [U32, C.POINTER(C.c_double)]),
    "tagc_kind_compressible": (C.c_int, [I32, I32, I32]),
    "tagc_sketch_geometry": (C.c_int, [U32, U32, U32, C.POINTER(SketchGeom)]),
    "tagc_index_words": (U32, [U32, U32]),
    "tagc_comm_volume_model": (C.c_int, [C.POINTER(Config), U32, U64, C.POINTER(CommVolume)]),
    "tagc_lhc_comm_volume_model": (C.c_int, [C.POINTER(Config), U32, U64, C.POINTER(CommVolume)]),
    "tagc_make_shards": (C.c_int, [C.POINTER(LayerSpecC), U32, U32, U32, C.POINTER(VP)]),
    "tagc_shard_set_count": (U32, [VP]),
    "tagc_shard_set_get": (C.c_int, [VP, U32, C.POINTER(Shard)]),
    "tagc_shard_set_destroy": (None, [VP]),
    "tagc_ctx_create": (C.c_int, [C.POINTER(Config), U32, U32, C.c_int, VP, VP, C.POINTER(VP)]),
    "tagc_ctx_destroy": (None, [VP]),
    "tagc_ctx_set_config": (C.c_int, [VP, C.POINTER(Config)]),
    "tagc_ctx_stream": (VP, [VP]),
    "tagc_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "tagc_ctx_init_nccl": (C.c_int, [VP, C.POINTER(C.c_uint8)]),
    "tagc_ctx_ledger_csv": (C.c_int, [VP, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "tagc_ledger_create": (VP, []),
    "tagc_ledger_destroy": (None, [VP]),
    "tagc_ledger_record": (C.c_int, [VP, C.c_int32, C.c_char_p, U64, U64]),
    "tagc_ledger_csv": (C.c_int, [VP, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "tagc_ledger_json": (C.c_int, [VP, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "tagc_ledger_bits_per_param": (C.c_int, [VP, C.c_char_p, C.POINTER(C.c_double)]),
    "tagc_ledger_clear": (C.c_int, [VP]),
    "tagc_ledger_row_count": (C.c_int, [VP, C.POINTER(U32)]),
    "tagc_ledger_row": (C.c_int, [VP, U32, C.POINTER(C.c_int32), C.c_char_p, C.c_size_t, C.POINTER(U64),
                                  C.POINTER(U64), C.POINTER(U64), C.POINTER(U64)]),
    "tagc_ctx_ledger": (VP, [VP]),
    "tagc_ctx_wire_bytes": (C.c_int, [VP, C.POINTER(U64)]),
    "tagc_wire_bytes_from_device": (C.c_int, [VP, VP, U64, VP]),
    "tagc_ctx_ledger_reset": (C.c_int, [VP]),
    "tagc_ctx_workspace_bytes": (U64, [VP]),
    "tagc_ctx_set_timing": (C.c_int, [VP, C.c_int]),
    "tagc_ctx_last_timing": (C.c_int, [VP, C.POINTER(C.c_float)]),
    "tagc_ctx_last_kernel_spans": (C.c_int, [VP, C.POINTER(C.c_float)]),
    "tagc_ctx_set_graphs": (C.c_int, [VP, C.c_int]),
    "tagc_ctx_last_launches": (U64, [VP]),
    "tagc_ctx_sync": (C.c_int, [VP]),
    "tagc_ctx_last_peel_rounds": (C.c_int, [VP, C.POINTER(U32)]),
    "tagc_reduce_shard_sim": (C.c_int, [VP, C.POINTER(Shard), U32, C.POINTER(VP), C.POINTER(VP), VP,
                                        C.POINTER(PeelStats)]),
    "tagc_baseline_reduce_shard_sim": (C.c_int, [VP, C.POINTER(Shard), U32, C.POINTER(VP), VP]),
    "tagc_reduce_shards": (C.c_int, [VP, C.POINTER(Shard), U32, VP, VP, VP, C.POINTER(PeelStats)]),
    "tagc_reduce_shards_host": (C.c_int, [VP, C.POINTER(Shard), U32, VP, VP, VP, C.POINTER(PeelStats)]),
    "tagc_ctx_host_join": (C.c_int, [VP]),
    "tagc_reduce_shards_begin": (C.c_int, [VP, C.POINTER(Shard), U32, VP, VP, VP, C.POINTER(VP), C.POINTER(VP),
                                            C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "tagc_reduce_shards_end": (C.c_int, [VP, VP, VP, C.POINTER(PeelStats)]),
    "tagc_reduce_shards_support": (C.c_int, [VP, C.POINTER(VP), C.POINTER(C.c_uint64)]),
    "tagc_reduce_shards_end_support": (C.c_int, [VP, VP, VP, VP, C.POINTER(PeelStats)]),
    "tagc_reduce_shards_audit": (C.c_int, [VP, C.POINTER(Shard), U32, VP, VP, VP, C.POINTER(PeelStats), VP]),
    "tagc_reduce_shard_sim_audit": (C.c_int, [VP, C.POINTER(Shard), U32, C.POINTER(VP), C.POINTER(VP), VP,
                                              C.POINTER(PeelStats), VP]),
    "tagc_ctx_peer_prepare": (C.c_int, [VP, C.POINTER(Shard), U32, C.c_char_p]),
    "tagc_ctx_peer_open": (C.c_int, [VP, C.c_char_p]),
    "tagc_ctx_peer_attach_local": (C.c_int, [VP, C.POINTER(VP), U32]),
    "tagc_reduce_shard": (C.c_int, [VP, C.POINTER(Shard), VP, VP, VP, C.POINTER(PeelStats)]),
    "tagc_baseline_reduce_shards": (C.c_int, [VP, C.POINTER(Shard), U32, VP, VP]),
    "tagc_plan_exchange": (C.c_int, [C.POINTER(Config), C.POINTER(Shard), U32, U32, U32,
                                     C.POINTER(SegPlan), C.POINTER(U32), C.POINTER(U64),
                                     C.POINTER(U64)]),
    "tagc_apply_accumulator": (C.c_int, [VP, VP, VP, VP, U64]),
    "tagc_sparsify": (C.c_int, [VP, VP, U32, C.c_double, VP, VP, C.POINTER(C.c_float),
                                C.POINTER(U64)]),
    "tagc_index_create": (C.c_int, [VP, VP, U32, U32, VP]),
    "tagc_merge_indices": (C.c_int, [VP, C.POINTER(VP), U32, U32, VP]),
    "tagc_index_presence": (C.c_int, [VP, VP, U32, U32, VP, C.POINTER(U32)]),
    "tagc_sketch_compress": (C.c_int, [VP, VP, U32, U32, U32, U64, VP]),
    "tagc_sketch_add": (C.c_int, [VP, VP, VP, VP, U64]),
    "tagc_apply_optimizer": (C.c_int, [VP, C.c_int32, C.c_double, C.c_double, U32, U32, VP, VP, VP, U64]),
    "tagc_allgather_params": (C.c_int, [VP, VP, U64]),
    "tagc_overlap_begin": (C.c_int, [VP, VP, U32, VP, VP, VP]),
    "tagc_overlap_ready": (C.c_int, [VP, U64, U64, VP]),
    "tagc_overlap_finish": (C.c_int, [VP, VP]),
    "tagc_reduce_shards_step": (C.c_int, [VP, VP, U32, VP, VP, VP, C.c_int32, C.c_double, C.c_double, U32, VP, VP,
                                          VP]),
    "tagc_peeling_decompress": (C.c_int, [VP, VP, U32, U32, U32, U32, U64, VP, VP, VP, C.POINTER(U32),
                                          C.POINTER(C.c_double)]),
    "tagc_estimation_decompress": (C.c_int, [VP, VP, U32, U32, U32, U32, U64, VP, VP, U32, VP]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU or Python fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int, what: str = ""):
    if status == OK:
        return
    msg = (lib.tagc_last_error() or b"").decode()
    if what:
        msg = f"{what}: {msg}"
    if status == INVALID:
        raise TagcInvalidArgument(status, msg)
    raise TagcError(status, msg)
