"""ctypes binding of libwavekv.so (include/wavekv.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no fallback: if the library is missing or the device is
not a CUDA GPU, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigError, IntegrityError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwavekv.so")

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64


class IndexViewC(ctypes.Structure):
    _fields_ = [("store_k", _P), ("store_v", _P), ("store_tok", _P), ("cl_off", _P),
                ("cl_size", _P), ("C64", _P), ("C32", _P), ("Cnorm", _P), ("VS32", _P),
                ("VS64", _P), ("s_cap", _I64), ("m_cap", _I64), ("Cmax", _P)]


class SegmentC(ctypes.Structure):
    _fields_ = [("keys", _P), ("values", _P), ("key_stride", _I64), ("L", _I32), ("k", _I32),
                ("unit", _I32), ("cid_base", _I32), ("row_base", _I32), ("tok_base", _I32),
                ("p_off", _I64), ("c_off", _I64), ("rng", ctypes.c_uint64 * 4)]


class BuildScratchC(ctypes.Structure):
    _fields_ = [("P", _P), ("C", _P), ("A", _P), ("perm", _P), ("sims", _P), ("md", _P),
                ("segs_dev", _P), ("status", _P), ("P16", _P)]


class SteadyViewC(ctypes.Structure):
    _fields_ = [("k", _P), ("v", _P), ("tok", _P), ("n", _P), ("next_tok", _P), ("t_cap", _I64)]


class StepViewC(ctypes.Structure):
    _fields_ = [("q", _P), ("m", _P), ("scores", _P), ("rlist", _P), ("elist", _P), ("nr", _P),
                ("ne", _P), ("zmask", _P), ("ru_ids", _P), ("ru_mask", _P), ("ru_pre", _P),
                ("eu_ids", _P), ("eu_mask", _P), ("cnt", _P), ("tail", _P), ("part", _P),
                ("out", _P), ("logden", _P), ("cov", _P), ("status", _P), ("r_cap", _I32),
                ("e_cap", _I32), ("ru_cap", _I32), ("eu_cap", _I32), ("rtok_row", _P),
                ("rtok_mask", _P), ("sel_done", _P), ("rt_cap", _I32), ("pad_", _I32),
                ("eu_x", _P), ("eu_sz", _P), ("rbits", _P), ("ebits", _P), ("pieces", _P),
                ("woff", _P), ("w_cap", _I32), ("pc_cap", _I32), ("arena_k", _P), ("arena_v", _P),
                ("slot_ids", _P), ("slot_off", _P), ("arena_rows", _I64), ("slot_cap", _I64),
                ("block_tokens", _I32), ("pstride", _I32), ("q64", _P), ("xscr", _P), ("xcount", _P)]


class CacheViewC(ctypes.Structure):
    _fields_ = [("nblk", _P), ("slot_off", _P), ("slot_ids", _P), ("cached", _P), ("prev", _P),
                ("next", _P), ("touched", _P), ("last_access", _P), ("lru_ht", _P), ("heap", _P),
                ("heap_n", _P), ("next_slot", _P), ("capacity", _P), ("occupied", _P),
                ("counters", _P), ("ids", _P), ("n_ids", _P), ("snapshot", _P), ("events", _P),
                ("ev_n", _P), ("m_live", _P), ("m_cap", _I64), ("slot_cap", _I64),
                ("heap_cap", _I64), ("ids_cap", _I64), ("ev_cap", _I64), ("block_bytes", _I32),
                ("token_bytes", _I32)]


class Cache2ViewC(ctypes.Structure):
    _fields_ = [(n, _P) for n in ("nblk", "slot_off", "slot_ids", "cached", "touched", "first", "lru",
                                  "lru_tmp", "lru_n", "freel", "free_n", "next_slot", "capacity",
                                  "occupied", "counters", "ids", "n_ids", "snapshot", "scratch",
                                  "m_live")] + [
        ("m_cap", _I64), ("slot_cap", _I64), ("lru_cap", _I64), ("ids_cap", _I64),
        ("block_bytes", _I32), ("token_bytes", _I32), ("block_tokens", _I32), ("piece_rows", _I32)]


class ZoneParamsC(ctypes.Structure):
    _fields_ = [("G", _I32), ("d", _I32), ("blas_threads", _I32),
                ("retrieval_fraction", ctypes.c_double), ("estimation_fraction", ctypes.c_double),
                ("tail_denominator_only", _I32), ("denominator_eq2", _I32), ("score_mode", _I32),
                ("piece_rows", _I32)]


_lib = None

# every symbol include/wavekv.h declares
EXPORTS = ("wk_version", "wk_kmeans_segments", "wk_append_tokens", "wk_score_topk",
           "wk_tripartite_attn", "wk_full_attn", "wk_cache_step", "wk_recall_at_k",
           "wk_cache_offload_step", "wk_host_alloc", "wk_host_free", "wk_decode_step",
           "wk_centroid_scan", "wk_plan_zones", "wk_cache_phase", "wk_attn_partial_f64",
           "wk_merge_f64", "wk_rank_f64", "wk_cluster_sums_f64")


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
                           "there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    R = ctypes.POINTER
    L.wk_version.restype = ctypes.c_int
    L.wk_kmeans_segments.argtypes = [R(IndexViewC), R(SegmentC), ctypes.c_int, R(BuildScratchC),
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, _P]
    L.wk_append_tokens.argtypes = [R(SteadyViewC), _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P]
    L.wk_score_topk.argtypes = [R(IndexViewC), R(StepViewC), R(ZoneParamsC), ctypes.c_int,
                                ctypes.c_int, _P]
    L.wk_tripartite_attn.argtypes = [R(IndexViewC), R(SteadyViewC), R(StepViewC), R(ZoneParamsC),
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]
    L.wk_full_attn.argtypes = [R(IndexViewC), R(SteadyViewC), R(StepViewC), _P, ctypes.c_int,
                               ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]
    L.wk_cache_step.argtypes = [R(CacheViewC), _P, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                _I64, ctypes.c_int, _P, _P]
    L.wk_recall_at_k.argtypes = [R(IndexViewC), R(SteadyViewC), R(StepViewC), _P, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _I64,
                                 ctypes.c_int, _P, _P]
    L.wk_cache_offload_step.argtypes = [R(Cache2ViewC), R(IndexViewC), R(SteadyViewC), R(StepViewC),
                                        ctypes.c_int, _I64, ctypes.c_int, _P]
    L.wk_decode_step.argtypes = [R(IndexViewC), R(SteadyViewC), R(StepViewC), R(ZoneParamsC), _P, _P,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]
    L.wk_centroid_scan.argtypes = [R(IndexViewC), R(StepViewC), R(ZoneParamsC), ctypes.c_int, ctypes.c_int, _P]
    L.wk_plan_zones.argtypes = [R(IndexViewC), R(SteadyViewC), R(StepViewC), R(ZoneParamsC), _P, _P,
                                ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]
    L.wk_cache_phase.argtypes = [R(CacheViewC), _P, _P, ctypes.c_int, _I64, _I64, ctypes.c_int, _P, _P, _P, _P]
    L.wk_attn_partial_f64.argtypes = [_P, _P, _P, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, _P, _P, _P]
    L.wk_merge_f64.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P]
    L.wk_rank_f64.argtypes = [_P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P]
    L.wk_cluster_sums_f64.argtypes = [_P, _P, _P, _P, ctypes.c_int, ctypes.c_int, _P, _P, _P]
    L.wk_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]
    L.wk_host_free.argtypes = [_P]
    for name in EXPORTS:
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def check(rc: int, what: str):
    if rc == 0:
        return
    if rc == -1:
        raise ConfigError(f"{what}: invalid arguments (WK_ECONFIG)")
    raise RuntimeError(f"{what}: CUDA launch failed (rc={rc})")


STATUS_TEXT = {
    1: "exact-rescoring band overflow",
    2: "empty cluster at finalize",
    3: "device block cache over capacity",
    4: "zone union overflow",
    5: "unknown cluster id",
    6: "merge requires at least one non-empty partial",
    7: "steady buffer full (decode capacity)",
}


def raise_status(code: int, what: str):
    if code == 0:
        return
    if code == 6:
        raise ConfigError(f"{what}: {STATUS_TEXT[6]}")
    raise IntegrityError(f"{what}: device status {code} ({STATUS_TEXT.get(code, '?')})")
