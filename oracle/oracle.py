"""ctypes front-end for the C oracle (oracle/wk_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module, and only as the
checker (or the timed CPU reference arm).  The product package
``paper_2505_02922_b200`` never imports it.

The oracle restates the reference package tierkv
(/root/reference/pkg/src/tierkv) in C with the exact numpy/OpenBLAS evaluation
orders; it is pinned against tierkv by oracle/make_golden.py, whose outputs are
committed under tests/golden/.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libwk_oracle.so")
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.wko_engine_new.restype = _P
        L.wko_engine_new.argtypes = [_P, _P]
        L.wko_engine_free.argtypes = [_P]
        L.wko_engine_clone.restype = _P
        L.wko_engine_clone.argtypes = [_P]
        L.wko_engine_prefill.argtypes = [_P, _P, _P, ctypes.c_int, ctypes.c_int]
        L.wko_engine_decode.argtypes = [_P, _P, _P, _P, ctypes.c_int, ctypes.c_int, _P, _P]
        L.wko_engine_m.argtypes = [_P]
        for fn in ("wko_engine_centroids", "wko_engine_value_sums", "wko_engine_sizes"):
            getattr(L, fn).restype = _P
            getattr(L, fn).argtypes = [_P]
        L.wko_engine_members.restype = _P
        L.wko_engine_members.argtypes = [_P, ctypes.c_int, _P]
        L.wko_engine_counters.argtypes = [_P, _P]
        L.wko_engine_last_retrieval.restype = _P
        L.wko_engine_last_retrieval.argtypes = [_P, _P]
        L.wko_engine_last_estimation.restype = _P
        L.wko_engine_last_estimation.argtypes = [_P, _P]
        L.wko_engine_events.restype = _I64
        L.wko_engine_events.argtypes = [_P, _I64, _P, _P, _P, _P]
        L.wko_spherical_kmeans.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, _P, ctypes.c_int, _P]
        L.wko_rank_clusters.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, ctypes.c_int, _P, _P]
        L.wko_sgemm_nt.argtypes = [_P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]
        L.wko_sgemv.argtypes = [_P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]
        L.wko_dgemv.argtypes = [_P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]
        L.wko_row_norms.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P]
        L.wko_einsum_row.restype = ctypes.c_float
        L.wko_einsum_row.argtypes = [_P, _P, ctypes.c_int]
        L.wko_rng_init.argtypes = [_P, _P]
        L.wko_next64.restype = ctypes.c_uint64
        L.wko_next64.argtypes = [_P]
        L.wko_next_double.restype = ctypes.c_double
        L.wko_next_double.argtypes = [_P]
        L.wko_integers.restype = _I64
        L.wko_integers.argtypes = [_P, _I64]
        L.wko_cache_new.restype = _P
        L.wko_cache_new.argtypes = [_I64, ctypes.c_int, ctypes.c_int]
        L.wko_cache_free.argtypes = [_P]
        L.wko_cache_register.argtypes = [_P, ctypes.c_int32, ctypes.c_int32]
        L.wko_cache_set_capacity.argtypes = [_P, _I64]
        L.wko_cache_step.argtypes = [_P, _P, ctypes.c_int, _I64, ctypes.c_int, _P]
        L.wko_cache_counters.argtypes = [_P, _P]
        L.wko_cache_events.restype = _I64
        L.wko_cache_events.argtypes = [_P, _I64, _P, _P, _P, _P]
        L.wko_cache_is_cached.argtypes = [_P, ctypes.c_int32]
        L.wko_cache_lru.restype = _I64
        L.wko_cache_lru.argtypes = [_P, _P, _I64]
        L.wko_cache_slots.argtypes = [_P, ctypes.c_int32, _P]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(_P)


def pcg64_words(seed) -> np.ndarray:
    """PCG64 state words (state_hi, state_lo, inc_hi, inc_lo) of
    np.random.default_rng(seed) -- clustering.py:81."""
    st = np.random.PCG64(seed).state["state"]
    s, i = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, i >> 64, i & m], dtype=np.uint64)


class Rng:
    def __init__(self, seed):
        self._st = (ctypes.c_uint64 * 6)()
        w = pcg64_words(seed)
        lib().wko_rng_init(ctypes.byref(self._st), _ptr(w))

    def next64(self):
        return lib().wko_next64(ctypes.byref(self._st))

    def random(self):
        return lib().wko_next_double(ctypes.byref(self._st))

    def integers(self, n):
        return lib().wko_integers(ctypes.byref(self._st), n)


# ---- numerics recipes ------------------------------------------------------

def sgemm_nt(P, C):
    P = np.ascontiguousarray(P, np.float32); C = np.ascontiguousarray(C, np.float32)
    out = np.empty((P.shape[0], C.shape[0]), np.float32)
    lib().wko_sgemm_nt(_ptr(P), _ptr(C), P.shape[0], C.shape[0], P.shape[1], _ptr(out))
    return out


def sgemv(A, x, threads=1):
    A = np.ascontiguousarray(A, np.float32); x = np.ascontiguousarray(x, np.float32)
    y = np.empty(A.shape[0], np.float32)
    lib().wko_sgemv(_ptr(A), _ptr(x), A.shape[0], A.shape[1], threads, _ptr(y))
    return y


def dgemv(A, x, threads=1):
    A = np.ascontiguousarray(A, np.float64); x = np.ascontiguousarray(x, np.float64)
    y = np.empty(A.shape[0], np.float64)
    lib().wko_dgemv(_ptr(A), _ptr(x), A.shape[0], A.shape[1], threads, _ptr(y))
    return y


def row_norms(x):
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty(x.shape[0], np.float32)
    lib().wko_row_norms(_ptr(x), x.shape[0], x.shape[1], _ptr(y))
    return y


# ---- clustering / ranking ---------------------------------------------------

def spherical_kmeans(keys, k, iters, seed, threads=1):
    """clustering.py:66-101"""
    keys = np.ascontiguousarray(keys, np.float32)
    n, d = keys.shape
    if k < 1 or k > n:
        raise ValueError(f"bad k={k} for n={n}")
    out = np.empty(n, np.int64)
    w = pcg64_words(seed)
    rc = lib().wko_spherical_kmeans(_ptr(keys), n, d, k, iters, _ptr(w), threads, _ptr(out))
    if rc:
        raise ValueError(f"kmeans rc={rc}")
    return out


def rank_clusters(q, C, threads=1):
    """index.py:61-76"""
    C = np.ascontiguousarray(C, np.float64)
    q = np.ascontiguousarray(q, np.float64)
    m = C.shape[0]
    order = np.empty(m, np.int64); scores = np.empty(m, np.float64)
    if m:
        lib().wko_rank_clusters(_ptr(C), m, C.shape[1], _ptr(q), threads, _ptr(order), _ptr(scores))
    return order, scores


# ---- engine -----------------------------------------------------------------

class _Cfg(ctypes.Structure):
    _fields_ = [("centroid_ratio", ctypes.c_int), ("segment_size", ctypes.c_int),
                ("kmeans_iters", ctypes.c_int), ("update_segment", ctypes.c_int),
                ("sink_tokens", ctypes.c_int), ("local_window", ctypes.c_int),
                ("retrieval_fraction", ctypes.c_double), ("estimation_fraction", ctypes.c_double),
                ("tail_denominator_only", ctypes.c_int), ("rng_seed", ctypes.c_int64),
                ("cache_fraction", ctypes.c_double), ("block_size_bytes", ctypes.c_int),
                ("denominator_eq2", ctypes.c_int), ("metrics_k", ctypes.c_int),
                ("blas_threads", ctypes.c_int)]


class _Met(ctypes.Structure):
    _fields_ = [("step", ctypes.c_int64), ("recall", ctypes.c_double),
                ("rel_error", ctypes.c_double), ("hits", ctypes.c_int64),
                ("misses", ctypes.c_int64), ("bytes_slow_to_fast", ctypes.c_int64),
                ("bytes_fast_internal", ctypes.c_int64), ("denominator_coverage", ctypes.c_double),
                ("log_denominator", ctypes.c_double), ("m", ctypes.c_int64),
                ("r", ctypes.c_int64), ("e", ctypes.c_int64)]


_SEED_CB = ctypes.CFUNCTYPE(None, ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                            ctypes.POINTER(ctypes.c_uint64))


@_SEED_CB
def _seed_cb(rng_seed, kind, idx, out):
    w = pcg64_words(np.random.SeedSequence([int(rng_seed), int(kind), int(idx)]))
    for i in range(4):
        out[i] = int(w[i])


DEFAULTS = dict(centroid_ratio=16, segment_size=8192, kmeans_iters=10, update_segment=1024,
                sink_tokens=4, local_window=64, retrieval_fraction=0.018,
                estimation_fraction=0.232, tail_mode="drop", rng_seed=0, cache_fraction=0.05,
                block_size_bytes=2048, denominator_mode="merged", metrics_k=100)


@dataclass
class OracleMetrics:
    step: int
    recall: float
    rel_error: float | None
    hits: int
    misses: int
    bytes_slow_to_fast: int
    bytes_fast_internal: int
    denominator_coverage: float
    log_denominator: float
    m: int
    r: int
    e: int


class OracleEngine:
    """Restatement of tierkv.HeadEngine (engine.py:40-237)."""

    def __init__(self, blas_threads=1, **cfg):
        c = dict(DEFAULTS)
        c.update(cfg)
        self.cfg = c
        s = _Cfg(c["centroid_ratio"], c["segment_size"], c["kmeans_iters"], c["update_segment"],
                 c["sink_tokens"], c["local_window"], c["retrieval_fraction"],
                 c["estimation_fraction"], int(c["tail_mode"] == "denominator_only"),
                 int(c["rng_seed"]), c["cache_fraction"], c["block_size_bytes"],
                 int(c["denominator_mode"] == "eq2"), c["metrics_k"], blas_threads)
        self._cfg = s
        self._h = lib().wko_engine_new(ctypes.byref(s), ctypes.cast(_seed_cb, _P))
        self.d = None

    def __del__(self):
        if getattr(self, "_h", None):
            lib().wko_engine_free(self._h)
            self._h = None

    def clone(self):
        """Independent copy of the engine state (one prefill serves the G
        heads of a GQA group: the index does not depend on the head)."""
        x = object.__new__(OracleEngine)
        x.cfg, x._cfg, x.d = dict(self.cfg), self._cfg, self.d
        x._h = lib().wko_engine_clone(self._h)
        return x

    def prefill(self, keys, values):
        keys = np.ascontiguousarray(keys, np.float32)
        values = np.ascontiguousarray(values, np.float32)
        self.d = keys.shape[1]
        rc = lib().wko_engine_prefill(self._h, _ptr(keys), _ptr(values), keys.shape[0], keys.shape[1])
        if rc:
            raise ValueError(f"prefill rc={rc}")
        return self

    def decode_step(self, q, k, v, with_oracle=False, with_recall=True):
        q = np.ascontiguousarray(q, np.float64)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        out = np.empty(self.d, np.float64)
        met = _Met()
        rc = lib().wko_engine_decode(self._h, _ptr(q), _ptr(k), _ptr(v), int(with_oracle),
                                     int(with_recall), _ptr(out), ctypes.byref(met))
        if rc:
            raise ValueError(f"decode rc={rc}")
        vals = {f: getattr(met, f) for f, _ in _Met._fields_}
        if not with_oracle:
            vals["rel_error"] = None
        return out, OracleMetrics(**vals)

    # -- state views ----------------------------------------------------------
    @property
    def m(self):
        return lib().wko_engine_m(self._h)

    def _view(self, fn, dtype, shape):
        p = getattr(lib(), fn)(self._h)
        n = int(np.prod(shape))
        if n == 0:
            return np.empty(shape, dtype)
        buf = (ctypes.c_char * (n * np.dtype(dtype).itemsize)).from_address(p)
        return np.frombuffer(buf, dtype=dtype).reshape(shape).copy()

    @property
    def centroids(self):
        return self._view("wko_engine_centroids", np.float64, (self.m, self.d))

    @property
    def value_sums(self):
        return self._view("wko_engine_value_sums", np.float64, (self.m, self.d))

    @property
    def sizes(self):
        return self._view("wko_engine_sizes", np.int64, (self.m,))

    def members(self, c):
        cnt = ctypes.c_int()
        p = lib().wko_engine_members(self._h, c, ctypes.byref(cnt))
        if cnt.value == 0:
            return np.empty(0, np.int32)
        buf = (ctypes.c_int32 * cnt.value).from_address(p)
        return np.frombuffer(buf, dtype=np.int32).copy()

    def counters(self):
        out = np.zeros(12, np.int64)
        lib().wko_engine_counters(self._h, _ptr(out))
        keys = ("hits", "misses", "bytes_slow_to_fast", "bytes_fast_internal", "capacity_blocks",
                "occupied_blocks", "bytes_read_total", "clusters", "n_blocks",
                "bytes_written_total", "total_tokens", "buffer_start")
        return dict(zip(keys, (int(x) for x in out)))

    def last_plan(self):
        res = []
        for fn in ("wko_engine_last_retrieval", "wko_engine_last_estimation"):
            cnt = ctypes.c_int()
            p = getattr(lib(), fn)(self._h, ctypes.byref(cnt))
            if cnt.value == 0:
                res.append(np.empty(0, np.int32))
            else:
                res.append(np.frombuffer((ctypes.c_int32 * cnt.value).from_address(p),
                                         dtype=np.int32).copy())
        return res

    def events(self):
        n = lib().wko_engine_events(self._h, 0, None, None, None, None)
        t = np.empty(n, np.int32); s = np.empty(n, np.int64)
        c = np.empty(n, np.int32); a = np.empty(n, np.int32)
        lib().wko_engine_events(self._h, n, _ptr(t), _ptr(s), _ptr(c), _ptr(a))
        return t, s, c, a


class OracleCache:
    """Restatement of tierkv.BlockCache driven by an explicit access stream."""

    def __init__(self, capacity_blocks, block_size_bytes=2048, d=128):
        self._h = lib().wko_cache_new(capacity_blocks, block_size_bytes, d)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().wko_cache_free(self._h)
            self._h = None

    def register(self, cid, n_blocks):
        rc = lib().wko_cache_register(self._h, cid, n_blocks)
        if rc:
            raise ValueError(f"register rc={rc}")

    def set_capacity(self, cap):
        lib().wko_cache_set_capacity(self._h, cap)

    def step(self, ids, step, n_steady=0):
        ids = np.ascontiguousarray(ids, np.int32)
        snap = np.zeros(max(1, len(ids)), np.uint8)
        rc = lib().wko_cache_step(self._h, _ptr(ids), len(ids), step, n_steady, _ptr(snap))
        if rc:
            raise ValueError(f"cache step rc={rc}")
        return snap[: len(ids)].astype(bool)

    def counters(self):
        out = np.zeros(8, np.int64)
        lib().wko_cache_counters(self._h, _ptr(out))
        keys = ("hits", "misses", "bytes_slow_to_fast", "bytes_fast_internal", "capacity_blocks",
                "occupied_blocks", "bytes_read_total", "clusters")
        return dict(zip(keys, (int(x) for x in out)))

    def events(self):
        n = lib().wko_cache_events(self._h, 0, None, None, None, None)
        t = np.empty(n, np.int32); s = np.empty(n, np.int64)
        c = np.empty(n, np.int32); a = np.empty(n, np.int32)
        lib().wko_cache_events(self._h, n, _ptr(t), _ptr(s), _ptr(c), _ptr(a))
        return t, s, c, a

    def lru(self):
        n = lib().wko_cache_lru(self._h, None, 0)
        out = np.empty(max(n, 1), np.int32)
        lib().wko_cache_lru(self._h, _ptr(out), n)
        return out[:n]

    def is_cached(self, cid):
        return bool(lib().wko_cache_is_cached(self._h, cid))
