"""Reference-shaped per-head engine over the B200 path.

``HeadEngine`` keeps tierkv's public surface (engine.py:40-237): ``prefill``,
``decode_step(q, new_k, new_v, with_oracle)`` -> (float64 output, StepMetrics)
and the state views the reference's tests read (``index``, ``cache``,
``store``, ``buffer``, ``n_sink``, ``total_tokens``, ``_steady_ids``).  It is a
WaveLayer with one unit and one head (fp32 store by default, so arbitrary fp32
inputs are held exactly), the device block cache in per-head mode and the
device recall@k metric.  Every number is computed by the sm_100a kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .block_cache import DeviceBlockCache
from .config import EngineConfig
from .errors import ConfigError
from .metrics import relative_l2
from .wave import WaveLayer, _stream

DEFAULT_MAX_DECODE = 4096


@dataclass
class StepMetrics:
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


class _IndexView:
    """ClusterIndex-shaped read-only view (index.py:96-139)."""

    def __init__(self, eng):
        self._e = eng

    @property
    def m(self):
        return self._e._lay.units[0].m if self._e._lay else 0

    @property
    def centroids(self):
        return self._e._lay.index_arrays(0)["C64"]

    @property
    def value_sums(self):
        return self._e._lay.index_arrays(0)["VS64"]

    @property
    def sizes(self):
        return self._e._lay.index_arrays(0)["sizes"]

    def member_token_ids(self, c):
        ix = self._e._lay.index_arrays(0)
        o, s = int(ix["offsets"][c]), int(ix["sizes"][c])
        return ix["store_tok"][o:o + s].tolist()

    @property
    def entries(self):
        """MetaIndexEntry list (index.py:24-31) read back from the device index."""
        from .index import MetaIndexEntry
        e = self._e
        ix = e._lay.index_arrays(0)
        desc = e._cache.descriptors(0, len(ix["sizes"]), e._sink_blocks)
        out = []
        for c in range(len(ix["sizes"])):
            o, sz = int(ix["offsets"][c]), int(ix["sizes"][c])
            out.append(MetaIndexEntry(c, ix["C64"][c], ix["VS64"][c], sz, desc[c].slow_block_ids,
                                      ix["store_tok"][o:o + sz].tolist()))
        return out

    def rank(self, q):
        from .index import rank_clusters
        return rank_clusters(q, self.centroids)


class _CacheView:
    """BlockCache-shaped read-only view (block_cache.py:52-225) of the
    engine's device cache: counters, LRU order, mapping table and the event
    log as the reference's dicts."""

    def __init__(self, eng):
        self._e = eng

    def stats(self):
        return self._e._cache.stats(0)

    @property
    def event_log(self):
        from .block_cache import event_dict
        e = self._e
        out, k = [], 0
        for t, s, c, a in e._cache.event_log(0):
            if t == "access":
                ids, cached = e._access[k]
                k += 1
                out.append({"type": "access", "step": s, "clusters": ids, "cached": cached})
            else:
                out.append(event_dict({"evict": 1, "admit": 2, "reject": 3}[t], s, c, a))
        return out

    @property
    def mapping(self):
        e = self._e
        return e._cache.descriptors(0, e._lay.units[0].m, e._sink_blocks)

    @property
    def lru(self):
        return self._e._cache.lru_order(0)

    def __getattr__(self, name):
        st = self._e._cache.stats(0)
        if name in st:
            return st[name]
        raise AttributeError(name)


class _StoreView:
    """SlowTierStore-shaped read-only view (store.py:48-105)."""

    def __init__(self, eng):
        self._e = eng

    @property
    def n_blocks(self):
        return self._e._cache.n_blocks[0]

    @property
    def block_size_bytes(self):
        return self._e.cfg.block_size_bytes

    @property
    def block_capacity(self):
        return self._e._cache.block_cap

    @property
    def bytes_read_total(self):
        return int(self._e._cache.counters[0, 4])

    @property
    def bytes_written_total(self):
        return self.n_blocks * self.block_size_bytes


def _copy_overlap(dst, src):
    """Copy every tensor attribute of ``src`` into the same attribute of
    ``dst`` over their overlapping index range (capacity growth)."""
    for name, a in vars(src).items():
        b = getattr(dst, name, None)
        if isinstance(a, torch.Tensor) and isinstance(b, torch.Tensor) and a.dim() == b.dim() \
                and a.dtype == b.dtype and a.device == b.device:
            sl = tuple(slice(0, min(x, y)) for x, y in zip(a.shape, b.shape))
            b[sl] = a[sl]


class HeadEngine:
    """One attention head's state machine on the GPU (engine.py:40-237)."""

    def __init__(self, cfg: EngineConfig, head: int = 0, *, device="cuda",
                 store_dtype=torch.float32, max_decode: int = DEFAULT_MAX_DECODE,
                 blas_threads: int | None = None, event_cap: int = 1 << 16):
        from .clustering import blas_threads as _bt
        self.cfg = cfg.validate()
        self.head = head
        self.device = torch.device(device)
        self.store_dtype = store_dtype
        self.max_decode = max_decode  # initial capacity; grows (doubling) on demand
        self.blas_threads = _bt() if blas_threads is None else blas_threads
        self.event_cap = event_cap
        self.d = None
        self.step = 0
        self._lay = None
        self._cache = None
        self._access = []       # per-step access stream + snapshot (event_log dicts)
        self._sink_blocks = 0
        self._kv = None         # host copy of every key / value seen (tierkv engine.py:59-82)
        self.index = _IndexView(self)
        self.cache = _CacheView(self)
        self.store = _StoreView(self)

    # -------------------------------------------------------------- state views
    @property
    def total_tokens(self):
        return self._lay.units[0].total if self._lay else 0

    @property
    def n_sink(self):
        return self._lay.units[0].n_sink if self._lay else 0

    @property
    def buffer_start(self):
        return self._lay.units[0].buffer_start

    @property
    def buffer(self):
        """Buffered (unclustered) token ids, oldest first."""
        s = self._lay.units[0]
        return list(range(s.buffer_start, s.total))

    def _steady_ids(self):
        s = self._lay.units[0]
        return list(range(s.n_sink)) + list(range(s.buffer_start, s.total))

    @property
    def _keys(self):
        """Every key seen so far, [total_tokens, d] float32 (engine.py:56)."""
        return None if self._kv is None else self._kv[0][: self.total_tokens]

    @property
    def _values(self):
        return None if self._kv is None else self._kv[1][: self.total_tokens]

    def _keep(self, keys, values):
        n = 0 if self._kv is None else self._kn
        need = n + len(keys)
        if self._kv is None or need > self._kv[0].shape[0]:
            cap = max(need, 1024, 2 * (0 if self._kv is None else self._kv[0].shape[0]))
            kv = (np.empty((cap, self.d), np.float32), np.empty((cap, self.d), np.float32))
            if self._kv is not None:
                kv[0][:n], kv[1][:n] = self._kv[0][:n], self._kv[1][:n]
            self._kv = kv
        self._kv[0][n:need] = keys
        self._kv[1][n:need] = values
        self._kn = need

    # ------------------------------------------------------------------ layers
    def _make_layer(self, n_prefill, max_decode):
        lay = WaveLayer(self.cfg, 1, 1, self.d, max_prefill=n_prefill, max_decode=max_decode,
                        store_dtype=self.store_dtype, device=self.device,
                        blas_threads=self.blas_threads, keep_vs64=True)
        cache = DeviceBlockCache(lay, "head", event_cap=self.event_cap)
        lay.on_clusters_added = lambda units, k: cache.register_new(units)
        # ranking uses the caller's fp64 query (index.py:74): exact re-scoring reads it
        lay.q64 = torch.zeros((1, 1, self.d), dtype=torch.float64, device=self.device)
        return lay, cache

    def _alloc_aux(self):
        lay = self._lay
        self._recall_s = torch.empty((1, lay.s_cap + lay.t_cap), dtype=torch.float32, device=self.device)
        self._recall_f = torch.empty((1, lay.s_cap), dtype=torch.uint8, device=self.device)
        self._recall = torch.zeros(1, dtype=torch.float32, device=self.device)
        self._oracle_out = torch.zeros((1, 1, self.d), dtype=torch.float32, device=self.device)

    def _grow(self):
        """Double the decode capacity: a larger layer + cache, state copied
        over (tierkv has no decode-length limit)."""
        old_lay, old_cache = self._lay, self._cache
        self.max_decode *= 2
        lay, cache = self._make_layer(self._n_prefill, self.max_decode)
        _copy_overlap(lay, old_lay)
        _copy_overlap(cache, old_cache)
        lay.units = [type(u)(**vars(u)) for u in old_lay.units]
        lay.prefilled = old_lay.prefilled
        for name in ("n_blocks", "cap_host", "_registered"):
            setattr(cache, name, list(getattr(old_cache, name)))
        self._lay, self._cache = lay, cache
        self._alloc_aux()

    # ------------------------------------------------------------------ prefill
    def prefill(self, keys, values):
        keys = np.asarray(keys, dtype=np.float32)
        values = np.asarray(values, dtype=np.float32)
        if keys.ndim != 2 or keys.shape != values.shape or keys.shape[0] < 1:
            raise ConfigError(f"bad prefill shapes {keys.shape} / {values.shape}")
        if self.d is not None:
            raise ConfigError("prefill called twice")
        n, d = keys.shape
        self.d = d
        self._n_prefill = n
        self._lay, self._cache = self._make_layer(n, self.max_decode)
        self._keep(keys, values)
        self._lay.prefill(torch.from_numpy(keys)[None].to(self.device),
                          torch.from_numpy(values)[None].to(self.device))
        self._cache.register_new()
        n_sink = self._lay.units[0].n_sink
        self._sink_blocks = -(-n_sink // self._cache.block_cap) if n_sink else 0
        self._alloc_aux()
        return self

    # ------------------------------------------------------------------- decode
    def decode_step(self, q, new_k, new_v, with_oracle: bool = False):
        if self.d is None:
            raise ConfigError("decode_step before prefill")
        d, dev = self.d, self.device
        q = np.asarray(q, dtype=np.float64)
        if q.shape != (d,):
            raise ConfigError(f"query dimension {q.shape} does not match {d}")
        if self.step >= self.max_decode or self._lay.units[0].n_steady + 1 > self._lay.t_cap:
            self._grow()
        lay = self._lay
        s = lay.units[0]
        new_k = np.asarray(new_k, np.float32).reshape(1, d)
        new_v = np.asarray(new_v, np.float32).reshape(1, d)
        self._keep(new_k, new_v)
        qt = torch.from_numpy(q.astype(np.float32)).to(dev).view(1, 1, d)
        lay.q64.copy_(torch.from_numpy(q).view(1, 1, d))
        kt = torch.from_numpy(new_k).to(dev)
        vt = torch.from_numpy(new_v).to(dev)
        c0 = self._cache.counters[0].clone()
        lay.launch_step(qt, kt, vt)
        self._cache.step(self.step)
        sv = lay._step_view(lay._q)
        rc = lay.L.wk_recall_at_k(ctypes.byref(lay._ixv), ctypes.byref(lay._stv), ctypes.byref(sv),
                                  lay.n_store_dev.data_ptr(), 1, 1, d, self.cfg.metrics_k,
                                  lay.blas_threads, self._recall_s.data_ptr(), self._recall_f.data_ptr(),
                                  self._recall_s.shape[1], lay.store_bf16, self._recall.data_ptr(),
                                  ctypes.c_void_p(_stream()))
        _lib.check(rc, "wk_recall_at_k")
        out = lay.out[0, 0].double().cpu().numpy()
        logden = float(lay.logden[0, 0])
        cov = float(lay.cov[0, 0])
        r, e = int(lay.nr[0]), int(lay.ne[0])
        rel = None
        if with_oracle:
            sv.out = self._oracle_out.data_ptr()
            rc = lay.L.wk_full_attn(ctypes.byref(lay._ixv), ctypes.byref(lay._stv), ctypes.byref(sv),
                                    lay.n_store_dev.data_ptr(), 1, 1, d, lay.S, lay.store_bf16,
                                    ctypes.c_void_p(_stream()))
            _lib.check(rc, "wk_full_attn")
            rel = relative_l2(out, self._oracle_out[0, 0].double().cpu().numpy())
        recall = float(self._recall[0])
        lay.check_status("decode_step")
        self._access.append(self._cache.access_stream(0))
        s.total += 1
        s.n_steady += 1
        lay.maybe_update()
        c1 = self._cache.counters[0]
        dk = (c1 - c0).tolist()
        met = StepMetrics(step=self.step, recall=recall, rel_error=rel, hits=int(dk[0]),
                          misses=int(dk[1]), bytes_slow_to_fast=int(dk[2]),
                          bytes_fast_internal=int(dk[3]), denominator_coverage=cov,
                          log_denominator=logden, m=s.m, r=r, e=e)
        self.step += 1
        return out, met

    def oracle_step_output(self, q) -> np.ndarray:
        """Exact attention over everything seen so far (engine.py:234-237)."""
        lay, d = self._lay, self.d
        qt = torch.from_numpy(np.asarray(q, np.float32)).to(self.device).view(1, 1, d)
        return lay.full_attention(qt, out=self._oracle_out)[0, 0].double().cpu().numpy()

    def last_plan(self):
        lay = self._lay
        return lay.rlist[0, 0, :int(lay.nr[0])].cpu().numpy()
