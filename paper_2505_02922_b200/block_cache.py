"""The wave buffer's block cache, device resident (tierkv block_cache.py:52-225).

``DeviceBlockCache`` owns the cache state of every cache unit of a
``WaveLayer`` in HBM; one ``step`` runs lookup + assemble accounting +
commit_update for all of them in one launch (wk_cache_step).  Cache units are
(unit, head) pairs (``mode="head"``: the reference's per-head HeadEngine,
bit-exact event stream) or kv-head units serving the union access stream of
their GQA group (``mode="union"``).  Slow-tier block accounting follows
store.py:38-105: a block holds ``block_size_bytes // (2*d*4)`` tokens,
clusters (and the sink pseudo-cluster) occupy private blocks.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .errors import ConfigError

EVENT_TYPES = {0: "access", 1: "evict", 2: "admit", 3: "reject"}


def block_capacity(block_size_bytes: int, d: int) -> int:
    """Tokens per logical block (store.py:38-45)."""
    cap = block_size_bytes // (2 * d * 4)
    if cap < 1:
        raise ConfigError(f"block_size_bytes={block_size_bytes} cannot hold a single token at d={d}")
    return cap


class DeviceBlockCache:
    def __init__(self, layer, mode: str = "head", event_cap: int = 0):
        if mode not in ("head", "union"):
            raise ConfigError("cache mode must be 'head' or 'union'")
        self.layer = layer
        self.mode = mode
        cfg = layer.cfg
        self.cfg = cfg
        U, G, d, dev = layer.U, layer.G, layer.d, layer.dev
        self.C = U * G if mode == "head" else U
        self.block_cap = block_capacity(cfg.block_size_bytes, d)
        m_cap = layer.m_cap
        self.slot_cap = max(1, layer.s_cap // self.block_cap + m_cap)
        self.ids_cap = layer.r_cap * (1 if mode == "head" else G)
        C, i32, i64 = self.C, torch.int32, torch.int64
        z = lambda *s, dt=i32: torch.zeros(s, dtype=dt, device=dev)
        self.nblk = z(C, m_cap)
        self.slot_off = z(C, m_cap)
        self.slot_ids = z(C, self.slot_cap)
        self.cached = z(C, m_cap, dt=torch.uint8)
        self.prev = torch.full((C, m_cap), -1, dtype=i32, device=dev)
        self.next = torch.full((C, m_cap), -1, dtype=i32, device=dev)
        self.touched = z(C, m_cap)
        self.last_access = torch.full((C, m_cap), -1, dtype=i64, device=dev)
        self.lru_ht = torch.full((C, 2), -1, dtype=i32, device=dev)
        self.heap = z(C, self.slot_cap)
        self.heap_n = z(C)
        self.next_slot = z(C)
        self.capacity = z(C, dt=i64)
        self.occupied = z(C, dt=i64)
        self.counters = z(C, 8, dt=i64)
        self.ids = z(C, self.ids_cap)
        self.n_ids = z(C)
        self.snapshot = z(C, self.ids_cap, dt=torch.uint8)
        self.ev_cap = int(event_cap)
        self.events = z(C, max(1, self.ev_cap), 4) if self.ev_cap else None
        self.ev_n = z(C, dt=i64)
        self.n_blocks = [0] * U          # slow-tier blocks per unit (store.n_blocks)
        self.cap_host = [0] * U
        self._view = _lib.CacheViewC(
            *(t.data_ptr() if t is not None else None for t in (
                self.nblk, self.slot_off, self.slot_ids, self.cached, self.prev, self.next,
                self.touched, self.last_access, self.lru_ht, self.heap, self.heap_n,
                self.next_slot, self.capacity, self.occupied, self.counters, self.ids,
                self.n_ids, self.snapshot, self.events, self.ev_n, layer.m_dev)),
            m_cap, self.slot_cap, self.slot_cap, self.ids_cap, self.ev_cap,
            cfg.block_size_bytes, 2 * d * 4)
        self._registered = [0] * U

    # ---------------------------------------------------------- registration
    def register_new(self, units=None):
        """Register clusters added since the last call (prefill or update) and
        grow capacity monotonically (engine.py:98-106)."""
        lay = self.layer
        units = range(lay.U) if units is None else units
        bc = self.block_cap
        for u in units:
            m0, m1 = self._registered[u], lay.units[u].m
            if self._registered[u] == 0 and m0 == 0:
                self.n_blocks[u] = math.ceil(lay.units[u].n_sink / bc) if lay.units[u].n_sink else 0
            if m1 > m0:
                sz = lay.cl_size[u, m0:m1].to(torch.int64)
                nb = (sz + bc - 1) // bc
                rows = self._rows(u)
                base = 0 if m0 == 0 else int(self.slot_off[rows[0], m0 - 1] + self.nblk[rows[0], m0 - 1])
                off = base + torch.cumsum(nb, 0) - nb
                for r in rows:
                    self.nblk[r, m0:m1] = nb.to(torch.int32)
                    self.slot_off[r, m0:m1] = off.to(torch.int32)
                self.n_blocks[u] += int(nb.sum())
                self._registered[u] = m1
            want = math.ceil(self.cfg.cache_fraction * self.n_blocks[u])
            if want > self.cap_host[u]:
                self.cap_host[u] = want
                for r in self._rows(u):
                    self.capacity[r] = want

    def _rows(self, u):
        G = self.layer.G
        return list(range(u * G, u * G + G)) if self.mode == "head" else [u]

    # ----------------------------------------------------------------- step
    def step(self, step_idx: int):
        lay = self.layer
        rc = lay.L.wk_cache_step(ctypes.byref(self._view), lay.rlist.data_ptr(), lay.nr.data_ptr(),
                                 lay.st_n.data_ptr(), lay.r_cap, lay.G, int(self.mode == "union"),
                                 step_idx, self.C, lay.status.data_ptr(),
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        _lib.check(rc, "wk_cache_step")

    # ---------------------------------------------------------------- views
    def stats(self, c: int = 0) -> dict:
        k = self.counters[c].tolist()
        acc = k[0] + k[1]
        return {"hits": k[0], "misses": k[1], "hit_ratio": k[0] / acc if acc else 0.0,
                "bytes_slow_to_fast": k[2], "bytes_fast_internal": k[3],
                "capacity_blocks": int(self.capacity[c]), "occupied_blocks": int(self.occupied[c])}

    def event_log(self, c: int = 0):
        if self.events is None:
            return []
        n = min(int(self.ev_n[c]), self.ev_cap)
        ev = self.events[c, :n].cpu().numpy()
        return [(EVENT_TYPES[int(t)], int(s), int(cl), int(a)) for t, s, cl, a in ev]

    def lru_order(self, c: int = 0):
        head = int(self.lru_ht[c, 0])
        nxt = self.next[c].cpu().numpy()
        out = []
        while head >= 0:
            out.append(head)
            head = int(nxt[head])
        return out


class HostBuffer:
    """Pinned, device-mapped host memory (wk_host_alloc) viewed as a CPU
    tensor; its ``data_ptr()`` is valid on the device (UVA).  Holds the
    offloaded cluster store (the reference's slow tier, store.py:48-105)."""

    def __init__(self, shape, dtype):
        L = _lib.lib()
        numel = int(np.prod(shape))
        nbytes = numel * torch.empty((), dtype=dtype).element_size()
        ptr = ctypes.c_void_p()
        _lib.check(L.wk_host_alloc(nbytes, ctypes.byref(ptr)), "wk_host_alloc")
        self._ptr = ptr.value
        self._L = L
        raw = (ctypes.c_uint8 * nbytes).from_address(self._ptr)
        self.tensor = torch.frombuffer(raw, dtype=torch.uint8).view(dtype).view(*shape)

    def __del__(self):
        try:
            if self._ptr:
                self._L.wk_host_free(ctypes.c_void_p(self._ptr))
                self._ptr = None
        except Exception:
            pass


class OffloadCache:
    """The wave buffer of the offload path: an HBM slot arena caching
    cluster blocks of the pinned host store, one cache per kv-head unit
    serving the union access stream of its GQA group (cache_v2.cu).  Lookup,
    replacement and the miss plan run on the device in one launch per step
    (wk_cache_offload_step); misses are fetched by the attention kernel with
    TMA from host memory and admitted misses are written through into their
    slots.  Accounting follows block_cache.py / store.py exactly."""

    def __init__(self, layer):
        cfg = layer.cfg
        U, G, d, dev = layer.U, layer.G, layer.d, layer.dev
        self.layer = layer
        self.cfg = cfg
        self.bt = block_capacity(cfg.block_size_bytes, d)
        m_cap = layer.m_cap
        self.list_cap = layer.s_cap // self.bt + m_cap + 4          # blocks of all clusters
        self.phys = max(1, math.ceil(cfg.cache_fraction * self.list_cap) + 2)  # arena slots
        self.lru_cap = self.phys + 1
        self.ids_cap = layer.r_cap * G
        i32, i64 = torch.int32, torch.int64
        z = lambda *s, dt=i32: torch.zeros(s, dtype=dt, device=dev)
        self.nblk = z(U, m_cap)
        self.slot_off = z(U, m_cap)
        self.slot_ids = z(U, self.list_cap)
        self.cached = z(U, m_cap, dt=torch.uint8)
        self.touched = z(U, m_cap)
        self.first = torch.full((U, m_cap), 0x7FFFFFFF, dtype=i32, device=dev)
        self.lru = z(U, self.lru_cap)
        self.lru_tmp = z(U, self.lru_cap)
        self.lru_n = z(U)
        self.freel = z(U, self.list_cap)
        self.free_n = z(U)
        self.next_slot = z(U)
        self.capacity = z(U, dt=i64)
        self.occupied = z(U, dt=i64)
        self.counters = z(U, 8, dt=i64)
        self.ids = z(U, self.ids_cap)
        self.n_ids = z(U)
        self.snapshot = z(U, self.ids_cap, dt=torch.uint8)
        self.scratch = z(U, self.lru_cap + 1 + 2 * self.ids_cap)
        self.arena_k = torch.zeros((U, self.phys * self.bt, d), dtype=layer.store_dtype, device=dev)
        self.arena_v = torch.zeros_like(self.arena_k)
        self.n_blocks = [0] * U
        self.cap_host = [0] * U
        self._registered = [0] * U
        self.step_idx = 0
        self._view = _lib.Cache2ViewC(
            *(t.data_ptr() for t in (self.nblk, self.slot_off, self.slot_ids, self.cached, self.touched,
                                     self.first, self.lru, self.lru_tmp, self.lru_n, self.freel, self.free_n,
                                     self.next_slot, self.capacity, self.occupied, self.counters, self.ids,
                                     self.n_ids, self.snapshot, self.scratch, layer.m_dev)),
            m_cap, self.list_cap, self.lru_cap, self.ids_cap, cfg.block_size_bytes, 2 * d * 4, self.bt, 0)

    def register_new(self, units=None):
        """Register clusters added since the last call; capacity grows
        monotonically to ceil(cache_fraction * n_blocks) (engine.py:98-106)."""
        lay = self.layer
        units = range(lay.U) if units is None else units
        bt = self.bt
        for u in units:
            m0, m1 = self._registered[u], lay.units[u].m
            if m0 == 0 and self.n_blocks[u] == 0 and lay.units[u].n_sink:
                self.n_blocks[u] = math.ceil(lay.units[u].n_sink / bt)  # sink pseudo-cluster
            if m1 > m0:
                sz = lay.cl_size[u, m0:m1].to(torch.int64)
                nb = (sz + bt - 1) // bt
                base = 0 if m0 == 0 else int(self.slot_off[u, m0 - 1] + self.nblk[u, m0 - 1])
                self.nblk[u, m0:m1] = nb.to(torch.int32)
                self.slot_off[u, m0:m1] = (base + torch.cumsum(nb, 0) - nb).to(torch.int32)
                self.n_blocks[u] += int(nb.sum())
                self._registered[u] = m1
            want = math.ceil(self.cfg.cache_fraction * self.n_blocks[u])
            if want > self.phys:
                raise ConfigError("offload cache capacity exceeds the slot arena")
            if want > self.cap_host[u]:
                self.cap_host[u] = want
                self.capacity[u] = want

    def step(self, sv):
        lay = self.layer
        rc = lay.L.wk_cache_offload_step(ctypes.byref(self._view), ctypes.byref(lay._ixv), ctypes.byref(lay._stv),
                                         ctypes.byref(sv), lay.G, self.step_idx, lay.U,
                                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        _lib.check(rc, "wk_cache_offload_step")
        self.step_idx += 1

    def stats(self, u: int = 0) -> dict:
        k = self.counters[u].tolist()
        acc = k[0] + k[1]
        return {"hits": k[0], "misses": k[1], "hit_ratio": k[0] / acc if acc else 0.0,
                "bytes_slow_to_fast": k[2], "bytes_fast_internal": k[3], "store_bytes_read": k[4],
                "evictions": k[5], "admissions": k[6], "rejections": k[7],
                "capacity_blocks": int(self.capacity[u]), "occupied_blocks": int(self.occupied[u])}

    def totals(self) -> dict:
        k = self.counters.sum(0).tolist()
        acc = k[0] + k[1]
        return {"hits": k[0], "misses": k[1], "hit_ratio": k[0] / acc if acc else 0.0,
                "bytes_slow_to_fast": k[2], "evictions": k[5], "admissions": k[6], "rejections": k[7]}
