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

from dataclasses import dataclass, field

from . import _lib
from .errors import ConfigError, IntegrityError
from .store import block_capacity

EVENT_TYPES = {0: "access", 1: "evict", 2: "admit", 3: "reject"}


@dataclass
class ClusterDescriptor:
    """Mapping-table entry (block_cache.py:22-31)."""
    cluster_id: int
    slow_block_ids: list[int]
    fast_slot_ids: list[int] | None = None
    last_access_step: int = -1

    @property
    def cached(self) -> bool:
        return self.fast_slot_ids is not None


@dataclass
class ExecutionBuffer:
    """Per-step staging area: steady tokens, then retrieval clusters in rank
    order; spans = (source, cluster_id, start, end) (block_cache.py:34-42)."""
    keys: np.ndarray
    values: np.ndarray
    token_ids: np.ndarray
    spans: list[tuple] = field(default_factory=list)


def event_dict(t, step, cl, aux):
    """A device event record (type, step, cluster, aux) as the reference's
    event_log dict (block_cache.py:92-95, 188-207)."""
    name = EVENT_TYPES[int(t)]
    e = {"type": name, "step": int(step), "cluster": int(cl)}
    if name == "admit":
        e["blocks"] = int(aux)
    return e


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
        """Raw device event records (type, step, cluster, aux)."""
        if self.events is None:
            return []
        n = min(int(self.ev_n[c]), self.ev_cap)
        ev = self.events[c, :n].cpu().numpy()
        return [(EVENT_TYPES[int(t)], int(s), int(cl), int(a)) for t, s, cl, a in ev]

    def access_stream(self, c: int = 0):
        """This step's access stream (rank order, distinct) and its residency
        snapshot -- the clusters / cached lists of the access event."""
        n = int(self.n_ids[c])
        return self.ids[c, :n].tolist(), [bool(x) for x in self.snapshot[c, :n].tolist()]

    def descriptors(self, c: int, m: int, first_block: int):
        """ClusterDescriptor of clusters 0..m-1 of cache unit c; slow block
        ids are numbered as the reference's store packs them (the sink
        pseudo-cluster's ``first_block`` blocks first, then clusters in id
        order, store.py:69-90)."""
        nb = self.nblk[c, :m].tolist()
        so = self.slot_off[c, :m].tolist()
        ca = self.cached[c, :m].tolist()
        la = self.last_access[c, :m].tolist()
        sl = self.slot_ids[c].tolist() if any(ca) else []
        return {i: ClusterDescriptor(i, list(range(first_block + so[i], first_block + so[i] + nb[i])),
                                     sl[so[i]:so[i] + nb[i]] if ca[i] else None, int(la[i]))
                for i in range(m)}

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
            m_cap, self.list_cap, self.lru_cap, self.ids_cap, cfg.block_size_bytes, 2 * d * 4, self.bt,
            layer.piece_rows)

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


class BlockCache:
    """tierkv's BlockCache (block_cache.py:52-225) as separately callable
    phases, its state machine on the device: ``lookup`` / ``assemble`` /
    ``commit_update`` launch wk_cache_phase on one cache unit (residency,
    LRU list, free-slot heap, byte counters and the event records live in
    HBM); block payloads of admitted clusters live in an HBM slot arena.
    Cluster ids may be any ints (mapped to dense device ids on the host)."""

    def __init__(self, store, capacity_blocks: int):
        if not torch.cuda.is_available():
            raise RuntimeError("BlockCache runs on a CUDA device (no CPU fallback)")
        self.store = store
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self._dense: dict[int, int] = {}
        self._cid: list[int] = []
        self._slow: list[list[int]] = []
        self._staged: dict[int, list] = {}
        self.event_log: list[dict] = []
        self._m_cap = self._slot_cap = self._heap_cap = 0
        self._arena_slots = 0
        self._t = {}
        self._cap = 0
        self._grow(64, 64, 64)
        self.capacity_blocks = capacity_blocks

    # ---------------------------------------------------------------- state
    def _grow(self, m_cap, slot_cap, heap_cap):
        m_cap, slot_cap, heap_cap = max(m_cap, self._m_cap), max(slot_cap, self._slot_cap), max(heap_cap, self._heap_cap)
        if (m_cap, slot_cap, heap_cap) == (self._m_cap, self._slot_cap, self._heap_cap):
            return
        dev, i32, i64 = self.dev, torch.int32, torch.int64
        spec = {"nblk": (m_cap, i32, 0), "slot_off": (m_cap, i32, 0), "slot_ids": (slot_cap, i32, 0),
                "cached": (m_cap, torch.uint8, 0), "prev": (m_cap, i32, -1), "next": (m_cap, i32, -1),
                "touched": (m_cap, i32, 0), "last_access": (m_cap, i64, -1), "heap": (heap_cap, i32, 0)}
        old = self._t
        t = {}
        for name, (n, dt, fill) in spec.items():
            a = torch.full((1, n), fill, dtype=dt, device=dev)
            if name in old:
                a[:, :old[name].shape[1]] = old[name]
            t[name] = a
        for name, shape, dt, fill in (("lru_ht", (1, 2), i32, -1), ("heap_n", (1,), i32, 0),
                                      ("next_slot", (1,), i32, 0), ("capacity", (1,), i64, 0),
                                      ("occupied", (1,), i64, 0), ("counters", (1, 8), i64, 0),
                                      ("n_ids", (1,), i32, 0), ("ev_n", (1,), i64, 0), ("m_live", (1,), i32, 0)):
            t[name] = old[name] if name in old else torch.full(shape, fill, dtype=dt, device=dev)
        self._ev_cap = 2 * m_cap + 16
        t["events"] = torch.zeros((1, self._ev_cap, 4), dtype=i32, device=dev)
        t["ids"] = torch.zeros((1, 1), dtype=i32, device=dev)
        t["snapshot"] = torch.zeros((1, 1), dtype=torch.uint8, device=dev)
        self._t = t
        self._m_cap, self._slot_cap, self._heap_cap = m_cap, slot_cap, heap_cap
        self._view = _lib.CacheViewC(
            *(t[n].data_ptr() for n in ("nblk", "slot_off", "slot_ids", "cached", "prev", "next", "touched",
                                        "last_access", "lru_ht", "heap", "heap_n", "next_slot", "capacity",
                                        "occupied", "counters", "ids", "n_ids", "snapshot", "events", "ev_n",
                                        "m_live")),
            m_cap, slot_cap, heap_cap, 1, self._ev_cap, self.store.block_size_bytes,
            2 * self.store.d * 4)
        self._status = torch.zeros(1, dtype=torch.int32, device=dev)

    def _arena(self, slots):
        """HBM slot arena: one block payload (keys, values, token ids, rows) per slot."""
        if slots <= self._arena_slots:
            return
        n = max(slots, 2 * self._arena_slots, 16)
        bc, d = self.store.block_capacity, self.store.d
        new = {"k": torch.zeros((n, bc, d), dtype=torch.float32, device=self.dev),
               "v": torch.zeros((n, bc, d), dtype=torch.float32, device=self.dev),
               "tok": torch.zeros((n, bc), dtype=torch.int64, device=self.dev),
               "rows": torch.zeros(n, dtype=torch.int32, device=self.dev)}
        if self._arena_slots:
            for key in new:
                new[key][: self._arena_slots] = self._slots[key]
        self._slots = new
        self._arena_slots = n

    @property
    def capacity_blocks(self) -> int:
        return self._cap

    @capacity_blocks.setter
    def capacity_blocks(self, cap: int):
        cap = int(cap)
        self._cap = cap
        self._grow(self._m_cap, self._slot_cap, max(self._heap_cap, cap + 1))
        self._t["capacity"].fill_(cap)
        self._arena(cap + 1)

    def register_cluster(self, cluster_id: int, slow_block_ids: list[int]):
        if cluster_id in self._dense:
            raise IntegrityError(f"cluster {cluster_id} already registered")
        i = len(self._cid)
        base = sum(len(b) for b in self._slow)
        nb = len(slow_block_ids)
        self._grow(max(self._m_cap, 2 * (i + 1)) if i + 1 > self._m_cap else self._m_cap,
                   max(self._slot_cap, 2 * (base + nb)) if base + nb > self._slot_cap else self._slot_cap,
                   self._heap_cap)
        self._t["nblk"][0, i] = nb
        self._t["slot_off"][0, i] = base
        self._t["m_live"][0] = i + 1
        self._dense[cluster_id] = i
        self._cid.append(cluster_id)
        self._slow.append(list(slow_block_ids))

    def _dense_ids(self, cluster_ids):
        out = []
        for cid in cluster_ids:
            if cid not in self._dense:
                raise IntegrityError(f"unknown cluster_id {cid}")
            out.append(self._dense[cid])
        return torch.tensor(out if out else [0], dtype=torch.int32).to(self.dev), len(out)

    def _phase(self, ids_t, n, snap, n_steady, step, phase, snap_out=None, n_out=None):
        st = torch.cuda.current_stream().cuda_stream
        rc = _lib.lib().wk_cache_phase(ctypes.byref(self._view), ids_t.data_ptr(),
                                       None if snap is None else snap.data_ptr(), n, n_steady, step, phase,
                                       None if snap_out is None else snap_out.data_ptr(),
                                       None if n_out is None else n_out.data_ptr(), self._status.data_ptr(),
                                       ctypes.c_void_p(st))
        _lib.check(rc, "wk_cache_phase")

    def _check(self, what):
        code = int(self._status.item())
        if code:
            self._status.zero_()
            if code == 3:
                raise IntegrityError("block cache exceeded its capacity")
            _lib.raise_status(code, what)

    def _drain_events(self):
        n = min(int(self._t["ev_n"][0]), self._ev_cap)
        ev = self._t["events"][0, :n].cpu().numpy()
        self._t["ev_n"].zero_()
        return [event_dict(t, s_, self._cid[c] if t != 0 else c, a) for t, s_, c, a in ev]

    # ------------------------------------------------------------ read path
    def lookup(self, cluster_ids, step: int) -> dict[int, bool]:
        """Residency snapshot as of the last commit, one access per distinct
        cluster, LRU untouched (block_cache.py:79-96)."""
        ids_t, n = self._dense_ids(list(cluster_ids))
        snap = torch.zeros(max(1, n), dtype=torch.uint8, device=self.dev)
        n_out = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._phase(ids_t, n, None, 0, step, 1, snap, n_out)
        self._check("lookup")
        k = int(n_out.item())
        seen = [self._cid[i] for i in ids_t[:k].tolist()] if k else []
        cached = [bool(x) for x in snap[:k].tolist()] if k else []
        self._drain_events()
        self.event_log.append({"type": "access", "step": step, "clusters": seen, "cached": cached})
        return dict(zip(seen, cached))

    def _slot_lists(self):
        nb = self._t["nblk"][0].tolist()
        so = self._t["slot_off"][0].tolist()
        sl = self._t["slot_ids"][0].tolist()
        return nb, so, sl

    def assemble(self, retrieval_cluster_ids, snapshot, steady_keys, steady_values,
                 steady_token_ids) -> ExecutionBuffer:
        """Steady tokens then retrieval clusters in rank order; hits come from
        the HBM slot arena, misses are read from the slow tier and staged for
        admission (block_cache.py:98-143)."""
        d = self.store.d
        ids = list(retrieval_cluster_ids)
        ids_t, n = self._dense_ids(ids)
        snap = torch.tensor([int(bool(snapshot[c])) for c in ids] or [0], dtype=torch.uint8).to(self.dev)
        n_steady = len(steady_token_ids)
        self._phase(ids_t, n, snap, n_steady, 0, 2)
        ks, vs, ts, spans = [], [], [], []
        pos = 0
        if n_steady:
            ks.append(np.asarray(steady_keys, np.float32).reshape(n_steady, d))
            vs.append(np.asarray(steady_values, np.float32).reshape(n_steady, d))
            ts.append(np.asarray(steady_token_ids, np.int64))
            spans.append(("steady", None, 0, n_steady))
            pos = n_steady
        nb = so = sl = None
        for cid in ids:
            di = self._dense[cid]
            if snapshot[cid]:
                if sl is None:
                    nb, so, sl = self._slot_lists()
                slots = torch.tensor(sl[so[di]:so[di] + nb[di]], dtype=torch.long, device=self.dev)
                rows = self._slots["rows"][slots].tolist()
                bk = [self._slots["k"][s_, :r] for s_, r in zip(slots.tolist(), rows)]
                bv = [self._slots["v"][s_, :r] for s_, r in zip(slots.tolist(), rows)]
                bt = [self._slots["tok"][s_, :r] for s_, r in zip(slots.tolist(), rows)]
                blocks = [(a.cpu().numpy(), b.cpu().numpy(), c.cpu().numpy()) for a, b, c in zip(bk, bv, bt)]
                src = "cache_hit"
            else:
                self.store.read_blocks(self._slow[di])  # whole-block read accounting (store.py:92-101)
                blocks = [tuple(np.array(x) for x in self.store.block_rows(b)) for b in self._slow[di]]
                self._staged[cid] = blocks
                src = "slow_miss"
            cnt = 0
            for bk_, bv_, bt_ in blocks:
                ks.append(bk_); vs.append(bv_); ts.append(bt_)
                cnt += len(bt_)
            spans.append((src, cid, pos, pos + cnt))
            pos += cnt
        self._check("assemble")
        if ks:
            return ExecutionBuffer(np.concatenate(ks), np.concatenate(vs), np.concatenate(ts), spans)
        return ExecutionBuffer(np.empty((0, d), np.float32), np.empty((0, d), np.float32),
                               np.empty(0, np.int64), spans)

    # ---------------------------------------------------------- update path
    def commit_update(self, retrieval_cluster_ids, snapshot, step: int) -> list[dict]:
        """Hits to MRU, misses admitted all-or-nothing in rank order evicting
        untouched LRU clusters, oversize / unfittable ones rejected
        (block_cache.py:163-213); admitted payloads copied into their slots."""
        ids = list(retrieval_cluster_ids)
        ids_t, n = self._dense_ids(ids)
        snap = torch.tensor([int(bool(snapshot[c])) for c in ids] or [0], dtype=torch.uint8).to(self.dev)
        self._phase(ids_t, n, snap, 0, step, 4)
        log = self._drain_events()
        self._check("commit_update")
        admitted = [e["cluster"] for e in log if e["type"] == "admit"]
        if admitted:
            nb, so, sl = self._slot_lists()
            for cid in admitted:
                di = self._dense[cid]
                blocks = self._staged.pop(cid)
                for s_, (bk, bv, bt) in zip(sl[so[di]:so[di] + nb[di]], blocks):
                    r = len(bt)
                    self._slots["k"][s_, :r] = torch.from_numpy(np.ascontiguousarray(bk, np.float32))
                    self._slots["v"][s_, :r] = torch.from_numpy(np.ascontiguousarray(bv, np.float32))
                    self._slots["tok"][s_, :r] = torch.from_numpy(np.asarray(bt, np.int64))
                    self._slots["rows"][s_] = r
        self._staged.clear()
        self.event_log.extend(log)
        return log

    # ---------------------------------------------------------------- views
    def _counter(self, i):
        return int(self._t["counters"][0, i])

    hits = property(lambda self: self._counter(0))
    misses = property(lambda self: self._counter(1))
    bytes_slow_to_fast = property(lambda self: self._counter(2))
    bytes_fast_internal = property(lambda self: self._counter(3))

    @property
    def occupied_blocks(self) -> int:
        return int(self._t["occupied"][0])

    @property
    def lru(self) -> list[int]:
        """Cached cluster ids, least recently used first."""
        head = int(self._t["lru_ht"][0, 0])
        nxt = self._t["next"][0].tolist()
        out = []
        while head >= 0:
            out.append(self._cid[head])
            head = nxt[head]
        return out

    @property
    def mapping(self) -> dict[int, ClusterDescriptor]:
        m = len(self._cid)
        nb, so, sl = self._slot_lists()
        ca = self._t["cached"][0, :m].tolist()
        la = self._t["last_access"][0, :m].tolist()
        return {self._cid[i]: ClusterDescriptor(self._cid[i], list(self._slow[i]),
                                                sl[so[i]:so[i] + nb[i]] if ca[i] else None, int(la[i]))
                for i in range(m)}

    @property
    def slots(self) -> dict[int, tuple]:
        out = {}
        for desc in self.mapping.values():
            for s_ in desc.fast_slot_ids or []:
                r = int(self._slots["rows"][s_])
                out[s_] = (self._slots["k"][s_, :r].cpu().numpy(), self._slots["v"][s_, :r].cpu().numpy(),
                           self._slots["tok"][s_, :r].cpu().numpy())
        return out

    def stats(self) -> dict:
        k = self._t["counters"][0].tolist()
        acc = k[0] + k[1]
        return {"hits": k[0], "misses": k[1], "hit_ratio": k[0] / acc if acc else 0.0,
                "bytes_slow_to_fast": k[2], "bytes_fast_internal": k[3],
                "capacity_blocks": self._cap, "occupied_blocks": self.occupied_blocks}
