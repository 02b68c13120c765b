"""Batched B200 wave-index state for one attention layer.

A ``WaveLayer`` holds U (request, kv-head) units, each serving G query heads
(GQA).  Everything lives in HBM; the host keeps only integer bookkeeping
(lengths, cluster counts, update schedule) and launches the sm_100a kernels of
libwavekv.so through the C ABI (include/wavekv.h):

  prefill  -> wk_kmeans_segments      (index.py:153-166 segmented build)
  decode   -> wk_append_tokens        (engine.py:178-182)
              wk_score_topk           (index.py:61-93 rank + plan_zones)
              wk_tripartite_attn      (attention.py:67-148, engine.py:150-172)
              [every update_segment tokens] wk_kmeans_segments
                                      (index.py:168-186 decode-time update)

Per-unit semantics are exactly ``tierkv.HeadEngine`` (engine.py:40-237) with
the index shared by the G heads of a kv head (the reference seeds do not
depend on the head, index.py:162, so each head's reference engine builds the
identical index).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import EngineConfig, round_half_up
from .errors import ConfigError

_SEED_CACHE: dict = {}


def pcg64_words(rng_seed: int, kind: int, idx: int):
    """numpy PCG64 state of default_rng(SeedSequence([rng_seed, kind, idx]))
    (index.py:162/181 -> clustering.py:81).  Host-side seed derivation; the
    stream itself is generated on the device."""
    key = (int(rng_seed), int(kind), int(idx))
    w = _SEED_CACHE.get(key)
    if w is None:
        st = np.random.PCG64(np.random.SeedSequence(list(key))).state["state"]
        s, i = int(st["state"]), int(st["inc"])
        m = (1 << 64) - 1
        w = (s >> 64, s & m, i >> 64, i & m)
        _SEED_CACHE[key] = w
    return w


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


@dataclass
class UnitState:
    """Host mirror of one unit's integer bookkeeping (engine.py:44-57)."""
    total: int = 0            # tokens seen (HeadEngine.total_tokens)
    n_sink: int = 0
    buffer_start: int = 0     # token id of the oldest buffered token
    m: int = 0                # clusters
    store_fill: int = 0       # store rows used
    update_round: int = 0     # ClusterIndex._update_round
    n_steady: int = 0         # sinks + buffer rows


def swizzle_rows(x: torch.Tensor, row0: int = 0) -> torch.Tensor:
    """The fast path's bf16 row layout (csrc/common.cuh swz_col): 16-byte piece
    c of row r (8 elements) sits at piece c ^ (r & 7), r = row0 + the row's index
    in x.  An involution: the same call un-swizzles."""
    n, d = x.shape[-2], x.shape[-1]
    pcs = d // 8
    key = (torch.arange(row0, row0 + n, device=x.device) & 7)[:, None]
    src = torch.arange(pcs, device=x.device)[None, :] ^ key
    xr = x.reshape(*x.shape[:-1], pcs, 8)
    idx = src[..., None].expand(*xr.shape)
    return torch.gather(xr, -2, idx).reshape(x.shape)


class WaveLayer:
    """U units x G heads of one layer; all tensors on ``device``."""

    def __init__(self, cfg: EngineConfig, U: int, G: int, d: int, *, max_prefill: int,
                 max_decode: int = 1024, store_dtype=torch.bfloat16, device="cuda",
                 blas_threads: int = 1, splits: int | None = None, keep_vs64: bool = False,
                 with_elist: bool = False, offload: bool = False,
                 split: int = 1):
        self.cfg = cfg.validate()
        ic = cfg.index
        if d <= 0 or d % 4 or d > 256:
            raise ConfigError(f"head dim {d} unsupported (need d % 4 == 0, d <= 256)")
        if not 1 <= G <= 8:
            raise ConfigError(f"G={G} query heads per kv head unsupported (1..8)")
        if store_dtype not in (torch.bfloat16, torch.float32):
            raise ConfigError("store_dtype must be bfloat16 or float32")
        self.U, self.G, self.d = U, G, d
        self.dev = torch.device(device)
        if self.dev.type != "cuda":
            raise ConfigError("WaveLayer runs on a CUDA device only (no CPU fallback)")
        self.store_dtype = store_dtype
        self.store_bf16 = int(store_dtype == torch.bfloat16)
        self.blas_threads = int(blas_threads)
        self.L = _lib.lib()
        # ---- capacities ----
        n_idx = max(0, max_prefill - min(ic.sink_tokens, max_prefill) - ic.local_window)
        n_upd = max_decode // ic.update_segment + 1
        k_upd = math.ceil(ic.update_segment / ic.centroid_ratio)
        m_pref = sum(math.ceil(min(ic.segment_size, n_idx - s) / ic.centroid_ratio)
                     for s in range(0, n_idx, ic.segment_size))
        # multiple of 128: float4 scans, zone bitmaps (4 words / 128 clusters)
        self.m_cap = max(128, -(-(m_pref + n_upd * k_upd) // 128) * 128)
        self.s_cap = max(1, n_idx + n_upd * ic.update_segment)
        self.t_cap = ic.sink_tokens + ic.update_segment + ic.local_window + max(0, ic.local_window) + 8
        self.t_cap = max(self.t_cap, min(max_prefill, ic.sink_tokens + ic.local_window) + 8)
        self.r_cap = max(1, min(self.m_cap, round_half_up(ic.retrieval_fraction * self.m_cap) + 2))
        self.e_cap = max(1, min(self.m_cap, round_half_up(ic.estimation_fraction * self.m_cap) + 2))
        # fast path (score_v5 / select_v6 / attend_v4): d in {64, 128}
        self.fast = d in (64, 128)
        # bf16 rows of the fast path are stored swizzled (csrc/common.cuh swz_col)
        self.swizzled = self.fast and store_dtype == torch.bfloat16
        hs = 4 if G <= 4 else 8
        # retrieval piece rows = the attention chunk rows: attend_v5 (bf16 stores,
        # tensor cores) 16; attend_v4 (fp32 stores) 16 for G <= 4, 8 for G <= 8
        self.piece_rows = 16 if (hs == 4 or store_dtype == torch.bfloat16) else 8
        if self.fast:
            sms = torch.cuda.get_device_properties(self.dev).multi_processor_count
            self.S = splits or max(1, min(sms, 4 * U))  # persistent attention grid: 1 CTA / SM
            self.attn_warps = 12  # upper bound of the attention kernels' warps per CTA (partial slots)
        else:
            self.S = splits or max(1, min(64, -(-2048 // U)))
        # the C32 scan accumulates in fp64 (the estimation logits need ~fp32 accuracy)
        self.score_mode = 1
        dev, f32, i32 = self.dev, torch.float32, torch.int32
        # ---- index arrays ----
        # offload (config 4): the cluster store is pinned host memory (the
        # reference's slow tier); an HBM slot arena caches its blocks
        self.offload = bool(offload)
        if self.offload:
            if not self.fast:
                raise ConfigError("offload needs the fast path (d in {64, 128})")
            from .block_cache import HostBuffer
            self._host_k = HostBuffer((U, self.s_cap, d), store_dtype)
            self._host_v = HostBuffer((U, self.s_cap, d), store_dtype)
            self.store_k, self.store_v = self._host_k.tensor, self._host_v.tensor
        else:
            self.store_k = torch.zeros((U, self.s_cap, d), dtype=store_dtype, device=dev)
            self.store_v = torch.zeros((U, self.s_cap, d), dtype=store_dtype, device=dev)
        self.store_tok = torch.full((U, self.s_cap), -1, dtype=i32, device=dev)
        self.cl_off = torch.zeros((U, self.m_cap), dtype=i32, device=dev)
        self.cl_size = torch.zeros((U, self.m_cap), dtype=i32, device=dev)
        self.C64 = torch.zeros((U, self.m_cap, d), dtype=torch.float64, device=dev)
        self.C32 = torch.zeros((U, self.m_cap, d), dtype=f32, device=dev)
        self.Cnorm = torch.zeros((U, self.m_cap), dtype=f32, device=dev)
        self.VS32 = torch.zeros((U, self.m_cap, d), dtype=f32, device=dev)
        self.VS64 = (torch.zeros((U, self.m_cap, d), dtype=torch.float64, device=dev)
                     if keep_vs64 else None)
        self.Cmax = torch.zeros(U, dtype=f32, device=dev)
        # ---- steady zone ----
        self.st_k = torch.zeros((U, self.t_cap, d), dtype=store_dtype, device=dev)
        self.st_v = torch.zeros((U, self.t_cap, d), dtype=store_dtype, device=dev)
        self.st_tok = torch.full((U, self.t_cap), -1, dtype=i32, device=dev)
        self.st_n = torch.zeros(U, dtype=i32, device=dev)
        self.next_tok = torch.zeros(U, dtype=i32, device=dev)
        # ---- step buffers ----
        self.m_dev = torch.zeros(U, dtype=i32, device=dev)
        self.scores = torch.zeros((U, G, self.m_cap), dtype=f32, device=dev)
        self.rlist = torch.zeros((U, G, self.r_cap), dtype=i32, device=dev)
        self.elist = torch.zeros((U, G, self.e_cap), dtype=i32, device=dev) if with_elist else None
        self.nr = torch.zeros(U, dtype=i32, device=dev)
        self.ne = torch.zeros(U, dtype=i32, device=dev)
        self.ru_cap = min(self.m_cap, G * self.r_cap)
        # multiple of 32: attend_v6 copies estimation logits / sizes a chunk (<= 32 rows) at a time
        self.eu_cap = -(-min(self.m_cap, G * self.e_cap) // 32) * 32
        self.ru_ids = torch.zeros((U, self.ru_cap), dtype=i32, device=dev)
        self.ru_mask = torch.zeros((U, self.ru_cap), dtype=torch.uint8, device=dev)
        self.eu_ids = torch.zeros((U, self.eu_cap), dtype=i32, device=dev)
        self.eu_mask = torch.zeros((U, self.eu_cap), dtype=torch.uint8, device=dev)
        self.cnt = torch.zeros((U, 4), dtype=i32, device=dev)
        if self.fast:
            self.zmask = self.ru_pre = self.rtok_mask = None
            # attend_v5 row mode (bf16 store in HBM): every retrieved token's
            # store row | head mask << 24, written by the zone planning
            self.rows_mode = store_dtype == torch.bfloat16 and not offload
            self.rt_cap = self.s_cap if self.rows_mode else 0
            if self.rows_mode and self.s_cap >= (1 << 24):
                raise ConfigError("row mode packs store rows in 24 bits")
            self.rtok_row = (torch.zeros((U, self.rt_cap), dtype=i32, device=dev) if self.rows_mode else None)
            self.w_cap = self.m_cap // 32
            self.rbits = torch.zeros((U, G, self.w_cap), dtype=i32, device=dev)
            self.ebits = torch.zeros((U, G, self.w_cap), dtype=i32, device=dev)
            if self.offload:  # hits may fragment over arena slots
                self.pc_cap = min(self.s_cap, 32 * self.ru_cap) + self.ru_cap + 1
            else:
                self.pc_cap = self.s_cap // self.piece_rows + self.ru_cap + 1
            self.pieces = torch.zeros((U, self.pc_cap, 4 if self.offload else 2), dtype=i32, device=dev)
            self.woff = torch.zeros(U + 1, dtype=i32, device=dev)
        else:
            self.zmask = torch.zeros((U, self.m_cap), dtype=i32, device=dev)
            self.ru_pre = torch.zeros((U, self.ru_cap + 1), dtype=i32, device=dev)
            self.rows_mode = False
            self.rt_cap = 0
            self.rtok_row = self.rtok_mask = None
            self.w_cap = self.pc_cap = 0
            self.rbits = self.ebits = self.pieces = self.woff = None
        self.sel_done = torch.zeros(U, dtype=i32, device=dev)
        self.eu_x = torch.zeros((U, self.eu_cap, G), dtype=f32, device=dev)
        self.eu_sz = torch.zeros((U, self.eu_cap), dtype=f32, device=dev)
        self.tail = torch.zeros((U, G, 4), dtype=f32, device=dev)
        # partial records: attend_v4 keys (CTA warp + unit), attend_v6 keys
        # consumers x (CTA + unit); attn_warps x (S + U) bounds both
        n_part = self.attn_warps * (self.S + U) if self.fast else U * self.S
        self.part = torch.zeros((n_part, 3, G, (4 + d) if self.fast else (2 + d)), dtype=f32, device=dev)
        self.out = torch.zeros((U, G, d), dtype=f32, device=dev)
        self.logden = torch.zeros((U, G), dtype=f32, device=dev)
        self.cov = torch.zeros((U, G), dtype=f32, device=dev)
        self.status = torch.zeros(1, dtype=i32, device=dev)
        # tie-safe exact selection: fp64 exact-score scratch + fallback counter
        self.xscr = torch.zeros((U, G, self.m_cap), dtype=torch.float64, device=dev)
        self.xcount = torch.zeros(1, dtype=i32, device=dev)
        self.q64 = None  # optional [U, G, d] fp64 queries for the exact re-scoring
        self.n_store_dev = torch.zeros(U, dtype=i32, device=dev)
        self.units = [UnitState() for _ in range(U)]
        self._q = None
        self._zp = _lib.ZoneParamsC(G, d, self.blas_threads, ic.retrieval_fraction,
                                    ic.estimation_fraction, int(ic.tail_mode == "denominator_only"),
                                    int(cfg.denominator_mode == "eq2"), self.score_mode,
                                    self.piece_rows if self.fast else 0)
        self._ixv = _lib.IndexViewC(
            _ptr(self.store_k), _ptr(self.store_v), _ptr(self.store_tok), _ptr(self.cl_off),
            _ptr(self.cl_size), _ptr(self.C64), _ptr(self.C32), _ptr(self.Cnorm), _ptr(self.VS32),
            _ptr(self.VS64), self.s_cap, self.m_cap, _ptr(self.Cmax))
        self._stv = _lib.SteadyViewC(_ptr(self.st_k), _ptr(self.st_v), _ptr(self.st_tok),
                                     _ptr(self.st_n), _ptr(self.next_tok), self.t_cap)
        self.cache = None
        if self.offload:
            from .block_cache import OffloadCache
            self.cache = OffloadCache(self)
        # split > 1: the units are processed in groups on separate streams so the
        # latency-bound zone planning of one group overlaps the HBM-bound
        # centroid scan of the next (in-HBM fast path only)
        self.split = int(split) if (self.fast and not self.offload and U >= 2 * int(split)) else 1
        self._groups = []
        if self.split > 1:
            for gi in range(self.split):
                u0, u1 = U * gi // self.split, U * (gi + 1) // self.split
                n = u1 - u0
                part = torch.zeros((self.attn_warps * (self.S + n), 3, G, 4 + d), dtype=f32, device=dev)
                woff = torch.zeros(n + 1, dtype=i32, device=dev)
                self._groups.append(dict(u0=u0, n=n, part=part, woff=woff,
                                         ixv=self._index_view(u0, u1), stv=self._steady_view(u0, u1)))
            self._streams = [torch.cuda.Stream(device=dev) for _ in range(self.split)]
        self.prefilled = False

    # ------------------------------------------------------------ row layout
    def _to_rows(self, x: torch.Tensor, row0: int) -> torch.Tensor:
        """fp32 rows -> the steady/store row format (bf16 fast path: swizzled)."""
        y = x.to(self.store_dtype)
        return swizzle_rows(y, row0) if self.swizzled else y

    def _from_rows(self, x: torch.Tensor, row0: int) -> torch.Tensor:
        """Stored rows (starting at row index row0 of their array) -> fp32."""
        return (swizzle_rows(x, row0) if self.swizzled else x).float()

    # ------------------------------------------------------------------ views
    def _index_view(self, u0, u1):
        sl = lambda t: None if t is None else t[u0:u1]
        return _lib.IndexViewC(
            _ptr(sl(self.store_k)), _ptr(sl(self.store_v)), _ptr(sl(self.store_tok)), _ptr(sl(self.cl_off)),
            _ptr(sl(self.cl_size)), _ptr(sl(self.C64)), _ptr(sl(self.C32)), _ptr(sl(self.Cnorm)),
            _ptr(sl(self.VS32)), _ptr(sl(self.VS64)), self.s_cap, self.m_cap, _ptr(sl(self.Cmax)))

    def _steady_view(self, u0, u1):
        return _lib.SteadyViewC(_ptr(self.st_k[u0:u1]), _ptr(self.st_v[u0:u1]), _ptr(self.st_tok[u0:u1]),
                                _ptr(self.st_n[u0:u1]), _ptr(self.next_tok[u0:u1]), self.t_cap)

    def _group_step_view(self, grp, q):
        u0, u1 = grp["u0"], grp["u0"] + grp["n"]
        sl = lambda t: None if t is None else t[u0:u1]
        return _lib.StepViewC(
            _ptr(q[u0:u1]), _ptr(sl(self.m_dev)), _ptr(sl(self.scores)), _ptr(sl(self.rlist)), _ptr(sl(self.elist)),
            _ptr(sl(self.nr)), _ptr(sl(self.ne)), None, _ptr(sl(self.ru_ids)), _ptr(sl(self.ru_mask)),
            None, _ptr(sl(self.eu_ids)), _ptr(sl(self.eu_mask)), _ptr(sl(self.cnt)),
            _ptr(sl(self.tail)), _ptr(grp["part"]), _ptr(sl(self.out)), _ptr(sl(self.logden)), _ptr(sl(self.cov)),
            _ptr(self.status), self.r_cap, self.e_cap, self.ru_cap, self.eu_cap,
            _ptr(sl(self.rtok_row)), None, _ptr(sl(self.sel_done)), self.rt_cap, 0,
            _ptr(sl(self.eu_x)), _ptr(sl(self.eu_sz)), _ptr(sl(self.rbits)), _ptr(sl(self.ebits)), _ptr(sl(self.pieces)),
            _ptr(grp["woff"]), self.w_cap, self.pc_cap, None, None, None, None, 0, 0, 0, 2,
            None, _ptr(sl(self.xscr)), _ptr(self.xcount))

    def _launch_split(self, q, k_new, v_new, m_max):
        """Two-stream pipeline over unit groups: scan(g) -> plan(g) -> attention(g),
        with scan(g+1) issued after scan(g) so it overlaps plan(g)."""
        L = self.L
        main = torch.cuda.current_stream()
        if not hasattr(self, "_ev"):
            self._ev = [torch.cuda.Event() for _ in range(2 * self.split + 1)]
            self._hs = [ctypes.c_void_p(st.cuda_stream) for st in self._streams]
        ev = self._ev
        ev[0].record(main)
        qp = q.data_ptr()
        gsz = self.G * self.d * 4
        for gi, grp in enumerate(self._groups):
            st = self._streams[gi]
            st.wait_event(ev[0])
            if gi:
                st.wait_event(ev[gi])
            sv = grp.get("sv")
            if sv is None:
                sv = grp["sv"] = self._group_step_view(grp, q)
            sv.q = qp + grp["u0"] * gsz
            _lib.check(L.wk_centroid_scan(ctypes.byref(grp["ixv"]), ctypes.byref(sv), ctypes.byref(self._zp),
                                          grp["n"], m_max, self._hs[gi]), "wk_centroid_scan")
            ev[gi + 1].record(st)
        kp, vp, dsz = k_new.data_ptr(), v_new.data_ptr(), self.d * 4
        for gi, grp in enumerate(self._groups):
            n, u0, h = grp["n"], grp["u0"], self._hs[gi]
            _lib.check(L.wk_plan_zones(ctypes.byref(grp["ixv"]), ctypes.byref(grp["stv"]), ctypes.byref(grp["sv"]),
                                       ctypes.byref(self._zp), kp + u0 * dsz, vp + u0 * dsz,
                                       n, m_max, self.store_bf16, h), "wk_plan_zones")
            _lib.check(L.wk_tripartite_attn(ctypes.byref(grp["ixv"]), ctypes.byref(grp["stv"]),
                                            ctypes.byref(grp["sv"]), ctypes.byref(self._zp), n, self.S,
                                            self.store_bf16, h), "wk_tripartite_attn")
            ev[self.split + 1 + gi].record(self._streams[gi])
        for gi in range(self.split):
            main.wait_event(ev[self.split + 1 + gi])

    def _step_view(self, q: torch.Tensor) -> _lib.StepViewC:
        return _lib.StepViewC(
            _ptr(q), _ptr(self.m_dev), _ptr(self.scores), _ptr(self.rlist), _ptr(self.elist),
            _ptr(self.nr), _ptr(self.ne), _ptr(self.zmask), _ptr(self.ru_ids), _ptr(self.ru_mask),
            _ptr(self.ru_pre), _ptr(self.eu_ids), _ptr(self.eu_mask), _ptr(self.cnt),
            _ptr(self.tail), _ptr(self.part), _ptr(self.out), _ptr(self.logden), _ptr(self.cov),
            _ptr(self.status), self.r_cap, self.e_cap, self.ru_cap, self.eu_cap,
            _ptr(self.rtok_row), _ptr(self.rtok_mask), _ptr(self.sel_done), self.rt_cap, 0,
            _ptr(self.eu_x), _ptr(self.eu_sz), _ptr(self.rbits), _ptr(self.ebits), _ptr(self.pieces),
            _ptr(self.woff), self.w_cap, self.pc_cap,
            _ptr(self.cache.arena_k) if self.cache else None, _ptr(self.cache.arena_v) if self.cache else None,
            _ptr(self.cache.slot_ids) if self.cache else None, _ptr(self.cache.slot_off) if self.cache else None,
            self.cache.phys * self.cache.bt if self.cache else 0, self.cache.list_cap if self.cache else 0,
            self.cache.bt if self.cache else 0, 4 if self.offload else 2,
            _ptr(self.q64), _ptr(self.xscr), _ptr(self.xcount))

    # --------------------------------------------------------------- clustering
    def _run_segments(self, segs: list[dict]):
        """Cluster + finalize + pack a list of segments (one wk_kmeans_segments
        call per chunk bounded by a scratch budget).

        Offload layers: the pack writes the cluster-contiguous K/V straight into
        the pinned host store over the host link (engine.py:133-135, store.py:88),
        so the segments are split into unit groups launched alternately on two
        streams -- group g's host writes (km_finalize) overlap group g + 1's
        clustering."""
        d = self.d
        budget = 1 << 26  # points per chunk (scratch ~ 0.6 KB/point at d=128)
        groups = 4 if (self.offload and len(segs) >= 32) else 1
        if groups > 1:
            units = sorted({s["unit"] for s in segs})
            cut = [units[len(units) * g // groups] for g in range(groups)] + [units[-1] + 1]
            main = torch.cuda.current_stream()
            streams = [torch.cuda.Stream(device=self.dev) for _ in range(2)]
            start = torch.cuda.Event()
            start.record(main)
            keep = []  # scratch of every group alive until both streams drained
            for g in range(groups):
                part = [s for s in segs if cut[g] <= s["unit"] < cut[g + 1]]
                st = streams[g % 2]
                st.wait_event(start)
                with torch.cuda.stream(st):
                    keep += self._run_segments_chunked(part, budget, sync=False)
            for st in streams:
                main.wait_stream(st)
            torch.cuda.synchronize(self.dev)
            del keep
            return
        self._run_segments_chunked(segs, budget, sync=True)

    def _run_segments_chunked(self, segs: list[dict], budget: int, sync: bool):
        d = self.d
        keep = []
        i = 0
        while i < len(segs):
            chunk, tot = [], 0
            while i < len(segs) and (not chunk or tot + segs[i]["L"] <= budget):
                chunk.append(segs[i]); tot += segs[i]["L"]; i += 1
            sumL = sum(s["L"] for s in chunk)
            sumK = sum(max(1, s["k"]) for s in chunk)
            dev = self.dev
            P = torch.empty((sumL, d), dtype=torch.float32, device=dev)
            P16 = torch.empty((sumL, d), dtype=torch.float16, device=dev)
            C = torch.empty((sumK, d), dtype=torch.float32, device=dev)
            A = torch.zeros(sumL, dtype=torch.int32, device=dev)
            perm = torch.empty(sumL, dtype=torch.int32, device=dev)
            sims = torch.empty(sumL, dtype=torch.float32, device=dev)
            md = torch.empty(2 * sumL, dtype=torch.float32, device=dev)
            segs_dev = torch.empty(len(chunk) * ctypes.sizeof(_lib.SegmentC), dtype=torch.uint8,
                                   device=dev)
            arr = (_lib.SegmentC * len(chunk))()
            po = co = 0
            for j, s in enumerate(chunk):
                a = arr[j]
                a.keys, a.values, a.key_stride = s["keys"], s["values"], s["stride"]
                a.L, a.k, a.unit = s["L"], s["k"], s["unit"]
                a.cid_base, a.row_base, a.tok_base = s["cid_base"], s["row_base"], s["tok_base"]
                a.p_off, a.c_off = po, co
                for t in range(4):
                    a.rng[t] = s["rng"][t]
                po += s["L"]; co += max(1, s["k"])
            scr = _lib.BuildScratchC(_ptr(P), _ptr(C), _ptr(A), _ptr(perm), _ptr(sims), _ptr(md),
                                     _ptr(segs_dev), _ptr(self.status), _ptr(P16))
            rc = self.L.wk_kmeans_segments(
                ctypes.byref(self._ixv), arr, len(chunk), ctypes.byref(scr), d, self.store_bf16,
                self.cfg.index.kmeans_iters, self.blas_threads, max(s["L"] for s in chunk),
                max(max(1, s["k"]) for s in chunk), ctypes.c_void_p(_stream()))
            _lib.check(rc, "wk_kmeans_segments")
            # keep scratch alive until the kernels ran
            if sync:
                torch.cuda.current_stream().synchronize()
                del P, P16, C, A, perm, sims, md, segs_dev
            else:
                keep.append((P, P16, C, A, perm, sims, md, segs_dev, arr))
        return keep

    # ------------------------------------------------------------------ prefill
    def prefill(self, keys: torch.Tensor, values: torch.Tensor, lengths=None):
        """keys/values: [U, n, d] float32 on the device (HeadEngine.prefill,
        engine.py:110-138).  ``lengths`` optionally gives per-unit prompt
        lengths (rows beyond are ignored)."""
        if self.prefilled:
            raise ConfigError("prefill called twice")
        U, d, ic = self.U, self.d, self.cfg.index
        if keys.dim() != 3 or keys.shape != values.shape or keys.shape[0] != U or keys.shape[2] != d:
            raise ConfigError(f"bad prefill shapes {tuple(keys.shape)} / {tuple(values.shape)}")
        keys = keys.to(self.dev, torch.float32).contiguous()
        values = values.to(self.dev, torch.float32).contiguous()
        n_all = keys.shape[1]
        lengths = [n_all] * U if lengths is None else [int(x) for x in lengths]
        if any(n < 1 or n > n_all for n in lengths):
            raise ConfigError("bad prefill lengths")
        segs = []
        for u, n in enumerate(lengths):
            st = self.units[u]
            st.total = n
            st.n_sink = min(ic.sink_tokens, n)
            index_end = max(st.n_sink, n - ic.local_window)
            st.buffer_start = index_end
            L = index_end - st.n_sink
            if L > self.s_cap:
                raise ConfigError("prefill longer than the configured capacity")
            cid = 0
            for seg_idx, s0 in enumerate(range(0, L, ic.segment_size)):
                ln = min(ic.segment_size, L - s0)
                k = math.ceil(ln / ic.centroid_ratio)
                base = (u * n_all + st.n_sink + s0) * d
                segs.append(dict(keys=keys.data_ptr() + 4 * base, values=values.data_ptr() + 4 * base,
                                 stride=d, L=ln, k=k, unit=u, cid_base=cid, row_base=s0,
                                 tok_base=st.n_sink + s0, rng=pcg64_words(ic.rng_seed, 1, seg_idx)))
                cid += k
            st.m = cid
            st.store_fill = L
            st.n_steady = st.n_sink + (n - index_end)
            # steady rows: sinks then the window (engine.py:126-130)
            rows = list(range(st.n_sink)) + list(range(index_end, n))
            if rows:
                idx = torch.tensor(rows, device=self.dev, dtype=torch.long)
                self.st_k[u, : len(rows)] = self._to_rows(keys[u, idx], 0)
                self.st_v[u, : len(rows)] = self._to_rows(values[u, idx], 0)
                self.st_tok[u, : len(rows)] = idx.to(torch.int32)
        if self.m_cap < max(s.m for s in self.units):
            raise ConfigError("cluster capacity exceeded")
        if segs:
            self._run_segments(segs)
        self.st_n.copy_(torch.tensor([s.n_steady for s in self.units], dtype=torch.int32))
        self.next_tok.copy_(torch.tensor([s.total for s in self.units], dtype=torch.int32))
        self.m_dev.copy_(torch.tensor([s.m for s in self.units], dtype=torch.int32))
        self.n_store_dev.copy_(torch.tensor([s.store_fill for s in self.units], dtype=torch.int32))
        self.check_status("prefill")
        if self.cache is not None:
            self.cache.register_new()
        self.prefilled = True
        return self

    # ------------------------------------------------------------------- decode
    def decode(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor,
               allow_update: bool = True):
        """One decode step for every unit (HeadEngine.decode_step,
        engine.py:174-232).  q: [U, G, d], k_new/v_new: [U, d] float32 device
        tensors.  Returns device views (out [U,G,d], logden [U,G], cov [U,G])
        valid until the next call."""
        if not self.prefilled:
            raise ConfigError("decode_step before prefill")
        self.launch_step(q, k_new, v_new)
        for s in self.units:
            s.total += 1
            s.n_steady += 1
        if allow_update:
            self.maybe_update()
        return self.out, self.logden, self.cov

    def launch_step(self, q, k_new, v_new, out=None):
        """Kernel launches of one decode step only (graph-capturable).  ``out``:
        optional [U, G, d] float32 device tensor the attention output is written
        to instead of ``self.out``."""
        q = q if (q.dtype == torch.float32 and q.is_contiguous()) else q.float().contiguous()
        self._q = q
        stream = ctypes.c_void_p(_stream())
        L = self.L
        sv = self._step_view(q)
        if out is not None:
            if out.dtype != torch.float32 or not out.is_contiguous() or out.shape != self.out.shape:
                raise ConfigError(f"out must be a contiguous float32 {tuple(self.out.shape)} tensor")
            if self.split > 1:
                raise ConfigError("out= is not supported with split > 1")
            sv.out = _ptr(out)
        m_max = max(s.m for s in self.units)
        if self.split > 1:
            k_new = k_new if (k_new.dtype == torch.float32 and k_new.is_contiguous()) else k_new.float().contiguous()
            v_new = v_new if (v_new.dtype == torch.float32 and v_new.is_contiguous()) else v_new.float().contiguous()
            self._launch_split(q, k_new, v_new, m_max)
            return
        if self.cache is None:  # one fused call: append + scan + zones + attention
            _lib.check(L.wk_decode_step(ctypes.byref(self._ixv), ctypes.byref(self._stv), ctypes.byref(sv),
                                        ctypes.byref(self._zp), _ptr(k_new), _ptr(v_new), self.U, m_max,
                                        self.S, self.store_bf16, stream), "wk_decode_step")
            return
        _lib.check(L.wk_append_tokens(ctypes.byref(self._stv), _ptr(k_new), _ptr(v_new), self.U,
                                      self.d, self.store_bf16, _ptr(self.status), stream), "wk_append_tokens")
        _lib.check(L.wk_score_topk(ctypes.byref(self._ixv), ctypes.byref(sv), ctypes.byref(self._zp),
                                   self.U, m_max, stream), "wk_score_topk")
        if self.cache is not None:  # wave buffer: lookup, replacement, miss plan
            self.cache.step(sv)
        _lib.check(L.wk_tripartite_attn(ctypes.byref(self._ixv), ctypes.byref(self._stv),
                                        ctypes.byref(sv), ctypes.byref(self._zp), self.U, self.S,
                                        self.store_bf16, stream), "wk_tripartite_attn")

    def needs_update(self):
        ic = self.cfg.index
        return [u for u, s in enumerate(self.units)
                if s.n_steady - s.n_sink >= ic.update_segment + ic.local_window]

    def maybe_update(self):
        """Fold full update segments of the decode buffer into the index
        (ClusterIndex.update, index.py:168-186)."""
        ic = self.cfg.index
        todo = self.needs_update()
        while todo:
            segs, keep = [], []
            k = math.ceil(ic.update_segment / ic.centroid_ratio)
            tmp_k = torch.empty((len(todo), ic.update_segment, self.d), dtype=torch.float32,
                                device=self.dev)
            tmp_v = torch.empty_like(tmp_k)
            sinks = {self.units[u].n_sink for u in todo}
            batched = len(sinks) == 1
            if batched:  # one gather for all units (the common case)
                r0 = next(iter(sinks))
                idx = torch.tensor(todo, device=self.dev, dtype=torch.long)
                tmp_k.copy_(self._from_rows(self.st_k[idx, r0:r0 + ic.update_segment], r0))
                tmp_v.copy_(self._from_rows(self.st_v[idx, r0:r0 + ic.update_segment], r0))
            for j, u in enumerate(todo):
                s = self.units[u]
                if s.m + k > self.m_cap or s.store_fill + ic.update_segment > self.s_cap:
                    raise ConfigError("index capacity exceeded: raise max_decode")
                r0 = s.n_sink
                if not batched:
                    tmp_k[j] = self._from_rows(self.st_k[u, r0:r0 + ic.update_segment], r0)
                    tmp_v[j] = self._from_rows(self.st_v[u, r0:r0 + ic.update_segment], r0)
                base = j * ic.update_segment * self.d
                segs.append(dict(keys=tmp_k.data_ptr() + 4 * base, values=tmp_v.data_ptr() + 4 * base,
                                 stride=self.d, L=ic.update_segment, k=k, unit=u, cid_base=s.m,
                                 row_base=s.store_fill, tok_base=s.buffer_start,
                                 rng=pcg64_words(ic.rng_seed, 2, s.update_round)))
            self._run_segments(segs)
            # keep the buffer tail (index.py:179-180): shift rows down.  Units
            # with the same (sink, steady) extent are shifted by one batched
            # copy; the swizzle keys are unchanged when the shift is a multiple
            # of 8 rows (the default 1,024), else the rows are re-keyed
            groups = {}
            for u in todo:
                s = self.units[u]
                groups.setdefault((s.n_sink, s.n_steady), []).append(u)
            rekey = self.swizzled and ic.update_segment % 8 != 0
            for (n_sink, n_steady), us in groups.items():
                r0, r1 = n_sink + ic.update_segment, n_steady
                idx = torch.tensor(us, device=self.dev, dtype=torch.long)
                for t in (self.st_k, self.st_v):
                    rows = t[idx, r0:r1]
                    if rekey:
                        rows = self._to_rows(self._from_rows(rows, r0), n_sink)
                    t[idx, n_sink:n_sink + (r1 - r0)] = rows.clone()
                self.st_tok[idx, n_sink:n_sink + (r1 - r0)] = self.st_tok[idx, r0:r1].clone()
            for u in todo:
                s = self.units[u]
                s.n_steady -= ic.update_segment
                s.m += k
                s.store_fill += ic.update_segment
                s.buffer_start += ic.update_segment
                s.update_round += 1
            self.st_n.copy_(torch.tensor([s.n_steady for s in self.units], dtype=torch.int32))
            self.m_dev.copy_(torch.tensor([s.m for s in self.units], dtype=torch.int32))
            self.n_store_dev.copy_(torch.tensor([s.store_fill for s in self.units], dtype=torch.int32))
            self.on_clusters_added(todo, k)
            todo = self.needs_update()

    def on_clusters_added(self, units, k):
        """Block-cache registration of the new clusters (engine.py:212-214)."""
        if self.cache is not None:
            self.cache.register_new(units)

    # ----------------------------------------------------------- full attention
    def full_attention(self, q: torch.Tensor, out=None):
        """Exact attention over every token of each unit (oracle_attention,
        attention.py:55-64; also the full-attention comparator)."""
        q = q.float().contiguous()
        sv = self._step_view(q)
        if out is not None:
            sv.out = out.data_ptr()
        rc = self.L.wk_full_attn(ctypes.byref(self._ixv), ctypes.byref(self._stv), ctypes.byref(sv),
                                 _ptr(self.n_store_dev), self.U, self.G, self.d, self.S,
                                 self.store_bf16, ctypes.c_void_p(_stream()))
        _lib.check(rc, "wk_full_attn")
        return self.out if out is None else out

    # ------------------------------------------------------- index injection
    def set_index(self, u: int, C64, sizes):
        """Install a given meta index (fp64 centroids [m, d], sizes [m]) as
        unit u's clusters -- the state ``ClusterIndex`` holds after a build
        (index.py:110-139).  Store rows are laid out cluster-contiguously in
        id order and left empty; used to run the zone planner on externally
        supplied indexes (rank goldens, function-level API)."""
        C64 = torch.as_tensor(np.asarray(C64, dtype=np.float64), device=self.dev)
        sizes = torch.as_tensor(np.asarray(sizes, dtype=np.int64), device=self.dev).to(torch.int32)
        m = C64.shape[0]
        if C64.dim() != 2 or C64.shape[1] != self.d or sizes.shape != (m,) or m > self.m_cap:
            raise ConfigError(f"bad index shapes {tuple(C64.shape)} / {tuple(sizes.shape)} (m_cap {self.m_cap})")
        off = torch.cumsum(sizes, 0, dtype=torch.int32) - sizes
        if m and int(off[-1] + sizes[-1]) > self.s_cap:
            raise ConfigError("index sizes exceed the store capacity")
        self.C64[u].zero_()
        self.C64[u, :m] = C64
        self.C32[u, :m] = C64.float()
        self.Cnorm[u, :m] = self.C32[u, :m].double().norm(dim=1).float()
        self.Cmax[u] = float(self.Cnorm[u, :m].max()) * (1 + 1e-6) if m else 0.0
        self.cl_size[u].zero_()
        self.cl_size[u, :m] = sizes
        self.cl_off[u, :m] = off
        st = self.units[u]
        st.m = m
        st.store_fill = int(sizes.sum())
        self.m_dev[u] = m
        self.n_store_dev[u] = st.store_fill
        self.prefilled = True

    def plan(self, q: torch.Tensor, q64: torch.Tensor | None = None):
        """Zone planning only (ClusterIndex.rank + plan_zones, index.py:61-93)
        for every unit: the centroid scan and exact selection of one decode
        step without the append or the attention.  Returns (rlist [U,G,r_cap],
        nr [U], elist [U,G,e_cap] or None, ne [U]) device views."""
        q = q.float().contiguous()
        self._q = q
        prev, q64 = self.q64, (None if q64 is None else q64.double().contiguous())
        if q64 is not None:
            self.q64 = q64
        sv = self._step_view(q)
        self.q64 = prev
        m_max = max(s.m for s in self.units)
        _lib.check(self.L.wk_score_topk(ctypes.byref(self._ixv), ctypes.byref(sv), ctypes.byref(self._zp),
                                        self.U, m_max, ctypes.c_void_p(_stream())), "wk_score_topk")
        self.check_status("plan")
        return self.rlist, self.nr, self.elist, self.ne

    # ---------------------------------------------------------------- checking
    def check_status(self, what="step"):
        code = int(self.status.item())
        if code:
            self.status.zero_()
            _lib.raise_status(code, what)

    # host views of the index (tests; not on the hot path)
    def index_arrays(self, u: int):
        m = self.units[u].m
        return dict(C64=self.C64[u, :m].cpu().numpy(), VS32=self.VS32[u, :m].cpu().numpy(),
                    VS64=None if self.VS64 is None else self.VS64[u, :m].cpu().numpy(),
                    sizes=self.cl_size[u, :m].cpu().numpy().astype(np.int64),
                    offsets=self.cl_off[u, :m].cpu().numpy(),
                    store_tok=self.store_tok[u, :self.units[u].store_fill].cpu().numpy())
