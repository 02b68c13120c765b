"""Trace replay with a JSON-ready report (tierkv runner.py:28-126).

The reference drives one ``HeadEngine`` per trace head, one head at a time.
Here all heads of the trace are the units of ONE ``WaveLayer`` (one kv-head
and one query per unit, G = 1) with the device block cache in per-head mode,
so every decode step of the whole trace is one batched launch sequence: the
fused decode step, the cache step, the device recall@k, and -- with
``with_oracle`` -- the full-attention oracle.  Per-step metrics are gathered
on the device and copied to the host once per step.  The report has the
reference's schema and field order; everything except ``timestamp`` is
deterministic for a fixed trace / config / BLAS thread count.
"""

from __future__ import annotations

import ctypes
import datetime
import json
import os
import time

import numpy as np
import torch

from . import _lib
from .block_cache import DeviceBlockCache
from .config import EngineConfig
from .metrics import relative_l2
from .errors import ConfigError
from .tracefile import TraceFile
from .wave import WaveLayer, _stream

SCHEMA_VERSION = 1
STEP_FIELDS = ("recall", "rel_error", "hits", "misses", "bytes_slow_to_fast", "bytes_fast_internal",
               "denominator_coverage", "m", "r", "e")


def _percentile(values, p):
    return None if not values else float(np.percentile(np.asarray(values, dtype=np.float64), p))


class TraceEngine:
    """All heads of a trace as one batched wave layer (U = heads, G = 1)."""

    def __init__(self, cfg: EngineConfig, n_heads: int, d: int, n_prefill: int, n_decode: int, *,
                 device="cuda", blas_threads: int | None = None, store_dtype=torch.float32):
        from .clustering import blas_threads as _bt
        self.cfg = cfg.validate()
        self.H, self.d = n_heads, d
        self.device = torch.device(device)
        self.blas_threads = _bt() if blas_threads is None else blas_threads
        self.lay = WaveLayer(self.cfg, n_heads, 1, d, max_prefill=n_prefill, max_decode=max(1, n_decode),
                             store_dtype=store_dtype, device=self.device, blas_threads=self.blas_threads,
                             keep_vs64=True)
        self.cache = DeviceBlockCache(self.lay, "head")
        self.lay.on_clusters_added = lambda units, k: self.cache.register_new(units)
        self.step = 0
        dev = self.device
        self._recall_s = torch.empty((n_heads, self.lay.s_cap + self.lay.t_cap), dtype=torch.float32, device=dev)
        self._recall_f = torch.empty((n_heads, self.lay.s_cap), dtype=torch.uint8, device=dev)
        self._recall = torch.zeros(n_heads, dtype=torch.float32, device=dev)
        self._oracle = torch.zeros((n_heads, 1, d), dtype=torch.float32, device=dev)

    def prefill(self, keys: np.ndarray, values: np.ndarray):
        dev = self.device
        self.lay.prefill(torch.from_numpy(np.ascontiguousarray(keys, np.float32)).to(dev),
                         torch.from_numpy(np.ascontiguousarray(values, np.float32)).to(dev))
        self.cache.register_new()
        return self

    def decode_step(self, q: np.ndarray, k: np.ndarray, v: np.ndarray, with_oracle: bool = False):
        """One step for every head: q, k, v [H, d] -> outputs [H, d] f64, per-head
        metric columns (HeadEngine.decode_step semantics, engine.py:174-232)."""
        lay, H, d, dev = self.lay, self.H, self.d, self.device
        if any(s.n_steady + 1 > lay.t_cap for s in lay.units):
            raise ConfigError("decode capacity exceeded")
        qt = torch.from_numpy(np.ascontiguousarray(q, np.float32)).to(dev).view(H, 1, d)
        kt = torch.from_numpy(np.ascontiguousarray(k, np.float32)).to(dev)
        vt = torch.from_numpy(np.ascontiguousarray(v, np.float32)).to(dev)
        c0 = self.cache.counters[:, :4].clone()
        lay.launch_step(qt, kt, vt)
        self.cache.step(self.step)
        sv = lay._step_view(lay._q)
        _lib.check(lay.L.wk_recall_at_k(ctypes.byref(lay._ixv), ctypes.byref(lay._stv), ctypes.byref(sv),
                                        lay.n_store_dev.data_ptr(), H, 1, d, self.cfg.metrics_k,
                                        lay.blas_threads, self._recall_s.data_ptr(), self._recall_f.data_ptr(),
                                        self._recall_s.shape[1], lay.store_bf16, self._recall.data_ptr(),
                                        ctypes.c_void_p(_stream())), "wk_recall_at_k")
        dk = (self.cache.counters[:, :4] - c0).cpu().numpy()
        out = lay.out[:, 0].double().cpu().numpy()
        cov = lay.cov[:, 0].double().cpu().numpy()
        rec = self._recall.double().cpu().numpy()
        nr, ne = lay.nr.cpu().numpy(), lay.ne.cpu().numpy()
        if with_oracle:  # after the reads: the full-attention merge rewrites out / cov / logden slots
            sv.out = self._oracle.data_ptr()
            _lib.check(lay.L.wk_full_attn(ctypes.byref(lay._ixv), ctypes.byref(lay._stv), ctypes.byref(sv),
                                          lay.n_store_dev.data_ptr(), H, 1, d, lay.S, lay.store_bf16,
                                          ctypes.c_void_p(_stream())), "wk_full_attn")
        oracle = self._oracle[:, 0].double().cpu().numpy() if with_oracle else None
        lay.check_status("decode_step")
        for s in lay.units:
            s.total += 1
            s.n_steady += 1
        lay.maybe_update()
        ms = [s.m for s in lay.units]  # after the index update, as HeadEngine.decode_step
        cols = {
            "recall": [float(x) for x in rec],
            "rel_error": ([relative_l2(out[h], oracle[h]) for h in range(H)] if with_oracle else [None] * H),
            "hits": [int(x) for x in dk[:, 0]], "misses": [int(x) for x in dk[:, 1]],
            "bytes_slow_to_fast": [int(x) for x in dk[:, 2]], "bytes_fast_internal": [int(x) for x in dk[:, 3]],
            "denominator_coverage": [float(x) for x in cov], "m": ms,
            "r": [int(x) for x in nr], "e": [int(x) for x in ne],
        }
        self.step += 1
        return out, cols, oracle

    def head_totals(self, h: int) -> dict:
        """Per-head totals (runner.py:83-88): cache stats + store accounting + m."""
        t = self.cache.stats(h)
        n_blocks = int(self.cache.n_blocks[h])
        t["bytes_offloaded"] = n_blocks * self.cfg.block_size_bytes
        t["slow_blocks"] = n_blocks
        t["clusters"] = self.lay.units[h].m
        return t


def run_trace(trace: TraceFile, cfg: EngineConfig, with_oracle: bool = False, *, device="cuda",
              blas_threads: int | None = None):
    """Replay a trace (runner.py:28-110); returns (report, outputs, oracle outputs),
    outputs shaped [n_decode, n_heads, d] float64."""
    cfg.validate()
    trace.validate()
    t0 = time.perf_counter()
    eng = TraceEngine(cfg, trace.n_heads, trace.d, trace.n_prefill, trace.n_decode, device=device,
                      blas_threads=blas_threads).prefill(trace.prefill_keys, trace.prefill_values)
    torch.cuda.synchronize()
    build_seconds = time.perf_counter() - t0
    H = trace.n_heads
    outputs = np.zeros((trace.n_decode, H, trace.d))
    oracle_outputs = np.zeros_like(outputs) if with_oracle else None
    steps = [{k: [] for k in STEP_FIELDS} for _ in range(H)]
    t1 = time.perf_counter()
    for t in range(trace.n_decode):
        out, cols, orc = eng.decode_step(trace.queries[t], trace.new_keys[t], trace.new_values[t], with_oracle)
        outputs[t] = out
        if with_oracle:
            oracle_outputs[t] = orc
        for h in range(H):
            for k in STEP_FIELDS:
                steps[h][k].append(cols[k][h])
    run_seconds = time.perf_counter() - t1
    per_head = [{"head": h, "steps": steps[h], "totals": eng.head_totals(h)} for h in range(H)]
    recalls = [x for s in steps for x in s["recall"]]
    errors = [x for s in steps for x in s["rel_error"] if x is not None]
    hits = sum(p["totals"]["hits"] for p in per_head)
    misses = sum(p["totals"]["misses"] for p in per_head)
    report = {
        "schema_version": SCHEMA_VERSION,
        "timestamp": {
            "generated_at": datetime.datetime.now(datetime.timezone.utc).isoformat(),
            "build_seconds": build_seconds,
            "run_seconds": run_seconds,
        },
        "config": cfg.to_dict(),
        "trace": {"n_heads": H, "d": trace.d, "n_prefill": trace.n_prefill, "n_decode": trace.n_decode},
        "per_head": per_head,
        "aggregates": {
            "mean_recall": float(np.mean(recalls)) if recalls else None,
            "mean_rel_error": float(np.mean(errors)) if errors else None,
            "p50_rel_error": _percentile(errors, 50),
            "p90_rel_error": _percentile(errors, 90),
            "p99_rel_error": _percentile(errors, 99),
            "cumulative_hit_ratio": hits / (hits + misses) if hits + misses else 0.0,
            "total_bytes_slow_to_fast": sum(p["totals"]["bytes_slow_to_fast"] for p in per_head),
            "total_bytes_fast_internal": sum(p["totals"]["bytes_fast_internal"] for p in per_head),
            "total_bytes_offloaded": sum(p["totals"]["bytes_offloaded"] for p in per_head),
        },
    }
    return report, outputs, oracle_outputs


def oracle_trace(trace: TraceFile, *, device="cuda") -> np.ndarray:
    """Exact attention of every step and head (runner.py:113-126), on the device:
    the full K/V history per head is resident, each step appends one row and
    runs the full-attention kernel over all heads at once."""
    trace.validate()
    H, n, d, T = trace.n_heads, trace.n_prefill, trace.d, trace.n_decode
    dev = torch.device(device)
    K = torch.zeros((H, n + T, d), dtype=torch.float64, device=dev)
    V = torch.zeros_like(K)
    K[:, :n] = torch.from_numpy(trace.prefill_keys).to(dev, torch.float64)
    V[:, :n] = torch.from_numpy(trace.prefill_values).to(dev, torch.float64)
    out = np.zeros((T, H, d))
    for t in range(T):
        K[:, n + t] = torch.from_numpy(trace.new_keys[t]).to(dev, torch.float64)
        V[:, n + t] = torch.from_numpy(trace.new_values[t]).to(dev, torch.float64)
        q = torch.from_numpy(trace.queries[t]).to(dev, torch.float64)
        s = torch.einsum("hnd,hd->hn", K[:, : n + t + 1], q) / float(np.sqrt(d))
        w = torch.exp(s - s.max(dim=1, keepdim=True).values)
        out[t] = (torch.einsum("hn,hnd->hd", w, V[:, : n + t + 1]) / w.sum(1, keepdim=True)).cpu().numpy()
    return out


# ---------------------------------------------------------------------------
# config sweeps (cli.py:19-24 SWEEP_AXES, cmd_sweep cli.py:84-97)
# ---------------------------------------------------------------------------
SWEEP_AXES = {
    "retrieval_fraction": float,
    "estimation_fraction": float,
    "segment_size": int,
    "cache_fraction": float,
}


def sweep_trace(trace: TraceFile, base: EngineConfig, axis: str, values, with_oracle: bool = False,
                out_dir: str | None = None, *, device="cuda", blas_threads: int | None = None):
    """Replay `trace` once per value of one config axis (tierkv's `sweep`
    command): each report is run_trace's with "sweep": {"axis", "value"}; with
    out_dir, written as report_<axis>_<value>.json like the reference.  `values`
    is a list or the reference's comma-separated string.  Returns the reports."""
    if axis not in SWEEP_AXES:
        raise ConfigError(f"unknown sweep axis {axis!r}; choose from {sorted(SWEEP_AXES)}")
    cast = SWEEP_AXES[axis]
    raws = [v.strip() for v in values.split(",")] if isinstance(values, str) else [str(v) for v in values]
    reports = []
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
    for raw in raws:
        value = cast(raw)
        cfg = EngineConfig.from_dict({**base.to_dict(), axis: value})
        report, _, _ = run_trace(trace, cfg, with_oracle=with_oracle, device=device, blas_threads=blas_threads)
        report["sweep"] = {"axis": axis, "value": value}
        if out_dir:
            with open(os.path.join(out_dir, f"report_{axis}_{raw}.json"), "w") as f:
                json.dump(report, f, indent=2, sort_keys=True, allow_nan=False)
                f.write("\n")
        reports.append(report)
    return reports

