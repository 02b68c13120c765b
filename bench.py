"""Decode-throughput benchmark: wave-index decode attention on B200.

Workload (BASELINE.json configs[1]): Llama-3-8B-shaped decode at 120K context,
batch 16, 32 layers (32 q / 8 kv heads, d=128) on one B200, against
full-attention decode over the same KV.  A "step" = one decode token for every
request through all 32 layers of attention.  Full KV at B=16 (257.7 GB) exceeds
HBM, so the 32 layers cycle over ``--layer-bufs`` distinct layer buffers
(each >> L2), as SURVEY.md 8(d) prescribes; both paths use the same buffers.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference's
CPU algorithm instead (the C oracle port of tierkv, oracle/), see DESIGN.md.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HQ, HKV, D = 32, 8, 128
# head shapes of the BASELINE configs (configs[1] Llama-3-8B, configs[4] Qwen2.5-7B)
MODELS = {"llama3-8b": (32, 8, 128, 32), "qwen2.5-7b": (28, 4, 128, 28)}
METRIC = "decode tokens/sec at 120K ctx (device-timed) and % HBM roofline vs full attn"
LAUNCHES_PER_LAYER = 4  # score_v5, select_v6 (+ fused append, union, estimation prep), attend_v4, att4_merge


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--model", default="llama3-8b", choices=sorted(MODELS))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="wave", choices=["wave", "reference"])
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=122880)
    ap.add_argument("--layers", type=int, default=0, help="0: the model's layer count")
    ap.add_argument("--layer-bufs", type=int, default=4)
    ap.add_argument("--fa-steps", type=int, default=3)
    ap.add_argument("--cpu-steps", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-group", type=int, default=4, help="layers per host-I/O group of the e2e leg")
    ap.add_argument("--no-flashinfer", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank serves --batch requests; strong: the --batch x H_kv units "
                         "are split over the ranks (parallel.shard_units)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the reduced configs[2]/[3]/[4] legs of the default run")
    ap.add_argument("--split", type=int, default=1, help="unit groups pipelined on streams")
    ap.add_argument("--build", action="store_true",
                    help="configs[2]: segmented clustering index build at 120K and 256K, "
                         "throughput + sampled assignment parity vs the CPU oracle")
    ap.add_argument("--offload", action="store_true",
                    help="configs[3]: host-KV offload (pinned store + HBM wave buffer); "
                         "use with e.g. --ctx 1048576 --batch 4")
    return ap.parse_args()


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.samples[0][1]),
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------ synthetic data
def gen_layer(torch, U, n, d, seed, dev, n_centers=32, seg=8192, noise=0.5):
    """Keys: per-8K-segment latent centres + Gaussian noise (spatial locality,
    like tierkv synth.py:46-70); values N(0,1); all bf16-representable."""
    g = torch.Generator(device=dev).manual_seed(seed)
    n_seg = -(-n // seg)
    centers = torch.randn((U, n_seg, n_centers, d), generator=g, device=dev)
    cidx = torch.randint(n_centers, (U, n), generator=g, device=dev)
    seg_id = (torch.arange(n, device=dev) // seg).expand(U, n)
    uidx = torch.arange(U, device=dev)[:, None].expand(U, n)
    keys = centers[uidx, seg_id, cidx]
    keys += noise * torch.randn((U, n, d), generator=g, device=dev)
    keys = keys.bfloat16().float()
    values = torch.randn((U, n, d), generator=g, device=dev).bfloat16().float()
    return keys, values, centers


def gen_queries(torch, centers, G, steps, seed, persistence=0.9, shared=0.25, per_head=0.25):
    """Per unit a persistent random walk over its latent centres (temporal
    locality, synth.py:57-67); each GQA group shares the walk + shared noise,
    each head adds its own noise.  Returns [steps, U, G, d] bf16-valued fp32."""
    import numpy as np
    U, n_seg, nc, d = centers.shape
    dev = centers.device
    rng = np.random.default_rng(seed)
    walk = rng.integers(n_seg * nc, size=U)
    idx = np.empty((steps, U), np.int64)
    for t in range(steps):
        jump = rng.random(U) >= persistence
        walk = np.where(jump, rng.integers(n_seg * nc, size=U), walk)
        idx[t] = walk
    flat = centers.reshape(U, n_seg * nc, d)
    it = torch.from_numpy(idx).to(dev)
    base = flat[torch.arange(U, device=dev)[None, :].expand(steps, U), it]  # [steps, U, d]
    g = torch.Generator(device=dev).manual_seed(seed)
    q = base[:, :, None, :] + shared * torch.randn((steps, U, 1, d), generator=g, device=dev)
    q = q + per_head * torch.randn((steps, U, G, d), generator=g, device=dev)
    return q.bfloat16().float().contiguous()


# ------------------------------------------- library full-attention comparator
def flashinfer_decode(torch, B, HQ, HKV, D, ctx, layers, reps, log, page=64):
    """Full-attention decode through flashinfer's trtllm-gen sm100a kernels
    (library code; SURVEY 8(d) names it as the comparator): same batch, heads,
    context, bf16 paged KV (one layer's KV, >> L2, reused for every layer)."""
    try:
        from flashinfer.decode import trtllm_batch_decode_with_kv_cache
        dev = torch.device("cuda")
        pages_per = ctx // page
        kv = torch.empty((B * pages_per, 2, HKV, page, D), device=dev, dtype=torch.bfloat16).normal_()
        bt = torch.arange(B * pages_per, device=dev, dtype=torch.int32).view(B, pages_per)
        sl = torch.full((B,), ctx, device=dev, dtype=torch.int32)
        q = torch.randn((B, HQ, D), device=dev, dtype=torch.bfloat16)
        ws = torch.zeros(256 << 20, device=dev, dtype=torch.uint8)
        out = trtllm_batch_decode_with_kv_cache(q, kv, ws, bt, sl, ctx, bmm1_scale=D ** -0.5)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps * layers):
            trtllm_batch_decode_with_kv_cache(q, kv, ws, bt, sl, ctx, bmm1_scale=D ** -0.5, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms_layer = e0.elapsed_time(e1) / (reps * layers)
        nbytes = kv.numel() * 2
        del kv, ws
        torch.cuda.empty_cache()
        return {"impl": "flashinfer trtllm_batch_decode_with_kv_cache (trtllm-gen sm100a, library)",
                "ms_per_step": ms_layer * layers, "bytes_per_layer": nbytes,
                "hbm_gbs": nbytes / (ms_layer / 1e3) / 1e9}
    except Exception as exc:  # library comparator is optional
        log(f"flashinfer comparator unavailable: {exc!r}")
        return None


# ------------------------------------------------------------- CPU reference
def cpu_sample(ctx, steps, seed=0):
    """One q-head unit of the workload through the C oracle (tierkv's
    algorithm): prefill untimed, `steps` decode steps timed (path only, no
    recall metric).  Returns seconds per unit-step."""
    import numpy as np
    from oracle import oracle as O
    rng = np.random.default_rng(seed)
    d = D
    n_seg = -(-ctx // 8192)
    cen = rng.standard_normal((n_seg, 32, d)).astype(np.float32)
    seg = np.arange(ctx) // 8192
    keys = cen[seg, rng.integers(32, size=ctx)] + 0.5 * rng.standard_normal((ctx, d)).astype(np.float32)
    keys = _bf16(keys)
    vals = _bf16(rng.standard_normal((ctx, d)).astype(np.float32))
    eng = O.OracleEngine().prefill(keys, vals)
    qs = _bf16(cen.reshape(-1, d)[rng.integers(n_seg * 32, size=steps)] +
               0.25 * rng.standard_normal((steps, d)).astype(np.float32))
    nk = _bf16(rng.standard_normal((steps, d)).astype(np.float32))
    t0 = time.perf_counter()
    for t in range(steps):
        eng.decode_step(qs[t], nk[t], nk[t], with_recall=False)
    return (time.perf_counter() - t0) / steps


def _bf16(x):
    import numpy as np
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def _cpu_worker(args):
    ctx, steps, seed = args
    return cpu_sample(ctx, steps, seed)


def run_reference(a):
    """--impl reference: the reference algorithm on all host cores (one
    oracle unit per core, units are independent)."""
    import multiprocessing as mp
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    steps = max(1, a.steps)
    hq, hkv, d, n_layers = MODELS[a.model]
    layers = a.layers if a.layers > 0 else n_layers
    with mp.get_context("spawn").Pool(cores) as pool:
        t0 = time.perf_counter()
        per = pool.map(_cpu_worker, [(a.ctx, steps, s) for s in range(cores)])
        wall = time.perf_counter() - t0
    # per[i]: seconds per unit-step (one q-head at full context) on core i;
    # a token of one request is hq x layers unit-steps
    unit_steps_per_s = sum(1.0 / p for p in per)
    tok_s = unit_steps_per_s / (hq * layers)
    world = max(1, a.gpus)
    cfg_name = "configs[1]" if a.model == "llama3-8b" else "configs[4]"
    line = {"impl": "reference", "metric": METRIC,
            "value": tok_s, "unit": "tokens/s", "n_gpus": a.gpus, "steps": steps,
            # one step of the bounded sample: every core runs one unit-step
            "warmup": a.warmup, "ms_per_step": max(per) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            # the wave arm's config of the same arguments (same workload)
            "config": {"workload": f"{a.model}-shape {layers}-layer decode, {a.ctx // 1024}K ctx, "
                                   f"batch {a.batch} ({cfg_name})",
                       "model_shape": a.model, "batch_per_gpu": a.batch, "global_batch": a.batch * world,
                       "units_this_rank": a.batch * hkv, "ctx": a.ctx, "layers": layers,
                       "layer_buffers": min(a.layer_bufs, layers), "heads": f"{hq}q/{hkv}kv", "d": d,
                       "l2": "inputs larger than L2 (each layer buffer >> 126 MB, cycled)"},
            "full_step_ms_extrapolated": a.batch * world / tok_s * 1e3,
            "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": cores, "kind": "port",
                             "sample": f"{cores} x one q-head unit at {a.ctx} ctx, {steps} decode "
                                       f"steps each (prefill untimed); a step of the sample is {cores} "
                                       f"unit-steps in parallel; extrapolated x{hq} heads x{layers} layers"},
            "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- build (config 3)
def run_build(a, torch, dev, log):
    """configs[2]: prefill index build (segmented spherical k-means, finalize,
    store pack) of B x H_kv units at 122,880 and 262,144 tokens.  Throughput in
    tokens/s and GFLOP/s (Lloyd 11 x 2Lkd + seeding 2Ld(k-1) per segment,
    SURVEY 8(d)); assignment parity: sampled segments of unit 0 re-clustered by
    the CPU oracle (tierkv's algorithm, oracle/) must match bit-for-bit."""
    import numpy as np
    from oracle import oracle as O
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    cfg = EngineConfig()
    ic = cfg.index
    G = HQ // HKV
    U = a.batch * HKV
    rows = []
    for ctx in (122880, 262144):
        keys, vals, _ = gen_layer(torch, U, ctx, D, 11, dev)
        lay = WaveLayer(cfg, U, G, D, max_prefill=ctx, max_decode=64, store_dtype=torch.bfloat16)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lay.prefill(keys, vals)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        n_idx = ctx - ic.sink_tokens - ic.local_window
        flop = 0.0
        for s0 in range(0, n_idx, ic.segment_size):
            L = min(ic.segment_size, n_idx - s0)
            k = math.ceil(L / ic.centroid_ratio)
            flop += (ic.kmeans_iters + 1) * 2.0 * L * k * D + 2.0 * L * D * (k - 1)
        flop *= U
        # parity on sampled segments of unit 0 (first and last)
        segs = list(range(0, n_idx, ic.segment_size))
        sample = sorted({0, len(segs) - 1})
        kh = keys[0].cpu().numpy()
        tok = lay.store_tok[0].cpu().numpy()
        off = lay.cl_off[0].cpu().numpy()
        size = lay.cl_size[0].cpu().numpy()
        ok, checked = True, 0
        cid = 0
        for si, s0 in enumerate(segs):
            L = min(ic.segment_size, n_idx - s0)
            k = math.ceil(L / ic.centroid_ratio)
            if si in sample:
                base = ic.sink_tokens + s0
                ref = O.spherical_kmeans(kh[base:base + L], k, ic.kmeans_iters,
                                         np.random.SeedSequence([ic.rng_seed, 1, si]))
                mine = np.empty(L, np.int64)
                for c in range(k):
                    o, z = int(off[cid + c]), int(size[cid + c])
                    mine[tok[o:o + z] - base] = c
                ok &= bool(np.array_equal(mine, ref))
                checked += L
            cid += k
        rows.append({"ctx": ctx, "units": U, "tokens": U * n_idx, "seconds": dt,
                     "tokens_per_s": U * n_idx / dt, "gflop_per_s": flop / dt / 1e9,
                     "segments": U * len(segs), "parity_segments_checked": len(sample),
                     "parity_points_checked": checked, "assignment_parity": ok})
        log(f"build ctx={ctx}: {dt:.2f}s, parity={ok}")
        del keys, vals, lay
        torch.cuda.empty_cache()
    return {"metric": "prefill index build throughput (segmented spherical k-means), tokens/s",
            "impl": "wave-build", "unit": "tokens/s", "value": rows[0]["tokens_per_s"],
            "higher_is_better": True, "data": "synthetic",
            "config": {"workload": f"{a.model}-shape build, {a.batch} requests x {HKV} kv heads "
                                   "(configs[2])", "kmeans_iters": ic.kmeans_iters},
            "runs": rows}


# ----------------------------------------------------------- offload (config 4)
def run_offload(a, torch, dev, log, ctx=None, batch=None, layer_bufs=None, steps=None, warmup=None):
    """configs[3]: long context with the cluster store in pinned host memory
    and the wave buffer (HBM slot arena, cache_fraction of the blocks) on the
    device.  Reports the cumulative hit ratio (per cluster), miss
    bytes, and stall time = offload step time - the same step with the store
    resident in HBM (same data, same zones)."""
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    import types
    a = types.SimpleNamespace(**{**vars(a), **{k: v for k, v in dict(
        ctx=ctx, batch=batch, layer_bufs=layer_bufs, steps=steps, warmup=warmup).items() if v is not None}})
    G = HQ // HKV
    U = a.batch * HKV
    n_bufs = min(a.layer_bufs, a.layers)
    per_buf = math.ceil(a.layers / n_bufs)
    total_steps = a.warmup + a.steps
    cfg = EngineConfig()
    lay_o, lay_h, qpool, kpool = [], [], [], []
    t_build = 0.0
    for li in range(n_bufs):
        keys, vals, cen = gen_layer(torch, U, a.ctx, D, li, dev)
        if li == 0 and not a.no_cpu:
            keys0, vals0 = keys[0].cpu().numpy(), vals[0].cpu().numpy()
        for off, dst in ((True, lay_o), (False, lay_h)):
            lay = WaveLayer(cfg, U, G, D, max_prefill=a.ctx, max_decode=64, store_dtype=torch.bfloat16,
                            offload=off)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            lay.prefill(keys, vals)
            torch.cuda.synchronize()
            t_build += time.perf_counter() - t0
            dst.append(lay)
        qpool.append(gen_queries(torch, cen, G, total_steps * per_buf + OFF_PAR_STEPS, 7 + li))
        kpool.append(torch.randn((total_steps * per_buf + OFF_PAR_STEPS, 2, U, D), device=dev).bfloat16().float())
        del keys, vals, cen
        torch.cuda.empty_cache()
        log(f"layer buffer {li}: m={lay_o[-1].units[0].m} built (offload + hbm) {t_build:.1f}s")

    def run(layers, steps, start):
        use = [start * per_buf] * n_bufs
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            for l in range(a.layers):
                b = l % n_bufs
                j = use[b]
                use[b] += 1
                layers[b].launch_step(qpool[b][j], kpool[b][j, 0], kpool[b][j, 1])
                for s_ in layers[b].units:
                    s_.total += 1
                    s_.n_steady += 1
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / max(1, steps)

    run(lay_o, a.warmup, 0)
    run(lay_h, a.warmup, 0)
    c0 = [l.cache.counters.sum(0).clone() for l in lay_o]
    with ClockSampler(0) as clk:
        ms_o = run(lay_o, a.steps, a.warmup)
    ms_h = run(lay_h, a.steps, a.warmup)
    for l in lay_o + lay_h:
        l.check_status("offload bench")
    # oracle parity of the offload layer (outside the timed region): OFF_PAR_STEPS
    # more recorded steps of unit 0 of layer buffer 0 after everything it decoded
    par = None
    if not a.no_cpu:
        lay0, j0 = lay_o[0], total_steps * per_buf
        recs = []
        for j in range(j0, j0 + OFF_PAR_STEPS):
            lay0.launch_step(qpool[0][j], kpool[0][j, 0], kpool[0][j, 1])
            for s_ in lay0.units:
                s_.total += 1
                s_.n_steady += 1
            nr0 = int(lay0.nr[0])
            recs.append((j, lay0.out[0].double().cpu().numpy(), lay0.logden[0].cpu().numpy(),
                         lay0.rlist[0, :, :nr0].cpu().numpy()))
        lay0.check_status("offload parity steps")
        hist = [(qpool[0][j][0].double().cpu().numpy(), kpool[0][j, 0][0].cpu().numpy(),
                 kpool[0][j, 1][0].cpu().numpy()) for j in range(j0 + OFF_PAR_STEPS)]
        try:
            par = parity_sample(lay0, keys0, vals0, hist, recs, G, log)
        except Exception as exc:  # reported, never silently passed
            par = {"pass": False, "error": repr(exc)}
    dk = sum((l.cache.counters.sum(0) - c) for l, c in zip(lay_o, c0)).tolist()
    tot = sum(l.cache.counters.sum(0) for l in lay_o).tolist()
    hits, misses = tot[0], tot[1]
    # physical miss bytes: bf16 K+V rows of missed clusters read over the host link
    per_step_miss_blocks = dk[2] / cfg.block_size_bytes / a.steps
    bt = lay_o[0].cache.bt
    line = {"metric": "decode tokens/sec with host-KV offload (device-timed); hit ratio, miss bytes, stall", "impl": "wave-offload", "value": a.batch / (ms_o / 1e3), "unit": "tokens/s",
            "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_o, "higher_is_better": True,
            "data": "synthetic", "dtype": "bf16 KV / fp32 accumulate (fp64 scoring)",
            "config": {"workload": f"{a.model}-shape {a.layers}-layer decode, {a.ctx} ctx, batch {a.batch}, "
                                   "host-KV offload (configs[3])",
                       "layer_buffers": n_bufs, "cache_fraction": cfg.cache_fraction,
                       "host_store_gb_per_layer_buffer": 2 * U * lay_o[0].s_cap * D * 2 / 1e9},
            "cache": {"hit_ratio_cumulative": hits / max(1, hits + misses), "hits": hits, "misses": misses,
                      "hit_ratio_timed": dk[0] / max(1, dk[0] + dk[1]),
                      "miss_blocks_per_step": per_step_miss_blocks,
                      "miss_bytes_per_step_bf16": per_step_miss_blocks * bt * 2 * D * 2,
                      "evictions_per_step": dk[5] / a.steps, "admissions_per_step": dk[6] / a.steps,
                      "rejections_per_step": dk[7] / a.steps},
            "hbm_resident": {"ms_per_step": ms_h, "value": a.batch / (ms_h / 1e3)},
            "stall_ms_per_step": ms_o - ms_h,
            "host_link_gbs": per_step_miss_blocks * bt * 2 * D * 2 / ((ms_o - ms_h) / 1e3) / 1e9
            if ms_o > ms_h else None,
            "build_s": t_build, "clocks": clk.summary(), "parity_sample": par}
    del lay_o, lay_h, qpool, kpool
    return line


# ------------------------------------------------------------------- GPU arm
def _ptr(t):
    return t.data_ptr()


PAR_STEPS = 8  # recorded decode steps of the parity sample
OFF_PAR_STEPS = 2  # recorded decode steps of the offload leg's parity sample


def parity_sample(lay, keys0, vals0, history, recs, G, log):
    """Sampled oracle check of the benchmarked layer (outside the timed
    region): unit 0 of layer buffer 0 -- its 120K index (C64, sizes, members)
    bit-exact against the C oracle's prefill of the same keys, then the oracle
    replays every decode step that buffer saw (G heads) and the ordered
    retrieval list, output and log-denominator of each recorded step (`recs`:
    the last PAR_STEPS steps) must match (SURVEY 8c bars: ids bit-exact,
    rel-L2 <= 1e-5, |dlogden| <= 1e-5)."""
    import numpy as np
    from oracle import oracle as O
    t0 = time.perf_counter()
    e0 = O.OracleEngine(blas_threads=lay.blas_threads).prefill(keys0, vals0)
    ix = lay.index_arrays(0)
    m = e0.m
    index_ok = bool(lay.units[0].m == m and np.array_equal(ix["C64"], e0.centroids)
                    and np.array_equal(ix["sizes"], e0.sizes))
    for c in range(0, m, max(1, m // 64)):  # members of every 64th cluster (+ last)
        o, s = int(ix["offsets"][c]), int(ix["sizes"][c])
        index_ok &= bool(np.array_equal(ix["store_tok"][o:o + s], e0.members(c)))
    o, s = int(ix["offsets"][m - 1]), int(ix["sizes"][m - 1])
    index_ok &= bool(np.array_equal(ix["store_tok"][o:o + s], e0.members(m - 1)))
    orcs = [e0] + [e0.clone() for _ in range(G - 1)]
    at = {r[0]: r for r in recs}
    ids_ok, worst, dlog = True, 0.0, 0.0
    for j, (q, k, v) in enumerate(history):
        outs = [orcs[g].decode_step(q[g], k, v, with_recall=False) for g in range(G)]
        if j not in at:
            continue
        _, out, logden, rl = at[j]
        for g in range(G):
            o_ref, sm = outs[g]
            r_ref, _ = orcs[g].last_plan()
            ids_ok &= bool(rl.shape[1] == sm.r and np.array_equal(rl[g], r_ref))
            worst = max(worst, float(np.linalg.norm(out[g] - o_ref) / np.linalg.norm(o_ref)))
            dlog = max(dlog, abs(float(logden[g]) - sm.log_denominator))
    res = {"what": "unit 0 of layer buffer 0 (the benchmarked layer) vs the C oracle (tierkv's algorithm): "
                   f"index after prefill, then the last {len(recs)} of the decode steps it replayed",
           "m": m, "decode_steps_replayed": len(history), "decode_steps_compared": len(recs), "heads": G,
           "index_bit_exact": index_ok, "retrieval_ids_bit_exact": ids_ok,
           "max_rel_l2": worst, "max_abs_dlogden": dlog,
           "pass": bool(index_ok and ids_ok and worst <= 1e-5 and dlog <= 1e-5),
           "seconds": time.perf_counter() - t0}
    log(f"parity sample: {res}")
    return res


def run_decode(a, torch, dev, model, log, rank=0, world=1, batch=None, ctx=None, steps=None,
               warmup=None, layer_bufs=None, headline=True):
    """Decode throughput of one BASELINE config (configs[1] llama3-8b or
    configs[4] qwen2.5-7b): returns the JSON dict."""
    import ctypes
    from paper_2505_02922_b200 import EngineConfig, WaveLayer, _lib
    from paper_2505_02922_b200.wave import _stream
    hq, hkv, d, n_layers = MODELS[model]
    layers_n = a.layers if (headline and a.layers > 0) else n_layers
    batch = batch or a.batch
    ctx = ctx or a.ctx
    steps = steps if steps is not None else a.steps
    warmup = warmup if warmup is not None else a.warmup
    G = hq // hkv
    shard = None
    if headline and a.scaling == "strong" and world > 1:
        from paper_2505_02922_b200.parallel import shard_units
        shard = shard_units(batch, hkv, world, rank)  # contiguous block of the global units
        U = shard.count
    else:
        U = batch * hkv  # per-rank units (weak scaling: each rank serves `batch` requests)
    n_bufs = min(layer_bufs or a.layer_bufs, layers_n)
    per_buf = math.ceil(layers_n / n_bufs)
    total_steps = warmup + steps + 2  # + the per-op breakdown step
    cfg = EngineConfig()
    layers, qpool, kpool = [], [], []
    keys0 = vals0 = None
    t_build = 0.0
    for li in range(n_bufs):
        keys, vals, cen = gen_layer(torch, U, ctx, d, 1000 * rank + li, dev)
        if li == 0 and rank == 0 and not a.no_cpu:
            keys0, vals0 = keys[0].cpu().numpy(), vals[0].cpu().numpy()
        lay = WaveLayer(cfg, U, G, d, max_prefill=ctx, max_decode=64, store_dtype=torch.bfloat16,
                        split=a.split)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lay.prefill(keys, vals)
        torch.cuda.synchronize()
        t_build += time.perf_counter() - t0
        layers.append(lay)
        qpool.append(gen_queries(torch, cen, G, total_steps * per_buf + PAR_STEPS, 7 + li))
        kpool.append(torch.randn((total_steps * per_buf + PAR_STEPS, 2, U, d), device=dev).bfloat16().float())
        del keys, vals, cen
        torch.cuda.empty_cache()
        log(f"[{model}] layer buffer {li}: m={lay.units[0].m} build {t_build:.1f}s")
    use = [0] * n_bufs
    # N > 1: the path's one collective -- every layer's attention outputs are
    # gathered (NCCL all-gather over NVLink) on a side stream, overlapping the
    # next layers' kernels; shards are padded to the largest
    gmax = (-(-batch * hkv // world) if shard else U) if world > 1 else 0
    slabs = torch.zeros((layers_n, gmax, G, d), device=dev) if world > 1 else None
    gbufs = torch.empty((layers_n, world * gmax, G, d), device=dev) if world > 1 else None
    comm = torch.cuda.Stream(device=dev) if world > 1 else None
    gev = [torch.cuda.Event() for _ in range(layers_n)] if world > 1 else None

    def wave_step():
        main_s = torch.cuda.current_stream()
        for l in range(layers_n):
            b = l % n_bufs
            lay = layers[b]
            j = use[b]
            use[b] += 1
            lay.launch_step(qpool[b][j], kpool[b][j, 0], kpool[b][j, 1],
                            out=slabs[l, :U] if world > 1 else None)
            for s in lay.units:
                s.total += 1
                s.n_steady += 1
            if world > 1:
                gev[l].record(main_s)
                comm.wait_event(gev[l])
                with torch.cuda.stream(comm):
                    _all_gather_into(dist, gbufs[l], slabs[l])
        if world > 1:
            main_s.wait_stream(comm)

    import torch.distributed as dist
    for _ in range(warmup):
        wave_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(steps):
            wave_step()
        ev1.record()
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    if world > 1:
        t = torch.tensor([ms], device=dev if not _DRY else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
    for lay in layers:
        lay.check_status("bench")
    tok_step = batch if shard else batch * world  # tokens one step produces over all ranks
    value = tok_step / (ms / 1e3)
    multi = None
    if world > 1:
        # the gathers alone, serialized on the main stream (their cost if nothing overlapped them)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        g0.record()
        for l in range(layers_n):
            _all_gather_into(dist, gbufs[l], slabs[l])
        g1.record()
        torch.cuda.synchronize()
        cdev = dev if not _DRY else "cpu"
        counts = [torch.zeros(1, device=cdev, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(counts, torch.tensor([U], device=cdev, dtype=torch.int64))
        counts = [int(c) for c in counts]
        multi = {"scaling": "strong" if shard else "weak", "units_per_gpu": counts,
                 "load_imbalance": max(counts) / (sum(counts) / len(counts)),
                 "per_gpu_tokens_per_s": value / world,
                 "gather": {"collective": "NCCL all_gather_into_tensor per layer, side stream",
                            "bytes_per_step": int(gbufs.numel() * 4),
                            "ms_per_step_serialized": g0.elapsed_time(g1)},
                 "nccl_debug": os.environ.get("NCCL_DEBUG"),
                 "backend": "gloo (dry run: ranks share one GPU)" if _DRY else "nccl"}

    # ---- per-op device time inside one more step (events on the launch stream) ----
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(layers_n)]
    torch.cuda.synchronize()
    for l in range(layers_n):
        b_ = l % n_bufs
        lay = layers[b_]
        j = use[b_]
        use[b_] += 1
        q = qpool[b_][j]
        stream = ctypes.c_void_p(_stream())
        ev[l][0].record()
        _lib.check(lay.L.wk_append_tokens(ctypes.byref(lay._stv), _ptr(kpool[b_][j, 0]), _ptr(kpool[b_][j, 1]),
                                          lay.U, lay.d, lay.store_bf16, _ptr(lay.status), stream), "append")
        ev[l][1].record()
        sv = lay._step_view(q)
        _lib.check(lay.L.wk_score_topk(ctypes.byref(lay._ixv), ctypes.byref(sv), ctypes.byref(lay._zp), lay.U,
                                       max(s.m for s in lay.units), stream), "score_topk")
        ev[l][2].record()
        _lib.check(lay.L.wk_tripartite_attn(ctypes.byref(lay._ixv), ctypes.byref(lay._stv), ctypes.byref(sv),
                                            ctypes.byref(lay._zp), lay.U, lay.S, lay.store_bf16, stream), "attn")
        ev[l][3].record()
        for s_ in lay.units:
            s_.total += 1
            s_.n_steady += 1
    torch.cuda.synchronize()
    for lay in layers:
        lay.check_status("bench breakdown")
    t_app = sum(ev[l][0].elapsed_time(ev[l][1]) for l in range(layers_n)) / layers_n
    t_score = sum(ev[l][1].elapsed_time(ev[l][2]) for l in range(layers_n)) / layers_n
    t_attn = sum(ev[l][2].elapsed_time(ev[l][3]) for l in range(layers_n)) / layers_n

    # ---- sampled oracle parity of the benchmarked layer (outside the timed region) ----
    par = None
    if keys0 is not None and not a.no_cpu:
        # PAR_STEPS more decode steps of layer buffer 0 (untimed), each step's
        # unit-0 output / log-denominator / retrieval list recorded
        lay0 = layers[0]
        recs = []
        for _ in range(PAR_STEPS):
            j = use[0]
            use[0] += 1
            lay0.launch_step(qpool[0][j], kpool[0][j, 0], kpool[0][j, 1])
            for s_ in lay0.units:
                s_.total += 1
                s_.n_steady += 1
            nr0 = int(lay0.nr[0])
            recs.append((j, lay0.out[0].double().cpu().numpy(), lay0.logden[0].cpu().numpy(),
                         lay0.rlist[0, :, :nr0].cpu().numpy()))
        lay0.check_status("parity steps")
        hist = []
        for j in range(use[0]):
            hist.append((qpool[0][j][0].double().cpu().numpy(), kpool[0][j, 0][0].cpu().numpy(),
                         kpool[0][j, 1][0].cpu().numpy()))
        try:
            par = parity_sample(lay0, keys0, vals0, hist, recs, G, log)
        except Exception as exc:  # reported, never silently passed
            par = {"pass": False, "error": repr(exc)}

    # ---- algorithmic bytes: per layer, from the live zone counts ----
    elem = 2
    zs = {"n_steady": 0.0, "n_retrieved_tokens": 0.0, "n_retrieval_pieces": 0.0, "n_estimation_rows": 0.0,
          "m": 0.0}
    attn_bytes_l, score_bytes_l = [], []
    for lay in layers:
        cnt = lay.cnt.cpu().double()
        n_st = lay.st_n.cpu().double()
        mm = torch.tensor([s_.m for s_ in lay.units], dtype=torch.float64)
        attn_bytes_l.append(float((cnt[:, 1] + n_st).sum() * 2 * d * elem + cnt[:, 2].sum() * (d * 4 + 4)))
        score_bytes_l.append(float(mm.sum() * d * 4))
        zs["n_steady"] += float(n_st.mean()) / n_bufs
        zs["n_retrieved_tokens"] += float(cnt[:, 1].mean()) / n_bufs
        zs["n_retrieval_pieces"] += float(cnt[:, 3].mean()) / n_bufs
        zs["n_estimation_rows"] += float(cnt[:, 2].mean()) / n_bufs
        zs["m"] += float(mm.mean()) / n_bufs
    attn_bytes = sum(attn_bytes_l) / n_bufs
    score_bytes = sum(score_bytes_l) / n_bufs
    step_bytes = (attn_bytes + score_bytes) * layers_n
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback"
    achieved = attn_bytes / (t_attn / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp) and model == "llama3-8b":  # captured on the configs[1] workload only
        traffic = json.load(open(tp)).get("wk_tripartite_attn")

    # ---- full-attention comparators (same batch, heads, context, bf16 KV) ----
    fa_ms = None
    fa_steps = a.fa_steps if headline else min(a.fa_steps, 2)
    if fa_steps > 0:
        outs = torch.empty((U, G, d), device=dev)
        for l in range(layers_n):
            layers[l % n_bufs].full_attention(qpool[l % n_bufs][0], out=outs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(fa_steps):
            for l in range(layers_n):
                layers[l % n_bufs].full_attention(qpool[l % n_bufs][i], out=outs)
        e1.record()
        torch.cuda.synchronize()
        fa_ms = e0.elapsed_time(e1) / fa_steps
    fa_bytes_layer = sum(s_.store_fill + s_.n_steady for s_ in layers[0].units) * 2 * d * elem

    # ---- e2e: host buffers, copies inside the timed region ----
    e2e = None
    if not a.no_e2e and headline:
        hq_ = torch.empty((layers_n, U, G, d), dtype=torch.float32).pin_memory()
        hkv_buf = torch.empty((layers_n, 2, U, d), dtype=torch.float32).pin_memory()
        hout = torch.empty((layers_n, U, G, d), dtype=torch.float32).pin_memory()
        dq = torch.empty((layers_n, U, G, d), device=dev)
        dkv = torch.empty((layers_n, 2, U, d), device=dev)
        hq_.copy_(qpool[0][: layers_n].cpu() if qpool[0].shape[0] >= layers_n else hq_)
        hkv_buf.copy_(kpool[0][: layers_n].cpu() if kpool[0].shape[0] >= layers_n else hkv_buf.normal_())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k_e2e = max(1, min(steps, 5))
        # Pipelined host I/O: the q/k/v of a group of GR layers go up on an H2D stream
        # while earlier layers compute; a group's outputs come down on a D2H stream
        # once its last layer is done (overlapping the next group).  Stream waits /
        # event records only at group boundaries, so the kernels of a group stay
        # back to back (programmatic dependent launch).  The timed region ends when
        # the last output has landed.
        GR = max(1, a.e2e_group)
        main_s = torch.cuda.current_stream()
        up, down = torch.cuda.Stream(), torch.cuda.Stream()
        ngr = -(-layers_n // GR)
        ev_in = [torch.cuda.Event() for _ in range(ngr)]
        ev_out = [torch.cuda.Event() for _ in range(ngr)]
        dout = torch.empty((layers_n, U, G, d), device=dev)
        torch.cuda.synchronize()
        e0.record()
        for i in range(k_e2e):
            up.wait_stream(main_s)
            with torch.cuda.stream(up):
                for gi in range(ngr):
                    l0, l1 = gi * GR, min(layers_n, gi * GR + GR)
                    dq[l0:l1].copy_(hq_[l0:l1], non_blocking=True)
                    dkv[l0:l1].copy_(hkv_buf[l0:l1], non_blocking=True)
                    ev_in[gi].record(up)
            for gi in range(ngr):
                l0, l1 = gi * GR, min(layers_n, gi * GR + GR)
                main_s.wait_event(ev_in[gi])
                for l in range(l0, l1):
                    layers[l % n_bufs].launch_step(dq[l], dkv[l, 0], dkv[l, 1], out=dout[l])
                ev_out[gi].record(main_s)
                down.wait_event(ev_out[gi])
                with torch.cuda.stream(down):
                    hout[l0:l1].copy_(dout[l0:l1], non_blocking=True)
            main_s.wait_stream(down)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / k_e2e
        e2e = {"value": tok_step / (e2e_ms / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": int(hq_.numel() * 4 + hkv_buf.numel() * 4),
               "d2h_bytes_per_step": int(hout.numel() * 4), "ms_per_step": e2e_ms}
    del layers, qpool, kpool
    torch.cuda.empty_cache()
    fi = None
    if fa_steps > 0 and not a.no_flashinfer:
        fi = flashinfer_decode(torch, batch, hq, hkv, d, ctx, layers_n, max(3, fa_steps), log)

    fa_block = {"impl": "wk_full_attn (this repo, same kernel family reading every token)",
                "ms_per_step": fa_ms,
                "value": (tok_step / (fa_ms / 1e3)) if fa_ms else None,
                "speedup_wave_vs_full": (fa_ms / ms) if fa_ms else None,
                "bytes_per_layer": fa_bytes_layer,
                "hbm_gbs": (fa_bytes_layer * layers_n / (fa_ms / 1e3) / 1e9) if fa_ms else None}
    if fi:
        fi["speedup_wave_vs_full"] = fi["ms_per_step"] / ms
        fi["value"] = tok_step / (fi["ms_per_step"] / 1e3)
    read_peak = fi["hbm_gbs"] if fi else None
    cfg_name = "configs[1]" if model == "llama3-8b" else "configs[4]"
    return {
        "metric": METRIC,
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if shard else "weak", "multi_gpu": multi,
        "vs_baseline": None, "dtype": "bf16 KV / fp32 accumulate (fp64 scoring)", "data": "synthetic",
        "config": {"workload": f"{model}-shape {layers_n}-layer decode, {ctx // 1024}K ctx, batch {batch} ({cfg_name})",
                   "model_shape": model,
                   "batch_per_gpu": batch if not shard else None, "global_batch": tok_step,
                   "units_this_rank": U, "ctx": ctx, "layers": layers_n,
                   "layer_buffers": n_bufs, "heads": f"{hq}q/{hkv}kv", "d": d,
                   "l2": "inputs larger than L2 (each layer buffer >> 126 MB, cycled)"},
        "full_attention": fi or fa_block,
        "full_attention_own_kernel": fa_block,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "wk_tripartite_attn (attend_v6 + att6_merge, bf16 store)",
                     "bytes_per_launch": attn_bytes, "ms_per_launch": t_attn,
                     "read_peak_demonstrated": read_peak,
                     "frac_vs_read_peak": (achieved / read_peak) if read_peak else None,
                     "read_peak_source": "flashinfer full-attention decode on the same box, same run "
                                         "(a read-only stream; the copy peak counts read+write)"},
        "step_roofline": {"bytes_per_step": step_bytes, "achieved": step_bytes / (ms / 1e3) / 1e9,
                          "frac": step_bytes / (ms / 1e3) / 1e9 / peak,
                          "frac_vs_read_peak": (step_bytes / (ms / 1e3) / 1e9 / read_peak) if read_peak else None,
                          "what": "HBM bytes touched per decode step (C32 scan + steady/retrieved K,V "
                                  "+ estimation value sums) / device step time"},
        "breakdown_ms_per_layer": {"append": t_app, "score_topk": t_score, "tripartite_attn": t_attn,
                                   "score_scan_gbs": score_bytes / (t_score / 1e3) / 1e9},
        "zone_stats_per_unit": zs,
        "build_s": t_build,
        "parity_sample": par,
        "e2e": e2e,
        "clocks": clk.summary(),
        "gpu_launches": steps * layers_n * LAUNCHES_PER_LAYER,
    }


_DRY = False  # world > visible GPUs: a 1-GPU dry run of the multi-rank path over gloo


def _all_gather_into(dist, dst, src):
    """The per-layer output gather (NCCL all-gather; host-staged on gloo dry runs)."""
    if not _DRY:
        dist.all_gather_into_tensor(dst, src)
        return
    parts = [torch_mod().empty_like(src, device="cpu") for _ in range(dist.get_world_size())]
    dist.all_gather(parts, src.cpu())
    dst.copy_(torch_mod().cat(parts).to(dst.device))


def torch_mod():
    import torch
    return torch


def _compact(line, keys):
    return {k: line.get(k) for k in keys}


def main():
    global HQ, HKV, D
    a = parse()
    HQ, HKV, D, n_layers = MODELS[a.model]
    if a.layers <= 0:
        a.layers = n_layers
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())  # (ranks share a GPU only in 1-GPU dry runs)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    global _DRY
    _DRY = world > torch.cuda.device_count()
    if world > 1 and _DRY:
        dist.init_process_group("gloo")  # NCCL refuses two ranks on one GPU
    elif world > 1:
        if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
            os.environ["NCCL_DEBUG"] = "INFO"  # the rank / transport lines on stderr
        dist.init_process_group("nccl", device_id=dev)
    log = lambda *x: print(*x, file=sys.stderr, flush=True) if rank == 0 else None
    if a.offload:
        print(json.dumps(run_offload(a, torch, dev, log)), flush=True)
        return
    if a.build:
        print(json.dumps(run_build(a, torch, dev, log)), flush=True)
        return
    line = run_decode(a, torch, dev, a.model, log, rank=rank, world=world)

    # ---- CPU baseline (oracle port of tierkv, one host core) ----
    cpu = None
    if rank == 0 and not a.no_cpu and a.cpu_steps > 0:
        t_unit = cpu_sample(a.ctx, a.cpu_steps)
        cpu_tok = 1.0 / (t_unit * HQ * a.layers)
        cpu = {"value": cpu_tok, "unit": "tokens/s", "cores": 1, "kind": "port",
               "sample": f"one q-head unit at {a.ctx} ctx, {a.cpu_steps} decode steps (prefill "
                         f"untimed, no recall metric), {t_unit * 1e3:.2f} ms/unit-step, "
                         f"extrapolated x{HQ} heads x{a.layers} layers",
               "host": host_info()}
    line["cpu_baseline"] = cpu

    # ---- the other BASELINE configs, reduced, in front of the driver (1 GPU only) ----
    if world == 1 and not a.no_extras:
        extras = {}
        for name, fn in (("qwen", lambda: _compact(
                              run_decode(a, torch, dev, "qwen2.5-7b", log, steps=5, warmup=3, headline=False),
                              ("value", "ms_per_step", "config", "full_attention", "full_attention_own_kernel",
                               "roofline", "step_roofline", "breakdown_ms_per_layer", "zone_stats_per_unit",
                               "clocks", "parity_sample"))),
                         ("build", lambda: run_build(a, torch, dev, log)),
                         ("offload", lambda: run_offload(a, torch, dev, log, ctx=1048576, batch=4, layer_bufs=2,
                                                         steps=3, warmup=2)),
                         ("index_update", lambda: run_update_cost(a, torch, dev, log, step_ms=line["ms_per_step"]))):
            try:
                t0 = time.perf_counter()
                extras[name] = fn()
                extras[name]["wall_s"] = time.perf_counter() - t0
            except Exception as exc:  # an extra leg never hides the headline
                extras[name] = {"error": repr(exc)}
            torch.cuda.empty_cache()
        line["configs_other"] = extras
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_update_cost(a, torch, dev, log, step_ms=None):
    """The decode-time index update at the configs[1] scale (ClusterIndex.update,
    index.py:168-186): one 120K layer of B x H_kv units decodes until its buffer
    holds update_segment + local_window tokens, then one update (k-means of the
    oldest 1,024 buffer tokens of every unit, finalize + pack, buffer shift) is
    timed.  Each layer updates once per 1,024 steps, so the amortised cost per
    decode step is layers x update / 1,024."""
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    cfg = EngineConfig()
    ic = cfg.index
    hq, hkv, d, n_layers = MODELS["llama3-8b"]
    U, G = a.batch * hkv, hq // hkv
    keys, vals, cen = gen_layer(torch, U, a.ctx, d, 5, dev)
    lay = WaveLayer(cfg, U, G, d, max_prefill=a.ctx, max_decode=2 * ic.update_segment, store_dtype=torch.bfloat16)
    lay.prefill(keys, vals)
    del keys, vals
    torch.cuda.empty_cache()
    s0 = lay.units[0]
    need = ic.update_segment + ic.local_window - (s0.n_steady - s0.n_sink)
    qs = gen_queries(torch, cen, G, 4, 3)
    kv = torch.randn((2, U, d), device=dev).bfloat16().float()
    for i in range(max(0, need)):
        lay.decode(qs[i % 4], kv[0], kv[1], allow_update=False)
    torch.cuda.synchronize()
    assert lay.needs_update()
    m0 = s0.m
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    lay.maybe_update()
    e1.record()
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - t0) * 1e3
    lay.check_status("index update")
    per_step = n_layers * wall_ms / ic.update_segment
    log(f"index update: {wall_ms:.1f} ms for {U} units (+{s0.m - m0} clusters each)")
    return {"what": "one ClusterIndex.update of a 120K layer (every unit: k-means of the oldest "
                    f"{ic.update_segment} buffer tokens, k={s0.m - m0}, finalize + pack, buffer shift)",
            "units": U, "update_ms_wall": wall_ms, "update_ms_device": e0.elapsed_time(e1),
            "decode_steps_between_updates": ic.update_segment,
            "amortised_ms_per_step": per_step,
            "fraction_of_step": (per_step / step_ms) if step_ms else None}


def host_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
            "oracle_threads": 1}


if __name__ == "__main__":
    main()
