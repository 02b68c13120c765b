"""Probe: per-layer GPU time and CPU enqueue time of launch_step with unit-group
splitting (split=k) vs one fused launch; variant 'seq' runs the groups'
planning on the main stream (no overlap) to separate launch-shape effects
from stream concurrency."""
import sys, time
import torch
sys.path.insert(0, ".")
import bench
from paper_2505_02922_b200 import EngineConfig, WaveLayer

dev = torch.device("cuda")
U, G, d, n = 128, 4, 128, 122880
keys, vals, cen = bench.gen_layer(torch, U, n, d, 0, dev)
res = {}
for sp in (1, 2, 4):
    lay = WaveLayer(EngineConfig(), U, G, d, max_prefill=n, max_decode=256, store_dtype=torch.bfloat16, split=sp)
    lay.prefill(keys, vals)
    qs = bench.gen_queries(torch, cen, G, 60, 7)
    kv = torch.randn((60, 2, U, d), device=dev).bfloat16().float()
    for mode in (["main"] if sp == 1 else ["side", "seq"]):
        if mode == "seq":
            lay._side = torch.cuda.current_stream()
            lay.__dict__.pop("_ev", None)
        for i in range(5):
            lay.launch_step(qs[i], kv[i, 0], kv[i, 1])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        for i in range(5, 45):
            lay.launch_step(qs[i], kv[i, 0], kv[i, 1])
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        print(f"split={sp} {mode}: gpu {e0.elapsed_time(e1) / 40 * 1e3:.1f} us/layer, cpu enqueue {(t1 - t0) / 40 * 1e6:.1f} us/layer", flush=True)
    del lay
    torch.cuda.empty_cache()
