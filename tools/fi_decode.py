"""Full-attention decode comparator: flashinfer trtllm-gen (sm100a cubins)
over the same Llama-3-8B-shaped workload (B=16, 32q/8kv, d=128, 120K ctx,
bf16 paged KV).  Prints ms per layer-call and achieved GB/s."""
import sys
import time

import torch


def run(B=16, HQ=32, HKV=8, D=128, ctx=122880, page=64, reps=20):
    from flashinfer.decode import trtllm_batch_decode_with_kv_cache
    dev = torch.device("cuda")
    pages_per = ctx // page
    npages = B * pages_per
    # HND layout: [num_pages, 2, HKV, page, D]
    kv = torch.randn((npages, 2, HKV, page, D), device=dev, dtype=torch.bfloat16)
    bt = torch.arange(npages, device=dev, dtype=torch.int32).view(B, pages_per)
    sl = torch.full((B,), ctx, device=dev, dtype=torch.int32)
    q = torch.randn((B, HQ, D), device=dev, dtype=torch.bfloat16)
    ws = torch.zeros(256 << 20, device=dev, dtype=torch.uint8)
    t0 = time.time()
    out = trtllm_batch_decode_with_kv_cache(q, kv, ws, bt, sl, ctx, bmm1_scale=D ** -0.5)
    torch.cuda.synchronize()
    print(f"first call (incl. JIT) {time.time() - t0:.1f}s", file=sys.stderr)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        trtllm_batch_decode_with_kv_cache(q, kv, ws, bt, sl, ctx, bmm1_scale=D ** -0.5, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gb = kv.numel() * 2 / 1e9
    return ms, gb / (ms / 1e3)


if __name__ == "__main__":
    ms, gbs = run()
    print(f"flashinfer trtllm decode: {ms:.3f} ms/layer, {gbs:.0f} GB/s, 32 layers = {32 * ms:.2f} ms/step")
