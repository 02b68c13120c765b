import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2505_02922_b200 import EngineConfig, WaveLayer
dev = torch.device("cuda")
U, G, d, n = 128, 4, 128, 65536
keys, vals, cen = bench.gen_layer(torch, U, n, d, 0, dev)
lay = WaveLayer(EngineConfig(), U, G, d, max_prefill=n, max_decode=64, store_dtype=torch.bfloat16)
lay.prefill(keys, vals)
torch.cuda.synchronize()
qs = bench.gen_queries(torch, cen, G, 8, 7)
kv = torch.randn((8, 2, U, d), device=dev).bfloat16().float()
for i in range(3):
    try:
        lay.launch_step(qs[i], kv[i, 0], kv[i, 1])
        torch.cuda.synchronize()
        print("step", i, "ok", lay.cnt[:2].tolist())
    except Exception as e:
        print("step", i, "error", repr(e)[:300]); break
