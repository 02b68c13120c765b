"""Offload vs in-HBM layer on identical keys: the cluster store (K, V, token
ids, offsets, sizes) of every unit must be byte-identical, and the decode
outputs identical up to the chunking of the retrieval zone."""
import os, sys
sys.path.insert(0, ".")
import torch
import bench
from paper_2505_02922_b200 import EngineConfig, WaveLayer
dev = torch.device("cuda")
U, G, d, n = int(os.environ.get("U", 4)), 4, 128, int(os.environ.get("N", 1048576))
keys, vals, cen = bench.gen_layer(torch, U, n, d, 0, dev)
lays = []
for off in (False, True):
    lay = WaveLayer(EngineConfig(), U, G, d, max_prefill=n, max_decode=64, offload=off)
    lay.prefill(keys, vals)
    torch.cuda.synchronize()
    lays.append(lay)
a, b = lays
for u in range(U):
    f = a.units[u].store_fill
    res = {}
    for nm in ("store_k", "store_v", "store_tok", "cl_off", "cl_size"):
        x, y = getattr(a, nm)[u], getattr(b, nm)[u]
        if nm.startswith("store"):
            x, y = x[:f], y[:f]
        else:
            x, y = x[:a.units[u].m], y[:b.units[u].m]
        x, y = x.cpu(), y.cpu()
        ne = (x.view(torch.int16 if x.dtype == torch.bfloat16 else x.dtype) != y.view(torch.int16 if y.dtype == torch.bfloat16 else y.dtype))
        ne = ne.reshape(ne.shape[0], -1).any(1) if ne.dim() > 1 else ne
        res[nm] = int(ne.sum())
        if nm == "store_k" and res[nm]:
            rows = torch.nonzero(ne).flatten()
            print("  unit", u, "differing K rows", rows[:20].tolist(), "of", f)
    print("unit", u, "fill", f, "differing rows/entries:", res)
qs = bench.gen_queries(torch, cen, G, 3, 7)
kv = torch.randn((3, 2, U, d), device=dev).bfloat16().float()
for t in range(3):
    outs = [l.decode(qs[t], kv[t, 0], kv[t, 1])[0].clone() for l in lays]
    rel = ((outs[0] - outs[1]).flatten(1).norm(dim=1) / outs[0].flatten(1).norm(dim=1))
    print("step", t, "offload vs HBM rel diff per unit:", [f"{v:.2e}" for v in rel.tolist()])
