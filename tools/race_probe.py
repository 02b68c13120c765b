"""Determinism probe: re-run score_topk + tripartite_attn of one decode step
(no append) on the default bench layer many times and compare every output
bitwise with the first run (select outputs, estimation logits, attention)."""
import ctypes, os, sys
sys.path.insert(0, ".")
import torch
import bench
from paper_2505_02922_b200 import EngineConfig, WaveLayer, _lib
from paper_2505_02922_b200.wave import _stream
dev = torch.device("cuda")
U, G, d, n = int(os.environ.get("U", 128)), 4, 128, 122880
keys, vals, cen = bench.gen_layer(torch, U, n, d, 0, dev)
lay = WaveLayer(EngineConfig(), U, G, d, max_prefill=n, max_decode=64, store_dtype=torch.bfloat16)
lay.prefill(keys, vals)
del keys, vals
qs = bench.gen_queries(torch, cen, G, 8, 7)
kv = torch.randn((8, 2, U, d), device=dev).bfloat16().float()
for i in range(4):
    lay.launch_step(qs[i], kv[i, 0], kv[i, 1])
    for s in lay.units:
        s.total += 1
        s.n_steady += 1
torch.cuda.synchronize()
L = lay.L
q = qs[5]
def run():
    sv = lay._step_view(q)
    st = ctypes.c_void_p(_stream())
    _lib.check(L.wk_score_topk(ctypes.byref(lay._ixv), ctypes.byref(sv), ctypes.byref(lay._zp), lay.U,
                               max(s.m for s in lay.units), st), "score_topk")
    _lib.check(L.wk_tripartite_attn(ctypes.byref(lay._ixv), ctypes.byref(lay._stv), ctypes.byref(sv),
                                    ctypes.byref(lay._zp), lay.U, lay.S, lay.store_bf16, st), "attn")
    torch.cuda.synchronize()
    lay.check_status("probe")
    return {k: getattr(lay, k).clone() for k in ("scores", "cnt", "rtok_row", "ru_ids", "eu_ids", "eu_mask",
                                                  "eu_x", "eu_sz", "out", "logden")}
ref = run()
cnt = ref["cnt"].view(U, 4).long()
bad = {}
for it in range(int(os.environ.get("ITERS", 30))):
    r = run()
    for k, v in r.items():
        a, b = ref[k], v
        diff = (a.view(-1) != b.view(-1)) & ~(torch.isnan(a.view(-1).float()) & torch.isnan(b.view(-1).float())) if a.is_floating_point() else (a.view(-1) != b.view(-1))
        nd = int(diff.sum())
        if nd:
            bad.setdefault(k, []).append(nd)
print("live counts unit0", cnt[0].tolist(), "eu_cap", lay.eu_cap)
print("nondeterministic outputs:", {k: (len(v), max(v)) for k, v in bad.items()} or "none")
if "out" in bad:
    o = torch.stack([run()["out"] for _ in range(5)])
    dev_ = (o - ref["out"]).abs().flatten(1).max(1).values
    print("max |out - out0| per rerun", dev_.tolist())
    per_u = (o[0] - ref["out"]).abs().view(U, -1).max(1).values
    print("units differing:", torch.nonzero(per_u).flatten().tolist()[:40])
