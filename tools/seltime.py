import sys, os, ctypes, numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2505_02922_b200 import EngineConfig, WaveLayer, _lib
dev = torch.device('cuda')
U, G, D, n = 128, 4, 128, 122880
keys, vals, cen = bench.gen_layer(torch, U, n, D, 0, dev)
lay = WaveLayer(EngineConfig(), U, G, D, max_prefill=n, max_decode=64)
lay.prefill(keys, vals); del keys, vals
q = bench.gen_queries(torch, cen, G, 4, 7)
kv = torch.randn((4, 2, U, D), device=dev).bfloat16().float()
for i in range(3):
    lay.launch_step(q[i], kv[i, 0], kv[i, 1])
torch.cuda.synchronize()
L0 = _lib.lib(); z = np.zeros((4096,16), np.int64); L0.wk_debug_select_timing(z.ctypes.data_as(ctypes.c_void_p), 0)
lay.launch_step(q[3], kv[3, 0], kv[3, 1]); torch.cuda.synchronize()
L = _lib.lib()
out = np.zeros((4096, 16), np.int64)
L.wk_debug_select_timing(out.ctypes.data_as(ctypes.c_void_p), 4096)
o = out[:U * G].astype(np.float64)
t0 = o[:, 0].min()
print("phase end times relative to first CTA start (us): median / max over CTAs")
names = ['start','passA','passB','passC+tau','passD','exact','order','marks','-','last-CTA','union']
for i in range(11):
    col = o[:, i]
    v = col[col > 0]
    if len(v): print(f"{i:2d} {names[i]:12s} med {np.median(v - t0)/1e3:8.1f}  max {np.max(v - t0)/1e3:8.1f}  n={len(v)}")
d = o[:, 1:9] - o[:, 0:8]
print("per-phase durations median (us):", np.round(np.median(d, axis=0) / 1e3, 1))
print("band sizes r/e: median", np.median(o[:, 12]), np.median(o[:, 13]), "max", o[:, 12].max(), o[:, 13].max())
print("bucket lists n1/n2 median", np.median(o[:,14]), np.median(o[:,15]), "max", o[:,14].max(), o[:,15].max())
