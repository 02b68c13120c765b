"""Phase timeline of select_v6 on the bench workload (globaltimer marks)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_2505_02922_b200 import EngineConfig, WaveLayer, _lib  # noqa: E402

dev = torch.device("cuda")
U, G, D, n = 128, 4, 128, 122880
keys, vals, cen = bench.gen_layer(torch, U, n, D, 0, dev)
lay = WaveLayer(EngineConfig(), U, G, D, max_prefill=n, max_decode=64,
                score_mode=int(os.environ.get("SCORE_MODE", "1")))
lay.prefill(keys, vals)
del keys, vals
q = bench.gen_queries(torch, cen, G, 4, 7)
kv = torch.randn((4, 2, U, D), device=dev).bfloat16().float()
L = _lib.lib()
for i in range(3):
    lay.launch_step(q[i], kv[i, 0], kv[i, 1])
torch.cuda.synchronize()
L.wk_debug_select_prof(1)
lay.launch_step(q[3], kv[3, 0], kv[3, 1])
torch.cuda.synchronize()
L.wk_debug_select_prof(0)
out = np.zeros((4096, 16), np.int64)
L.wk_debug_select_timing(out.ctypes.data_as(ctypes.c_void_p), 4096)
o = out[:U * G].astype(np.float64)
t0 = o[:, 0].min()
names = ["start", "histogram", "bucket lists", "tau done", "cand/pass D", "sort+xpos", "exact",
         "winners+compact", "clump sort", "outputs", "pre-union (last)", "union done"]
print("mark (us from first CTA start): median / max")
for i in range(12):
    v = o[:, i]
    v = v[v > 0]
    if len(v):
        print(f"{i:2d} {names[i]:18s} med {np.median(v - t0) / 1e3:8.1f} max {np.max(v - t0) / 1e3:8.1f} n={len(v)}")
d = o[:, 1:10] - o[:, 0:9]
for i, nm in ((15, "union pass1+xchg"), (13, "pass2 word loop start"), (14, "pass2 word loop end")):
    v = o[:, i]
    if (v > 1e9).any():
        print(f"{i} {nm} med {np.median(v[v > 1e9] - t0) / 1e3:8.1f} max {np.max(v[v > 1e9] - t0) / 1e3:8.1f}")
print("per-phase median durations (us):", np.round(np.median(d, axis=0) / 1e3, 2))
print("ncand/nx/nband_e median", np.median(o[:, 12]), np.median(o[:, 13]), np.median(o[:, 14]),
      "max", o[:, 12].max(), o[:, 13].max(), o[:, 14].max())
