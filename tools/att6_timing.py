"""attend_v6 producer / consumer split: per warp, cycles waiting on the ring
barriers vs total (a -DATT6_TIMING build into build_a6timing/; the product
library is untouched).  Workload: one 120K-context layer of the bench."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2505_02922_b200 import _build
HERE = os.path.dirname(os.path.abspath(_build.__file__))
VAR = os.environ.get("A6_VARIANT", "")
_build.LIB = os.path.join(HERE, "build_a6timing", "libwavekv_timing.so")
_build.OBJ = os.path.join(HERE, "build_a6timing")
os.environ["WK_EXTRA_NVCC_FLAGS"] = " ".join(["-DATT6_TIMING"] + ["-D" + v for v in VAR.split()])
os.makedirs(_build.OBJ, exist_ok=True)
_build.build(force=True)
from paper_2505_02922_b200 import _lib
_lib.LIB_PATH = _build.LIB
import torch
import bench
from paper_2505_02922_b200 import EngineConfig, WaveLayer
dev = torch.device("cuda")
U, G, d, n = 128, 4, 128, 122880
keys, vals, cen = bench.gen_layer(torch, U, n, d, 0, dev)
lay = WaveLayer(EngineConfig(), U, G, d, max_prefill=n, max_decode=64, store_dtype=torch.bfloat16)
lay.prefill(keys, vals)
qs = bench.gen_queries(torch, cen, G, 8, 7)
kv = torch.randn((8, 2, U, d), device=dev).bfloat16().float()
for i in range(6):
    lay.launch_step(qs[i], kv[i, 0], kv[i, 1])
torch.cuda.synchronize()
L = _lib.lib()
L.wk_att6_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
ts = np.zeros(148 * 16 * 4, np.int64)
assert L.wk_att6_timing(ts.ctypes.data, ts.size) == 0
ts = ts.reshape(148, 16, 4)
NP = int(os.environ.get("NP", 4))
for nm, sl in (("producers", slice(0, NP)), ("consumers", slice(NP, 16))):
    w, tot = ts[:, sl, 0].astype(float), ts[:, sl, 1].astype(float)
    ok = tot > 0
    print(f"{nm}: total cycles median {np.median(tot[ok]):.0f}, waiting {np.median(w[ok] / tot[ok]) * 100:.1f}% (median)")
