"""Phase timeline of select_v6 (clock64 marks of a -DWK_SEL_TIMING build of
libwavekv into build_timing/; the product library is untouched): median
cycles spent between consecutive marks over the CTAs of one launch on the
default bench layer."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2505_02922_b200 import _build
HERE = os.path.dirname(os.path.abspath(_build.__file__))
VAR = os.environ.get("SEL_VARIANT", "")  # extra -D flags of an experiment build
tag = "_".join(v.lower() for v in VAR.split())
_build.LIB = os.path.join(HERE, "build_timing" + tag, "libwavekv_timing.so")
_build.OBJ = os.path.join(HERE, "build_timing" + tag)
os.environ["WK_EXTRA_NVCC_FLAGS"] = " ".join(["-DWK_SEL_TIMING"] + ["-D" + v for v in VAR.split()])
os.makedirs(_build.OBJ, exist_ok=True)
_build.build(force=not os.path.exists(_build.LIB))
from paper_2505_02922_b200 import _lib
_lib.LIB_PATH = _build.LIB
import torch
import bench
from paper_2505_02922_b200 import EngineConfig, WaveLayer
dev = torch.device("cuda")
U, G, d, n = int(os.environ.get("U", 128)), 4, 128, 122880
keys, vals, cen = bench.gen_layer(torch, U, n, d, 0, dev)
lay = WaveLayer(EngineConfig(), U, G, d, max_prefill=n, max_decode=64, store_dtype=torch.bfloat16)
lay.prefill(keys, vals)
qs = bench.gen_queries(torch, cen, G, 8, 7)
kv = torch.randn((8, 2, U, d), device=dev).bfloat16().float()
for i in range(6):
    lay.launch_step(qs[i], kv[i, 0], kv[i, 1])
torch.cuda.synchronize()
L = _lib.lib()
L.wk_sel_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
ts = np.zeros(U * G * 16, np.int64)
assert L.wk_sel_timing(ts.ctypes.data, ts.size) == 0
ts_all = ts.reshape(U * G, 16)
ts = ts_all[:, :13]
d_ = np.diff(ts, axis=1)
names = ["passA+reduce", "hist+buckets", "passD classify", "rank cands", "exact round", "winners..outputs",
         "cluster sync 1", "union stage+count", "cl.sync+bases", "emit", "cl.sync 2", "est logits"]
tot = np.median(ts[:, 12] - ts[:, 0])
print(f"U={U}: median CTA cycles {tot:.0f} ({tot / 1.9e3:.1f} us at 1.9 GHz)")
for i, nm in enumerate(names):
    print(f"  {nm:18s} median {np.median(d_[:, i]):8.0f}  p90 {np.percentile(d_[:, i], 90):8.0f}")
print("emit detail (thread 0): prefixes", np.median(ts_all[:, 13] - ts_all[:, 9]),
      " word loop", np.median(ts_all[:, 14] - ts_all[:, 13]), " to cl.sync 2", np.median(ts_all[:, 10] - ts_all[:, 14]))
