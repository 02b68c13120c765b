"""Cycle split of the k-means++ seeding kernel (km_seed_v2): per segment, the
centre-distance bounds, the min-distance row pass, and the sequential fp32
cumsum + draw, from a -DWK_SEED_TIMING build into build_seedtiming/ (the
product library is untouched).  Workload: one 120K-context layer of the bench."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2505_02922_b200 import _build
HERE = os.path.dirname(os.path.abspath(_build.__file__))
_build.LIB = os.path.join(HERE, "build_seedtiming", "libwavekv_timing.so")
_build.OBJ = os.path.join(HERE, "build_seedtiming")
os.environ["WK_EXTRA_NVCC_FLAGS"] = "-DWK_SEED_TIMING"
os.makedirs(_build.OBJ, exist_ok=True)
_build.build(force=True)
from paper_2505_02922_b200 import _lib
_lib.LIB_PATH = _build.LIB
import time, torch
import bench
from paper_2505_02922_b200 import EngineConfig, WaveLayer
dev = torch.device("cuda")
U = int(os.environ.get("U", 128))
keys, vals, _ = bench.gen_layer(torch, U, 122880, 128, 11, dev)
lay = WaveLayer(EngineConfig(), U, 4, 128, max_prefill=122880, max_decode=64, store_dtype=torch.bfloat16)
torch.cuda.synchronize(); t0 = time.perf_counter()
lay.prefill(keys, vals)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
L = _lib.lib()
L.wk_seed_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
n = U * 15
ts = np.zeros(8192 * 4, np.int64)
assert L.wk_seed_timing(ts.ctypes.data, ts.size) == 0
ts = ts[:n * 4].reshape(n, 4)
tot = ts.sum(1)
print(f"build {dt:.3f} s ({U * 122812 / dt / 1e6:.1f} M tok/s); per-segment seeding cycles median {np.median(tot):.0f}")
for i, nm in enumerate(["centre + bounds (ccd)", "row compaction", "row pass (active rows)", "cumsum + draw"]):
    print(f"  {nm:22s} median {np.median(ts[:, i]):10.0f}  ({np.median(ts[:, i] / tot) * 100:.1f}%)")

