"""Small index build (U units at 120K) for profiling the k-means kernels."""
import os
import sys
import time

import torch

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_2505_02922_b200 import EngineConfig, WaveLayer  # noqa: E402

U = int(os.environ.get("U", "16"))
dev = torch.device("cuda")
keys, vals, _ = bench.gen_layer(torch, U, 122880, 128, 0, dev)
lay = WaveLayer(EngineConfig(), U, 4, 128, max_prefill=122880, max_decode=64)
torch.cuda.synchronize()
t0 = time.perf_counter()
lay.prefill(keys, vals)
torch.cuda.synchronize()
print(f"U={U} build {time.perf_counter() - t0:.3f}s")
