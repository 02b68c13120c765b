"""Function-level spherical k-means on the GPU (tierkv clustering.py:66-101).

``spherical_kmeans(keys, k, iters, seed)`` keeps the reference signature and
returns the same int64 assignment bit-for-bit (same seeds, same tie-breaking).
It runs the batched segment kernels of libwavekv.so on a single segment; the
engine uses them batched over every segment of every unit.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import ConfigError

_BLAS_THREADS = 1


def set_blas_threads(n: int):
    """OPENBLAS_NUM_THREADS of the reference run whose bits are reproduced
    (only chunk-tail rows of large sgemv/dgemv calls depend on it)."""
    global _BLAS_THREADS
    _BLAS_THREADS = int(n)


def blas_threads() -> int:
    return _BLAS_THREADS


def _seed_words(seed):
    st = np.random.PCG64(seed).state["state"]
    s, i = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return (s >> 64, s & m, i >> 64, i & m)


def spherical_kmeans(keys, k: int, iters: int, seed, device="cuda", threads=None) -> np.ndarray:
    keys_np = np.asarray(keys, dtype=np.float32)
    if keys_np.ndim != 2:
        raise ConfigError("keys must be 2-D")
    n, d = keys_np.shape
    k = int(k)
    if k < 1:
        raise ConfigError(f"k must be >= 1, got {k}")
    if k > n:
        raise ConfigError(f"k={k} exceeds number of keys n={n}")
    if k == 1:
        return np.zeros(n, dtype=np.int64)
    if d > 256:
        raise ConfigError(f"head dim {d} unsupported (d <= 256)")
    if d % 4:
        # the kernels stream rows as float4: zero columns leave every dot
        # product, norm and centroid of the real columns unchanged (bit-exact
        # reproduction of numpy's evaluation order is for d % 4 == 0, i.e.
        # every head dim the engine serves)
        pad = np.zeros((n, 4 - d % 4), np.float32)
        keys_np = np.concatenate([keys_np, pad], axis=1)
        d = keys_np.shape[1]
    dev = torch.device(device)
    kt = torch.from_numpy(np.ascontiguousarray(keys_np)).to(dev)
    # a throwaway one-unit index receives finalize/pack output
    f32, i32 = torch.float32, torch.int32
    store = torch.empty((1, n, d), dtype=f32, device=dev)
    store_v = torch.empty((1, n, d), dtype=f32, device=dev)
    tok = torch.empty((1, n), dtype=i32, device=dev)
    off = torch.empty((1, k), dtype=i32, device=dev)
    size = torch.empty((1, k), dtype=i32, device=dev)
    c64 = torch.empty((1, k, d), dtype=torch.float64, device=dev)
    c32 = torch.empty((1, k, d), dtype=f32, device=dev)
    cn = torch.empty((1, k), dtype=f32, device=dev)
    vs = torch.empty((1, k, d), dtype=f32, device=dev)
    ix = _lib.IndexViewC(store.data_ptr(), store_v.data_ptr(), tok.data_ptr(), off.data_ptr(),
                         size.data_ptr(), c64.data_ptr(), c32.data_ptr(), cn.data_ptr(),
                         vs.data_ptr(), None, n, k)
    P = torch.empty((n, d), dtype=f32, device=dev)
    P16 = torch.empty((n, d), dtype=torch.float16, device=dev)
    C = torch.empty((k, d), dtype=f32, device=dev)
    A = torch.zeros(n, dtype=i32, device=dev)
    perm = torch.empty(n, dtype=i32, device=dev)
    sims = torch.empty(n, dtype=f32, device=dev)
    md = torch.empty(2 * n, dtype=f32, device=dev)
    status = torch.zeros(1, dtype=i32, device=dev)
    segs_dev = torch.empty(ctypes.sizeof(_lib.SegmentC), dtype=torch.uint8, device=dev)
    seg = (_lib.SegmentC * 1)()
    s = seg[0]
    s.keys, s.values, s.key_stride = kt.data_ptr(), kt.data_ptr(), d
    s.L, s.k, s.unit, s.cid_base, s.row_base, s.tok_base, s.p_off, s.c_off = n, k, 0, 0, 0, 0, 0, 0
    for t, w in enumerate(_seed_words(seed)):
        s.rng[t] = w
    scr = _lib.BuildScratchC(P.data_ptr(), C.data_ptr(), A.data_ptr(), perm.data_ptr(),
                             sims.data_ptr(), md.data_ptr(), segs_dev.data_ptr(), status.data_ptr(),
                             P16.data_ptr())
    rc = _lib.lib().wk_kmeans_segments(ctypes.byref(ix), seg, 1, ctypes.byref(scr), d, 0, iters,
                                       threads if threads is not None else _BLAS_THREADS, n, k,
                                       ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    _lib.check(rc, "wk_kmeans_segments")
    out = A.cpu().numpy().astype(np.int64)
    code = int(status.item())
    _lib.raise_status(code, "spherical_kmeans")
    return out
