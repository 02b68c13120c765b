"""Function-level attention API on the device (tierkv attention.py:17-148).

Each call runs one fp64 kernel of libwavekv.so (csrc/api.cu): an exact or
centroid-estimated streaming-softmax partial, the LSE merge, the full
attention oracle.  Inputs are caller-owned arrays (copied to the device),
outputs fresh float64 numpy arrays, exactly the reference's types.  The
batched decode path fuses the same math into one fp32-accumulating kernel
(attend_v4 + att4_merge); this module is the per-call form tierkv exposes.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ConfigError


@dataclass
class PartialAttention:
    """Streaming-softmax accumulator (attention.py:17-32); numerator and
    denominator are scaled by exp(-running_max); count 0 = merge identity."""
    running_max: float
    numerator: np.ndarray
    denominator: float
    count: int

    @classmethod
    def empty(cls, d: int) -> "PartialAttention":
        return cls(-np.inf, np.zeros(d), 0.0, 0)


@dataclass
class AttentionOutput:
    output: np.ndarray
    denominator_exact_coverage: float
    log_denominator: float


@dataclass
class OpCounter:
    count: int = 0

    def reset(self):
        self.count = 0


# cluster terms evaluated by estimate_partial (attention.py:42-52): one per
# estimated cluster, independent of cluster sizes (acceptance criterion 9)
estimation_ops = OpCounter()

_DEV = None


def _dev():
    global _DEV
    if _DEV is None:
        if not torch.cuda.is_available():
            raise RuntimeError("the attention API runs on a CUDA device (no CPU fallback)")
        _DEV = torch.device("cuda", torch.cuda.current_device())
    return _DEV


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _d64(x, shape=None):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return torch.from_numpy(a).to(_dev())


def _partial(q, rows, vals, sizes, scores, n, d, mode) -> PartialAttention:
    out = torch.empty(3 + d, dtype=torch.float64, device=_dev())
    scratch = torch.empty(max(1, n), dtype=torch.float64, device=_dev())
    p = lambda t: None if t is None else t.data_ptr()
    rc = _lib.lib().wk_attn_partial_f64(p(q), p(rows), p(vals), p(sizes), p(scores), n, d, mode, 1,
                                        scratch.data_ptr(), out.data_ptr(), _stream())
    _lib.check(rc, "wk_attn_partial_f64")
    o = out.cpu().numpy()
    return PartialAttention(float(o[0]), o[3:].copy(), float(o[1]), int(o[2]))


def exact_partial(q, keys, values) -> PartialAttention:
    """Exact partial over a token subset, empty allowed (attention.py:67-78)."""
    qn = np.asarray(q, dtype=np.float64)
    d = qn.shape[0]
    kn = np.asarray(keys, dtype=np.float64).reshape(-1, d)
    if kn.shape[0] == 0:
        return PartialAttention.empty(d)
    vn = np.asarray(values, dtype=np.float64).reshape(-1, d)
    return _partial(_d64(qn), _d64(kn), _d64(vn), None, None, kn.shape[0], d, 0)


def estimate_partial(q, centroids, value_sums, sizes, scores=None) -> PartialAttention:
    """Clusters through their centroids and value sums, one term per cluster
    (attention.py:81-104); optional precomputed q.C scores."""
    qn = np.asarray(q, dtype=np.float64)
    d = qn.shape[0]
    C = np.asarray(centroids, dtype=np.float64).reshape(-1, d)
    e = C.shape[0]
    if e == 0:
        return PartialAttention.empty(d)
    VS = np.asarray(value_sums, dtype=np.float64).reshape(-1, d)
    sz = np.asarray(sizes, dtype=np.float64).reshape(-1)
    sc = None if scores is None else _d64(scores, (-1,))
    estimation_ops.count += e
    return _partial(_d64(qn), _d64(C), _d64(VS), _d64(sz), sc, e, d, 1)


def tail_denominator_partial(q, centroids, sizes, scores=None) -> PartialAttention:
    """Dropped clusters' denominator-only term (attention.py:107-112)."""
    qn = np.asarray(q, dtype=np.float64)
    d = qn.shape[0]
    C = np.asarray(centroids, dtype=np.float64).reshape(-1, d)
    e = C.shape[0]
    if e == 0:
        return PartialAttention.empty(d)
    sz = np.asarray(sizes, dtype=np.float64).reshape(-1)
    sc = None if scores is None else _d64(scores, (-1,))
    estimation_ops.count += e
    return _partial(_d64(qn), _d64(C), None, _d64(sz), sc, e, d, 2)


def _pack(partials):
    d = partials[0].numerator.shape[0]
    rows = np.empty((len(partials), 3 + d), np.float64)
    for i, p in enumerate(partials):
        rows[i, 0], rows[i, 1], rows[i, 2] = p.running_max, p.denominator, p.count
        rows[i, 3:] = p.numerator
    return rows, d


def _merge_dev(partials, exact_mask=None):
    if not any(p.count > 0 and (exact_mask is None or exact_mask[i] != 2) for i, p in enumerate(partials)):
        raise ConfigError("merge requires at least one non-empty partial")
    rows, d = _pack(partials)
    out = torch.empty(2 * d + 3, dtype=torch.float64, device=_dev())
    status = torch.zeros(1, dtype=torch.int32, device=_dev())
    mask = None if exact_mask is None else torch.from_numpy(np.asarray(exact_mask, np.uint8)).to(_dev())
    rc = _lib.lib().wk_merge_f64(_d64(rows).data_ptr(), len(partials), d,
                                 None if mask is None else mask.data_ptr(), out.data_ptr(),
                                 status.data_ptr(), _stream())
    _lib.check(rc, "wk_merge_f64")
    _lib.raise_status(int(status.item()), "merge")
    return out.cpu().numpy(), d


def merged_sums(partials) -> tuple[float, np.ndarray, float, int]:
    """Rescale the live partials to a common max and sum them
    (attention.py:115-130): (gmax, numerator, denominator, count)."""
    live = [p for p in partials if p.count > 0]
    if not live:
        raise ConfigError("merge requires at least one non-empty partial")
    o, d = _merge_dev(live)
    gmax = max(p.running_max for p in live)
    return gmax, o[d + 3:].copy(), float(o[d + 2]), sum(p.count for p in live)


def merge(partials, exact_partials=None) -> AttentionOutput:
    """LSE merge of zone partials (attention.py:133-148); exact_partials
    marks the subset whose denominator mass counts as exact coverage."""
    partials = list(partials)
    if exact_partials is None:
        o, d = _merge_dev(partials)
        return AttentionOutput(o[:d].copy(), 1.0, float(o[d + 1]))
    # exact partials that are not zone partials add coverage mass only
    extra = [p for p in exact_partials if not any(p is z for z in partials)]
    mask = [1 if any(p is e for e in exact_partials) else 0 for p in partials] + [2] * len(extra)
    o, d = _merge_dev(partials + extra, mask)
    return AttentionOutput(o[:d].copy(), float(o[d]), float(o[d + 1]))


def oracle_attention(q, keys, values) -> np.ndarray:
    """Full softmax(q.K^T / sqrt(d)).V in fp64 (attention.py:55-64)."""
    kn = np.asarray(keys, dtype=np.float64)
    if kn.shape[0] == 0:
        raise ConfigError("oracle_attention needs at least one token")
    p = exact_partial(q, kn, values)
    o, d = _merge_dev([p])
    return o[:d].copy()
