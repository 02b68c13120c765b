"""WKT1 trace files (tierkv tracefile.py): the reader parses the reference
writer's bytes, the writer reproduces them byte for byte, and malformed files
raise TraceFormatError at the reference's byte offsets (tests mirror tierkv
tests/test_tracefile.py)."""
import os
import struct

import numpy as np
import pytest

from paper_2505_02922_b200.errors import TraceFormatError
from paper_2505_02922_b200.tracefile import HEADER, TraceFile, read_trace, write_trace

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("name", ["trace_a", "trace_b"])
def test_reads_reference_file_and_rewrites_it_byte_identical(name, tmp_path):
    path = os.path.join(GOLD, f"{name}.wkt")
    tr = read_trace(path)
    raw = open(path, "rb").read()
    _, _, h, d, n, t = HEADER.unpack_from(raw)
    assert (tr.n_heads, tr.d, tr.n_prefill, tr.n_decode) == (h, d, n, t)
    body = np.frombuffer(raw, "<f4", offset=HEADER.size)
    # first prefill key row of head 0, first query of step 0 / head 0
    assert np.array_equal(tr.prefill_keys[0, 0], body[:d])
    off = 2 * h * n * d
    assert np.array_equal(tr.queries[0, 0], body[off:off + d])
    assert np.array_equal(tr.new_values[t - 1, h - 1], body[-d:])
    out = tmp_path / "copy.wkt"
    write_trace(out, tr)
    assert open(out, "rb").read() == raw


def _tiny(h=2, n=3, d=4, t=2, seed=0):
    r = np.random.default_rng(seed)
    f = lambda *s: r.standard_normal(s).astype(np.float32)
    return TraceFile(d=d, prefill_keys=f(h, n, d), prefill_values=f(h, n, d), queries=f(t, h, d),
                     new_keys=f(t, h, d), new_values=f(t, h, d))


def test_round_trip(tmp_path):
    tr = _tiny()
    write_trace(tmp_path / "a.wkt", tr)
    back = read_trace(tmp_path / "a.wkt")
    for k in ("prefill_keys", "prefill_values", "queries", "new_keys", "new_values"):
        assert np.array_equal(getattr(back, k), getattr(tr, k))


def test_zero_decode_steps(tmp_path):
    tr = _tiny(t=0)
    write_trace(tmp_path / "a.wkt", tr)
    assert read_trace(tmp_path / "a.wkt").n_decode == 0


def _write_raw(path, data):
    with open(path, "wb") as f:
        f.write(data)
    return path


@pytest.mark.parametrize("case,offset", [("short", 10), ("magic", 0), ("version", 4), ("d0", 12),
                                         ("heads0", 8), ("body", None)])
def test_malformed_files(tmp_path, case, offset):
    good = HEADER.pack(b"WKT1", 1, 1, 4, 2, 1) + b"\0" * 4 * (2 * 2 * 4 + 3 * 4)
    if case == "short":
        data = good[:10]
    elif case == "magic":
        data = b"XXXX" + good[4:]
    elif case == "version":
        data = HEADER.pack(b"WKT1", 2, 1, 4, 2, 1) + good[HEADER.size:]
    elif case == "d0":
        data = HEADER.pack(b"WKT1", 1, 1, 0, 2, 1)
    elif case == "heads0":
        data = HEADER.pack(b"WKT1", 1, 0, 4, 2, 1)
    else:
        data = good[:-4]
        offset = len(data)
    with pytest.raises(TraceFormatError) as ei:
        read_trace(_write_raw(tmp_path / "bad.wkt", data))
    assert ei.value.offset == offset


def test_validate_rejects_inconsistent_shapes():
    tr = _tiny()
    with pytest.raises(TraceFormatError):
        TraceFile(d=5, prefill_keys=tr.prefill_keys, prefill_values=tr.prefill_values, queries=tr.queries,
                  new_keys=tr.new_keys, new_values=tr.new_values).validate()
    with pytest.raises(TraceFormatError):
        TraceFile(d=4, prefill_keys=tr.prefill_keys, prefill_values=tr.prefill_values[:, :2],
                  queries=tr.queries, new_keys=tr.new_keys, new_values=tr.new_values).validate()
    with pytest.raises(TraceFormatError):
        TraceFile(d=4, prefill_keys=tr.prefill_keys, prefill_values=tr.prefill_values, queries=tr.queries,
                  new_keys=tr.new_keys[:1], new_values=tr.new_values).validate()
    assert struct.calcsize("<4sIIIQQ") == HEADER.size == 32


def test_sweep_rejects_unknown_axis():
    """runner.sweep_trace mirrors cli.py's SWEEP_AXES (cli.py:19-24): any other
    axis is a ConfigError before anything runs."""
    import pytest
    from paper_2505_02922_b200 import EngineConfig
    from paper_2505_02922_b200.errors import ConfigError
    from paper_2505_02922_b200.runner import SWEEP_AXES, sweep_trace
    assert sorted(SWEEP_AXES) == ["cache_fraction", "estimation_fraction", "retrieval_fraction", "segment_size"]
    with pytest.raises(ConfigError):
        sweep_trace(None, EngineConfig(), "kmeans_iters", "5,10")
