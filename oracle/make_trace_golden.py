"""Trace-replay golden fixtures from the UNMODIFIED reference (tierkv) -> tests/golden/.

TEST INFRASTRUCTURE.  Runs only in the dev container where /root/reference is
mounted:   python oracle/make_trace_golden.py
Writes, per case, the WKT1 file produced by tierkv's own writer
(tracefile.py:58-68), the report of tierkv's run_trace (runner.py:28-110) with
the wall-clock "timestamp" removed, and its output / oracle arrays.  Inputs are
bf16-representable so the bf16-capable device store holds them exactly; BLAS
threads are pinned (dgemv chunk tails depend on them) and recorded.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
from threadpoolctl import threadpool_limits

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
CASES = [
    # name, synth params, engine config, BLAS threads
    ("trace_a", dict(heads=3, n_prefill=700, n_decode=10, d=64, seed=21), {"cache_fraction": 0.1}, 1),
    ("trace_b", dict(heads=2, n_prefill=300, n_decode=6, d=16, seed=22), {}, 1),
]


def bf16_round(x):
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def main():
    sys.path.insert(0, REF)
    from tierkv import EngineConfig, SynthParams, gen_trace
    from tierkv.runner import run_trace
    from tierkv.tracefile import TraceFile, read_trace, write_trace

    for name, sp, ecfg, thr in CASES:
        tr = gen_trace(SynthParams(**sp))
        tr = TraceFile(d=tr.d, prefill_keys=bf16_round(tr.prefill_keys), prefill_values=bf16_round(tr.prefill_values),
                       queries=bf16_round(tr.queries), new_keys=bf16_round(tr.new_keys),
                       new_values=bf16_round(tr.new_values))
        path = os.path.join(OUT, f"{name}.wkt")
        write_trace(path, tr)
        tr = read_trace(path)
        cfg = EngineConfig.from_dict(ecfg)
        with threadpool_limits(thr):
            report, outs, orc = run_trace(tr, cfg, with_oracle=True)
        report.pop("timestamp")
        report["blas_threads"] = thr
        with open(os.path.join(OUT, f"{name}_report.json"), "w") as f:
            json.dump(report, f, indent=1, sort_keys=True)
        np.savez_compressed(os.path.join(OUT, f"{name}_out.npz"), outputs=outs, oracle=orc)
        print(name, os.path.getsize(path), "bytes;", report["aggregates"])


if __name__ == "__main__":
    main()
