"""Config-sweep golden fixtures from the UNMODIFIED reference (tierkv) -> tests/golden/.

TEST INFRASTRUCTURE.  Runs only in the dev container where /root/reference is
mounted:   python oracle/make_sweep_golden.py
Drives tierkv's own `sweep` command (cli.py:84-97, SWEEP_AXES cli.py:19-24) on
the committed trace_a.wkt (oracle/make_trace_golden.py) for two axes and keeps
each report with its wall-clock "timestamp" removed.
"""

from __future__ import annotations

import glob
import json
import os
import sys
import tempfile

from threadpoolctl import threadpool_limits

REF = "/root/reference/pkg/src"
GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
SWEEPS = [("retrieval_fraction", "0.018,0.06"), ("cache_fraction", "0.05,0.3")]


def main():
    sys.path.insert(0, REF)
    from tierkv.cli import main as tierkv_main
    out = {}
    with tempfile.TemporaryDirectory() as tmp, threadpool_limits(1):
        for axis, values in SWEEPS:
            rc = tierkv_main(["sweep", "--trace", os.path.join(GOLD, "trace_a.wkt"), "--axis", axis,
                              "--values", values, "--out-dir", tmp])
            assert rc == 0
        for path in sorted(glob.glob(os.path.join(tmp, "report_*.json"))):
            rep = json.load(open(path))
            rep.pop("timestamp")
            out[os.path.basename(path)] = rep
    with open(os.path.join(GOLD, "sweep_trace_a.json"), "w") as f:
        json.dump({"blas_threads": 1, "sweeps": SWEEPS, "reports": out}, f, indent=1, sort_keys=True)
    print(sorted(out))


if __name__ == "__main__":
    main()
