"""GPU: batched trace replay (runner.run_trace over one WaveLayer, heads as
units) against the reference's own run_trace report on the same WKT1 file
(tests/golden/trace_*; oracle/make_trace_golden.py)."""
import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _compare_reports(rep, ref, name):
    """the fields tierkv's report pins bit-for-bit / to the stated tolerances"""
    assert rep["config"] == ref["config"] and rep["trace"] == ref["trace"]
    assert rep["schema_version"] == ref["schema_version"]
    for mine, theirs in zip(rep["per_head"], ref["per_head"]):
        assert mine["head"] == theirs["head"]
        for k in ("hits", "misses", "bytes_slow_to_fast", "bytes_fast_internal", "m", "r", "e"):
            assert mine["steps"][k] == theirs["steps"][k], (name, mine["head"], k)
        assert np.allclose(mine["steps"]["recall"], theirs["steps"]["recall"], atol=1e-6)
        for k in ("hits", "misses", "hit_ratio", "bytes_slow_to_fast", "bytes_fast_internal", "capacity_blocks",
                  "occupied_blocks", "bytes_offloaded", "slow_blocks", "clusters"):
            assert mine["totals"][k] == theirs["totals"][k], (name, k)
    for k in ("cumulative_hit_ratio", "total_bytes_slow_to_fast", "total_bytes_fast_internal",
              "total_bytes_offloaded"):
        assert rep["aggregates"][k] == ref["aggregates"][k], k
    assert rep["aggregates"]["mean_recall"] == pytest.approx(ref["aggregates"]["mean_recall"], abs=1e-6)


def test_sweep_matches_reference_reports():
    """tierkv's `sweep` command (cli.py:84-97) over two axes of trace_a vs
    runner.sweep_trace (oracle/make_sweep_golden.py)."""
    from paper_2505_02922_b200 import EngineConfig
    from paper_2505_02922_b200.runner import sweep_trace
    from paper_2505_02922_b200.tracefile import read_trace
    gold = json.load(open(os.path.join(GOLD, "sweep_trace_a.json")))
    tr = read_trace(os.path.join(GOLD, "trace_a.wkt"))
    for axis, values in gold["sweeps"]:
        reps = sweep_trace(tr, EngineConfig(), axis, values, blas_threads=gold["blas_threads"])
        for raw, rep in zip(values.split(","), reps):
            ref = gold["reports"][f"report_{axis}_{raw}.json"]
            assert rep["sweep"] == ref["sweep"]
            _compare_reports(rep, ref, f"{axis}={raw}")


@pytest.mark.parametrize("name", ["trace_a", "trace_b"])
def test_run_trace_matches_reference_report(name):
    from paper_2505_02922_b200 import EngineConfig
    from paper_2505_02922_b200.runner import oracle_trace, run_trace
    from paper_2505_02922_b200.tracefile import read_trace
    ref = json.load(open(os.path.join(GOLD, f"{name}_report.json")))
    z = np.load(os.path.join(GOLD, f"{name}_out.npz"))
    tr = read_trace(os.path.join(GOLD, f"{name}.wkt"))
    cfg = EngineConfig.from_dict(ref["config"])
    rep, outs, orc = run_trace(tr, cfg, with_oracle=True, blas_threads=ref["blas_threads"])
    json.dumps(rep, allow_nan=False)
    assert rep["config"] == ref["config"] and rep["trace"] == ref["trace"]
    assert rep["schema_version"] == ref["schema_version"]
    for mine, theirs in zip(rep["per_head"], ref["per_head"]):
        assert mine["head"] == theirs["head"]
        for k in ("hits", "misses", "bytes_slow_to_fast", "bytes_fast_internal", "m", "r", "e"):
            assert mine["steps"][k] == theirs["steps"][k], (name, mine["head"], k)
        assert np.allclose(mine["steps"]["recall"], theirs["steps"]["recall"], atol=1e-6)
        assert np.allclose(mine["steps"]["denominator_coverage"], theirs["steps"]["denominator_coverage"],
                           atol=1e-5)
        a, b = np.array(mine["steps"]["rel_error"]), np.array(theirs["steps"]["rel_error"])
        assert np.all(np.abs(a - b) <= 2e-5 + 1e-3 * b)
        for k in ("hits", "misses", "hit_ratio", "bytes_slow_to_fast", "bytes_fast_internal", "capacity_blocks",
                  "occupied_blocks", "bytes_offloaded", "slow_blocks", "clusters"):
            assert mine["totals"][k] == theirs["totals"][k], (name, k)
    for k in ("cumulative_hit_ratio", "total_bytes_slow_to_fast", "total_bytes_fast_internal",
              "total_bytes_offloaded"):
        assert rep["aggregates"][k] == ref["aggregates"][k], k
    assert rep["aggregates"]["mean_recall"] == pytest.approx(ref["aggregates"]["mean_recall"], abs=1e-6)
    # outputs: rel-L2 <= 1e-5 per (step, head) vs the reference engine's fp64 outputs
    num = np.linalg.norm(outs - z["outputs"], axis=-1)
    assert np.all(num <= 1e-5 * np.linalg.norm(z["outputs"], axis=-1))
    # the fp64 oracle of every step and head
    exact = oracle_trace(tr)
    assert np.allclose(exact, z["oracle"], rtol=1e-10, atol=1e-12)
    assert np.all(np.linalg.norm(orc - z["oracle"], axis=-1) <= 1e-5 * np.linalg.norm(z["oracle"], axis=-1))
