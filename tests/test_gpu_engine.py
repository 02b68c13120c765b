"""GPU: the tierkv-shaped HeadEngine facade vs the reference's golden runs
(every StepMetrics field, the block-cache event stream, store accounting) and
the reference's own engine-level properties (tests mirror tierkv
tests/test_engine.py)."""
import math

import numpy as np
import pytest
import torch

from tests import golden_util as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _engine(cfgd, threads=1, **kw):
    from paper_2505_02922_b200 import EngineConfig
    from paper_2505_02922_b200.engine import HeadEngine
    return HeadEngine(EngineConfig.from_dict(cfgd), blas_threads=threads, **kw)


@pytest.mark.parametrize("name", G.manifest()["files"]["engine"])
def test_step_metrics_and_events_match_reference(name):
    z, cfgd = G.engine_case(name)
    eng = _engine(cfgd, int(z["threads"])).prefill(z["prefill_keys"], z["prefill_values"])
    assert np.array_equal(eng.index.centroids, z["centroids0"])
    for t in range(len(z["queries"])):
        out, sm = eng.decode_step(z["queries"][t], z["new_keys"][t], z["new_values"][t],
                                  with_oracle=True)
        ref = z["metrics"][t]
        assert [sm.step, sm.hits, sm.misses, sm.bytes_slow_to_fast, sm.bytes_fast_internal,
                sm.m, sm.r, sm.e] == [int(ref[i]) for i in (0, 3, 4, 5, 6, 9, 10, 11)], t
        assert sm.recall == pytest.approx(ref[1], abs=1e-6)
        assert abs(sm.rel_error - ref[2]) <= 2e-5 + 1e-3 * ref[2]
        assert abs(sm.log_denominator - ref[8]) <= 1e-5
        assert abs(sm.denominator_coverage - ref[7]) <= 1e-5
        assert np.linalg.norm(out - z["outputs"][t]) <= 1e-5 * np.linalg.norm(z["outputs"][t])
    log = eng.cache.event_log  # the reference's dicts (block_cache.py:92-95, 188-207)
    ev = [(e["type"], e["step"], e["cluster"]) for e in log if e["type"] != "access"]
    names = {1: "evict", 2: "admit", 3: "reject"}
    ref_ev = [(names[int(a)], int(b), int(c)) for a, b, c, _ in z["events"]]
    assert ev == ref_ev
    acc = [e for e in log if e["type"] == "access"]
    assert len(acc) == len(z["queries"])
    assert sum(sum(e["cached"]) for e in acc) == eng.cache.hits
    assert sum(len(e["clusters"]) - sum(e["cached"]) for e in acc) == eng.cache.misses
    import json
    st = json.loads(str(z["final_stats"]))
    mine = eng.cache.stats()
    for k in ("hits", "misses", "bytes_slow_to_fast", "bytes_fast_internal", "capacity_blocks",
              "occupied_blocks"):
        assert mine[k] == st[k], k
    store = json.loads(str(z["store"]))
    assert eng.store.n_blocks == store["n_blocks"]
    assert eng.store.bytes_read_total == store["bytes_read_total"]
    assert eng.store.bytes_written_total == store["bytes_written_total"]


def _trace(n_prefill, n_decode, d=16, seed=0, **kw):
    """Small bf16-representable trace (tierkv synth.py-style latent centres)."""
    rng = np.random.default_rng(seed)
    cen = rng.standard_normal((32, d)).astype(np.float32)
    k = G.bf16_round(cen[rng.integers(32, size=n_prefill)] + 0.25 * rng.standard_normal((n_prefill, d)))
    v = G.bf16_round(rng.standard_normal((n_prefill, d)))
    q = G.bf16_round(cen[rng.integers(32, size=n_decode)] + 0.25 * rng.standard_normal((n_decode, d)))
    nk = G.bf16_round(cen[rng.integers(32, size=n_decode)] + 0.25 * rng.standard_normal((n_decode, d)))
    nv = G.bf16_round(rng.standard_normal((n_decode, d)))
    return k, v, q, nk, nv


def test_prefill_short_prompt_all_steady():
    k, v, *_ = _trace(68, 0)
    eng = _engine({"kmeans_iters": 3}).prefill(k, v)
    assert eng.index.m == 0 and eng.n_sink == 4 and len(eng.buffer) == 64
    assert len(eng._steady_ids()) == 68


def test_prefill_single_segment_cluster_count():
    k, v, *_ = _trace(8260, 0, d=8)
    eng = _engine({"kmeans_iters": 3}).prefill(k, v)
    assert eng.index.m == 512 and int(eng.index.sizes.sum()) == 8192


def test_full_retrieval_matches_oracle_attention():
    k, v, q, nk, nv = _trace(1024, 16, seed=5)
    eng = _engine({"kmeans_iters": 3, "retrieval_fraction": 1.0, "estimation_fraction": 0.0,
                   "cache_fraction": 1.0}).prefill(k, v)
    for t in range(16):
        _, sm = eng.decode_step(q[t], nk[t], nv[t], with_oracle=True)
        assert sm.rel_error <= 1e-5 and sm.e == 0 and sm.r == sm.m


def test_step_barrier_first_touch_misses_then_hits():
    k, v, q, nk, nv = _trace(1024, 2)
    q[1] = q[0]
    eng = _engine({"kmeans_iters": 3, "retrieval_fraction": 0.1, "cache_fraction": 1.0}).prefill(k, v)
    _, s0 = eng.decode_step(q[0], nk[0], nv[0])
    _, s1 = eng.decode_step(q[1], nk[1], nv[1])
    assert s0.hits == 0 and s0.misses > 0
    assert s1.misses == 0 and s1.hits > 0


def test_update_fires_on_schedule_and_conserves_tokens():
    k, v, q, nk, nv = _trace(512, 1100, seed=2)
    eng = _engine({"kmeans_iters": 3}).prefill(k, v)
    ms = []
    for t in range(1100):
        _, sm = eng.decode_step(q[t], nk[t], nv[t])
        ms.append(sm.m)
    changes = [t for t in range(1, len(ms)) if ms[t] != ms[t - 1]]
    assert len(changes) == 1 and ms[-1] == ms[0] + math.ceil(1024 / 16)
    assert int(eng.index.sizes.sum()) + eng.n_sink + len(eng.buffer) == eng.total_tokens


def test_determinism_bitwise():
    k, v, q, nk, nv = _trace(512, 8, seed=8)
    runs = []
    for _ in range(2):
        eng = _engine({"kmeans_iters": 3}).prefill(k, v)
        runs.append([eng.decode_step(q[t], nk[t], nv[t]) for t in range(8)])
    for (oa, sa), (ob, sb) in zip(*runs):
        assert np.array_equal(oa, ob) and sa == sb


def test_errors_match_reference_conventions():
    from paper_2505_02922_b200 import ConfigError
    k, v, *_ = _trace(100, 0)
    eng = _engine({})
    with pytest.raises(ConfigError):
        eng.decode_step(np.zeros(16), np.zeros(16), np.zeros(16))
    eng.prefill(k, v)
    with pytest.raises(ConfigError):
        eng.prefill(k, v)
