"""Pin the C oracle (oracle/wk_oracle.c) against fixtures produced by the
unmodified reference tierkv (oracle/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import golden_util as G


def test_rng_draws_match_numpy_generator():
    z = G.load("rng.npz")
    for s, row in zip(z["seeds"], z["draws"]):
        r = O.Rng(np.random.SeedSequence([int(x) for x in s]))
        got = [r.integers(8124), r.random(), r.integers(8192), r.random(), r.integers(3),
               r.integers(1024), r.random()]
        assert np.array_equal(np.array(got, dtype=np.float64), row)


@pytest.mark.parametrize("name", G.manifest()["files"]["kmeans"])
def test_kmeans_bit_exact(name):
    z = G.load(name)
    a = O.spherical_kmeans(z["keys"], int(z["k"]), int(z["iters"]),
                           np.random.SeedSequence([int(x) for x in z["seed"]]),
                           threads=int(z["threads"]))
    assert np.array_equal(a.astype(np.int32), z["assignment"])


@pytest.mark.parametrize("case", G.rank_cases(), ids=lambda c: c[0])
def test_rank_bit_exact(case):
    _, c = case
    for i, q in enumerate(c["Q"]):
        order, scores = O.rank_clusters(q, c["C"], threads=int(c["threads"]))
        assert np.array_equal(order.astype(np.int32), c["orders"][i])
        assert np.array_equal(scores.view(np.uint64), c["scores"][i].view(np.uint64))


def test_topk_tokens_bit_exact():
    keys, z = G.topk_case()
    for thr, key in ((8, "top_t8"), (1, "top_t1")):
        s = O.dgemv(keys.astype(np.float64), z["q"], threads=thr)
        order = np.lexsort((np.arange(len(s)), -s))[:100]
        assert np.array_equal(order.astype(np.int32), z[key])


@pytest.mark.parametrize("name", G.manifest()["files"]["engine"])
def test_engine_matches_reference(name):
    z, cfg = G.engine_case(name)
    eng = O.OracleEngine(blas_threads=int(z["threads"]), **cfg)
    eng.prefill(z["prefill_keys"], z["prefill_values"])
    assert np.array_equal(eng.centroids, z["centroids0"])
    assert np.array_equal(eng.value_sums, z["value_sums0"])
    assert np.array_equal(eng.sizes, z["sizes0"])
    rids = G.split(z["retrieval_flat"], z["retrieval_len"])
    eids = G.split(z["estimation_flat"], z["estimation_len"])
    for t in range(len(z["queries"])):
        out, sm = eng.decode_step(z["queries"][t], z["new_keys"][t], z["new_values"][t],
                                  with_oracle=True)
        ref = z["metrics"][t]
        r, e = eng.last_plan()
        assert np.array_equal(r, rids[t])
        assert np.array_equal(np.sort(e), eids[t])
        assert [sm.step, sm.hits, sm.misses, sm.bytes_slow_to_fast, sm.bytes_fast_internal,
                sm.m, sm.r, sm.e] == [int(ref[i]) for i in (0, 3, 4, 5, 6, 9, 10, 11)]
        assert sm.recall == ref[1]
        assert np.linalg.norm(out - z["outputs"][t]) <= 1e-12 * np.linalg.norm(z["outputs"][t])
        assert abs(sm.log_denominator - ref[8]) <= 1e-12
        assert abs(sm.denominator_coverage - ref[7]) <= 1e-12
    t, s, c, a = eng.events()
    mine = np.stack([t, s, c, a], 1)[t != 0].astype(np.int64)
    ev = z["events"]
    assert np.array_equal(mine[:, :3], ev[:, :3])
    adm = ev[:, 0] == 2
    assert np.array_equal(mine[adm, 3], ev[adm, 3])
