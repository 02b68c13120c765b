"""The drop-in proof: tierkv's own unit and acceptance checks, restated
against this package's public API (import ``paper_2505_02922_b200`` where a
tierkv user imports ``tierkv``).  Each test cites the reference test it
restates (pkg/tests/<file>:<lines>); the known answers and tolerances are the
reference's.  Everything computes on the GPU (fp64 function-level kernels of
csrc/api.cu, the device block-cache state machine, the batched engine).

Not restated: acceptance criterion 06 (wall-clock build speed-up of the CPU
reference), criterion 10 (the reference's CLI), test_cli / test_synth /
test_tracefile (harness; the WKT1 reader is covered by tests/test_trace.py).
"""
import math

import numpy as np
import pytest
import torch

import paper_2505_02922_b200 as tk
from paper_2505_02922_b200 import (BlockCache, ClusterIndex, ConfigError, EngineConfig, HeadEngine,
                                   IndexConfig, IntegrityError, PartialAttention, SlowTierStore, TokenKV)
from paper_2505_02922_b200.attention import (estimate_partial, estimation_ops, exact_partial, merge,
                                             oracle_attention, tail_denominator_partial)
from paper_2505_02922_b200.index import finalize_cluster, plan_zones, rank_clusters

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def tokens(rng, n, d, start=0):
    k = rng.standard_normal((n, d)).astype(np.float32)
    v = rng.standard_normal((n, d)).astype(np.float32)
    return [TokenKV(k[i], v[i], start + i) for i in range(n)]


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


def softmax_ref(q, K, V):
    """Independent two-pass reference (materialised softmax)."""
    s = np.asarray(K, np.float64) @ np.asarray(q, np.float64) / np.sqrt(len(q))
    w = np.exp(s - s.max())
    return (w / w.sum()) @ np.asarray(V, np.float64)


class Trace:
    """Synthetic per-head trace in the shape tierkv's tests use: per-segment
    latent centres + noise for keys, a persistent random walk over the
    centres for queries (the structure of synth.py:46-70)."""

    def __init__(self, n_prefill, n_decode, d=16, seed=0, persistence=0.9, noise=0.25,
                 heavy_tail=0.0, seg=8192, centres=32):
        r = np.random.default_rng(seed)
        ns = -(-n_prefill // seg)
        C = r.standard_normal((ns, centres, d))
        self.keys = (C[np.arange(n_prefill) // seg, r.integers(centres, size=n_prefill)]
                     + noise * r.standard_normal((n_prefill, d))).astype(np.float32)
        self.values = r.standard_normal((n_prefill, d)).astype(np.float32)
        flat = C.reshape(-1, d)
        walk = int(r.integers(len(flat)))
        self.q = np.empty((n_decode, d), np.float32)
        self.nk = np.empty((n_decode, d), np.float32)
        for t in range(n_decode):
            if r.random() >= persistence:
                walk = int(r.integers(len(flat)))
            self.q[t] = (1 + heavy_tail) * flat[walk] + noise * r.standard_normal(d)
            self.nk[t] = C[-1, r.integers(centres)] + noise * r.standard_normal(d)
        self.nv = r.standard_normal((n_decode, d)).astype(np.float32)
        self.d, self.n_decode = d, n_decode

    def run(self, cfg, with_oracle=False):
        eng = HeadEngine(cfg).prefill(self.keys, self.values)
        rows = [eng.decode_step(self.q[t], self.nk[t], self.nv[t], with_oracle=with_oracle)
                for t in range(self.n_decode)]
        return eng, rows


def small(**idx):
    return EngineConfig(index=IndexConfig(**{"kmeans_iters": 3, **idx}))


# ------------------------------------------------------------------ attention
# pkg/tests/test_attention.py

def test_oracle_single_token_and_identical_keys(rng):
    v = rng.standard_normal(4)  # :27-30
    assert np.allclose(oracle_attention(rng.standard_normal(4), rng.standard_normal((1, 4)), v[None]), v)
    K = np.tile(rng.standard_normal(6), (9, 1))  # :33-37
    V = rng.standard_normal((9, 6))
    assert np.allclose(oracle_attention(rng.standard_normal(6), K, V), V.mean(axis=0))


def test_oracle_matches_two_pass_and_rejects_empty(rng):
    q, K, V = rng.standard_normal(32), rng.standard_normal((256, 32)), rng.standard_normal((256, 32))
    assert rel(oracle_attention(q, K, V), softmax_ref(q, K, V)) < 1e-6  # :40-45
    with pytest.raises(ConfigError):  # :48-50
        oracle_attention(np.zeros(3), np.empty((0, 3)), np.empty((0, 3)))


def test_merge_identity_single_partition_permutation(rng):
    q = rng.standard_normal(5)  # :55-60
    K, V = rng.standard_normal((7, 5)), rng.standard_normal((7, 5))
    full = exact_partial(q, K, V)
    ident = merge([full, PartialAttention.empty(5), exact_partial(q, [], [])])
    assert np.allclose(ident.output, merge([full]).output)
    q = rng.standard_normal(8)  # :63-67
    K, V = rng.standard_normal((50, 8)), rng.standard_normal((50, 8))
    assert rel(merge([exact_partial(q, K, V)]).output, oracle_attention(q, K, V)) < 1e-6
    K, V = rng.standard_normal((60, 8)), rng.standard_normal((60, 8))  # :82-89
    parts = [exact_partial(q, K[i:i + 20], V[i:i + 20]) for i in (0, 20, 40)]
    base = merge(parts).output
    for _ in range(5):
        assert rel(merge([parts[i] for i in rng.permutation(3)]).output, base) < 1e-6
    with pytest.raises(ConfigError):  # :92-94
        merge([PartialAttention.empty(4)])


@pytest.mark.parametrize("trial", range(10))
def test_random_partition_merge_matches_oracle(rng, trial):
    n, d = 120, 16  # :70-79
    q, K, V = rng.standard_normal(d), rng.standard_normal((n, d)), rng.standard_normal((n, d))
    cuts = np.sort(rng.choice(np.arange(1, n), size=2, replace=False))
    parts = [exact_partial(q, K[a:b], V[a:b]) for a, b in zip([0, *cuts], [*cuts, n])]
    assert rel(merge(parts).output, oracle_attention(q, K, V)) < 1e-6


def test_merge_associativity_property():
    """:97-110 (hypothesis, 40 examples) as 40 seeded draws of the same space."""
    draw = np.random.default_rng(97)
    for _ in range(40):
        sizes = draw.integers(1, 31, size=int(draw.integers(1, 7)))
        r = np.random.default_rng(int(draw.integers(2 ** 32)))
        d = 6
        q, K, V = r.standard_normal(d), r.standard_normal((sizes.sum(), d)), r.standard_normal((sizes.sum(), d))
        off = np.cumsum([0, *sizes])
        parts = [exact_partial(q, K[a:b], V[a:b]) for a, b in zip(off[:-1], off[1:])]
        assert rel(merge(parts).output, oracle_attention(q, K, V)) < 1e-6


def test_estimation_exact_on_singleton_and_identical_members(rng):
    q = rng.standard_normal(8)  # :119-128
    K, V = rng.standard_normal((1, 8)), rng.standard_normal((1, 8))
    est = estimate_partial(q, K.mean(0)[None], V.sum(0)[None], [1])
    ex = exact_partial(q, K, V)
    assert np.allclose(est.numerator * np.exp(est.running_max), ex.numerator * np.exp(ex.running_max))
    assert np.isclose(est.denominator * np.exp(est.running_max), ex.denominator * np.exp(ex.running_max))
    q = rng.standard_normal(4)  # :131-140
    K = np.tile(rng.standard_normal(4), (7, 1))
    V = rng.standard_normal((7, 4))
    a = merge([estimate_partial(q, K.mean(0)[None], V.sum(0)[None], [7])]).output
    assert rel(a, merge([exact_partial(q, K, V)]).output) < 1e-12


def test_estimated_denominator_below_exact(rng):
    q = rng.standard_normal(8)  # :143-154
    for _ in range(20):
        n = int(rng.integers(2, 40))
        K, V = rng.standard_normal((n, 8)), rng.standard_normal((n, 8))
        est = estimate_partial(q, K.mean(0)[None], V.sum(0)[None], [n])
        ex = exact_partial(q, K, V)
        assert est.denominator * np.exp(est.running_max) <= ex.denominator * np.exp(ex.running_max) * (1 + 1e-5)


def test_estimation_ops_and_tail_partial(rng):
    q = rng.standard_normal(8)  # :157-167
    C, VS = rng.standard_normal((10, 8)), rng.standard_normal((10, 8))
    estimation_ops.reset()
    estimate_partial(q, C, VS, np.full(10, 5))
    small_ = estimation_ops.count
    estimation_ops.reset()
    estimate_partial(q, C, VS, np.full(10, 5000))
    assert estimation_ops.count == small_ == 10
    p = tail_denominator_partial(q, rng.standard_normal((5, 8)), np.arange(1, 6))  # :170-175
    assert np.array_equal(p.numerator, np.zeros(8)) and p.denominator > 0


def test_partials_agree_with_fp64_numpy(rng):
    """The device partials are fp64: exact / estimated partials and the merge
    equal the reference's numpy expressions to ~1e-13."""
    q = rng.standard_normal(64)
    K, V = rng.standard_normal((300, 64)), rng.standard_normal((300, 64))
    p = exact_partial(q, K, V)
    s = K @ q / 8.0
    w = np.exp(s - s.max())
    assert abs(p.running_max - s.max()) <= 1e-13 * abs(s.max())
    assert rel(p.numerator, w @ V) < 1e-13 and abs(p.denominator - w.sum()) < 1e-13 * w.sum()
    sz = rng.integers(1, 9, size=300)
    e = estimate_partial(q, K, V, sz, scores=K @ q)
    assert abs(e.denominator - (sz * w).sum()) < 1e-13 * (sz * w).sum()
    out = merge([p, e], exact_partials=[p])
    g = max(p.running_max, e.running_max)
    den = p.denominator * np.exp(p.running_max - g) + e.denominator * np.exp(e.running_max - g)
    assert abs(out.denominator_exact_coverage - p.denominator * np.exp(p.running_max - g) / den) < 1e-13
    assert abs(out.log_denominator - (g + np.log(den))) < 1e-12
    gm, num, dd, cnt = tk.merged_sums([p, e])
    assert gm == g and cnt == 600 and abs(dd - den) < 1e-12 * den


# ---------------------------------------------------------------------- index
# pkg/tests/test_index.py

def test_finalize_cluster(rng):
    store = SlowTierStore(d=8, block_size_bytes=256)
    (t,) = tokens(rng, 1, 8)  # :20-25
    e = finalize_cluster([t], store, 0)
    assert np.allclose(e.centroid, t.key) and np.allclose(e.value_sum, t.value) and e.size == 1
    t1, t2 = tokens(rng, 2, 8, start=1)  # :28-32
    e = finalize_cluster([t1, t2], store, 1)
    assert np.allclose(e.centroid, (t1.key.astype(np.float64) + t2.key) / 2)
    with pytest.raises(IntegrityError):  # :35-37
        finalize_cluster([], store, 0)
    toks = tokens(rng, 50, 8, start=3)  # :40-50 (Jensen bound)
    e = finalize_cluster(toks, store, 2)
    K = np.stack([t.key for t in toks]).astype(np.float64)
    for q in rng.standard_normal((1000, 8)):
        assert math.exp(q @ e.centroid / math.sqrt(8)) <= np.exp(K @ q / math.sqrt(8)).mean() * (1 + 1e-5)
    # bit-exact vs numpy's mean / sum (index.py:53-54)
    assert np.array_equal(e.centroid, K.mean(axis=0))
    assert np.array_equal(e.value_sum, np.stack([t.value for t in toks]).astype(np.float64).sum(axis=0))


def test_rank_clusters(rng):
    order, scores = rank_clusters(np.array([1.0]), np.array([[3.0], [5.0], [5.0], [1.0]]))  # :56-60
    assert order.tolist() == [1, 2, 0, 3] and scores.tolist() == [3.0, 5.0, 5.0, 1.0]
    C = np.zeros((12, 4))  # :63-70
    C[:, 0] = rng.standard_normal(12)
    order, scores = rank_clusters(np.array([0.0, 1.0, 0.0, 0.0]), C)
    assert order.tolist() == list(range(12)) and (scores == 0).all()
    C, q = rng.standard_normal((64, 8)), rng.standard_normal(8)  # :73-78
    order, scores = rank_clusters(q, C)
    assert order.tolist() == sorted(range(64), key=lambda c: (-scores[c], c))
    # the scores are tierkv's dgemv bits (index.py:74; C oracle pinned to tierkv)
    from oracle import oracle as O
    assert np.array_equal(scores, O.rank_clusters(q, C, threads=1)[1])
    with pytest.raises(ConfigError):
        rank_clusters(np.ones(3), C)


def test_rank_clusters_large_matches_numpy_order(rng):
    C, q = rng.standard_normal((5000, 128)), rng.standard_normal(128)
    C[100:200] = C[0]  # duplicated rows: ties resolve to the lower id
    from oracle import oracle as O
    from paper_2505_02922_b200.clustering import set_blas_threads
    for threads in (1, 8):  # 5000 x 128 >= 460,800: OpenBLAS's threaded chunk tails
        set_blas_threads(threads)
        order, scores = rank_clusters(q, C)
        ref_order, ref = O.rank_clusters(q, C, threads=threads)
        assert np.array_equal(scores, ref)
        assert np.array_equal(order, ref_order)
        assert np.array_equal(order, np.lexsort((np.arange(5000), -ref)))
    set_blas_threads(1)


def test_plan_zones():
    cfg = IndexConfig(retrieval_fraction=150 / 8192, estimation_fraction=0.232)  # :83-90
    plan = plan_zones(np.arange(8192), -np.arange(8192.0), cfg, steady_token_ids=[0, 1])
    assert (len(plan.retrieval_cluster_ids), len(plan.estimation_cluster_ids),
            len(plan.dropped_cluster_ids)) == (150, 1901, 8192 - 150 - 1901)
    plan = plan_zones(np.empty(0, np.int64), np.empty(0), IndexConfig(), [5, 6])  # :93-98
    assert plan.steady_token_ids == [5, 6] and plan.retrieval_cluster_ids == [] == plan.estimation_cluster_ids
    plan = plan_zones(np.arange(10), np.zeros(10), IndexConfig(retrieval_fraction=1e-4,  # :101-105
                                                                estimation_fraction=0.5), [])
    assert len(plan.retrieval_cluster_ids) == 1


def test_plan_zones_partition_property(rng):
    cfg = IndexConfig(retrieval_fraction=0.1, estimation_fraction=0.3)  # :108-118
    for m in (1, 2, 5, 37, 200):
        order, scores = rank_clusters(rng.standard_normal(4), rng.standard_normal((m, 4)))
        plan = plan_zones(order, scores, cfg, [])
        union = plan.retrieval_cluster_ids + plan.estimation_cluster_ids + plan.dropped_cluster_ids
        assert sorted(union) == list(range(m))


def make_index(d=8, block=256, **kw):
    store = SlowTierStore(d=d, block_size_bytes=block)
    return ClusterIndex(IndexConfig(**kw).validate(), store), store


def test_segmented_build_counts_and_invariants(rng):
    index, _ = make_index(segment_size=64, centroid_ratio=16, kmeans_iters=3)  # :123-130
    entries = index.segmented_build(tokens(rng, 200, 8))
    assert len(entries) == 13 and [e.cluster_id for e in entries] == list(range(13))
    assert int(index.sizes.sum()) == 200
    index, _ = make_index(segment_size=8192, centroid_ratio=16, kmeans_iters=2)  # :133-136
    assert len(index.segmented_build(tokens(rng, 100, 8))) == math.ceil(100 / 16)
    index, _ = make_index()  # :139-142
    assert index.segmented_build([]) == [] and index.m == 0
    index, _ = make_index(segment_size=64, centroid_ratio=8, kmeans_iters=4)  # :145-160
    toks = tokens(rng, 150, 8)
    index.segmented_build(toks)
    by_id = {t.token_id: t for t in toks}
    seen = []
    for e in index.entries:
        K = np.stack([by_id[t].key for t in e.member_token_ids]).astype(np.float64)
        V = np.stack([by_id[t].value for t in e.member_token_ids]).astype(np.float64)
        np.testing.assert_allclose(e.centroid, K.mean(axis=0), rtol=1e-5)
        np.testing.assert_allclose(e.value_sum, V.sum(axis=0), rtol=1e-5)
        assert e.size == len(e.member_token_ids)
        seen += e.member_token_ids
    assert sorted(seen) == [t.token_id for t in toks]


def test_build_deterministic_and_matches_oracle(rng):
    from oracle import oracle as O
    K = rng.standard_normal((150, 8)).astype(np.float32)  # :163-176
    V = rng.standard_normal((150, 8)).astype(np.float32)

    def build():
        index, _ = make_index(segment_size=64, centroid_ratio=8, kmeans_iters=4, rng_seed=9)
        index.segmented_build([TokenKV(K[i], V[i], i) for i in range(150)])
        return index

    a, b = build(), build()
    assert np.array_equal(a.centroids, b.centroids) and np.array_equal(a.value_sums, b.value_sums)
    assert all(x.member_token_ids == y.member_token_ids for x, y in zip(a.entries, b.entries))
    # the assignments are tierkv's bits (C oracle, pinned to tierkv)
    for si, s0 in enumerate(range(0, 150, 64)):
        L = min(64, 150 - s0)
        ref = O.spherical_kmeans(K[s0:s0 + L], math.ceil(L / 8), 4, np.random.SeedSequence([9, 1, si]))
        assert np.array_equal(tk.spherical_kmeans(K[s0:s0 + L], math.ceil(L / 8), 4,
                                                  np.random.SeedSequence([9, 1, si])), ref)


def test_index_update(rng):
    index, _ = make_index(update_segment=64, local_window=8, centroid_ratio=16)  # :181-186
    buf = tokens(rng, 50, 8)
    new, kept = index.update(buf)
    assert new == [] and kept == buf
    index, _ = make_index(update_segment=64, local_window=8, centroid_ratio=16, kmeans_iters=3)  # :189-197
    buf = tokens(rng, 72, 8)
    new, kept = index.update(buf)
    assert len(new) == 4 and [t.token_id for t in kept] == [t.token_id for t in buf[64:]]
    assert int(index.sizes.sum()) == 64
    index, _ = make_index(update_segment=32, local_window=8, centroid_ratio=8, kmeans_iters=2)  # :200-212
    buf, total = [], 0
    for i in range(500):
        buf.append(TokenKV(rng.standard_normal(8).astype(np.float32), rng.standard_normal(8).astype(np.float32), i))
        total += 1
        _, buf = index.update(buf)
        assert int(index.sizes.sum()) + len(buf) == total and len(buf) >= min(total, 8)


# ----------------------------------------------------------------- clustering
# pkg/tests/test_clustering.py

def test_spherical_kmeans_contract(rng):
    assert (tk.spherical_kmeans(rng.standard_normal((17, 6)), 1, 5, seed=0) == 0).all()  # :11-13
    with pytest.raises(ConfigError):  # :16-18
        tk.spherical_kmeans(rng.standard_normal((3, 4)), 4, 5, seed=0)
    u = rng.standard_normal(8)  # :21-30
    u /= np.linalg.norm(u)
    keys = np.concatenate([u + 0.01 * rng.standard_normal((10, 8)), -u + 0.01 * rng.standard_normal((10, 8))])
    a = tk.spherical_kmeans(keys, 2, 10, seed=7)
    assert len(set(a[:10])) == 1 and len(set(a[10:])) == 1 and set(a[:10]) != set(a[10:])
    a = tk.spherical_kmeans(np.ones((10, 4)), 2, 5, seed=3)  # :33-40 (degenerate repair)
    assert (np.bincount(a, minlength=2) > 0).all()
    keys = rng.standard_normal((40, 5))  # :43-47
    for k in (2, 7, 15, 40):
        assert (np.bincount(tk.spherical_kmeans(keys, k, 8, seed=k), minlength=k) > 0).all()
    keys = rng.standard_normal((64, 8))  # :50-55
    assert np.array_equal(tk.spherical_kmeans(keys, 6, 10, seed=42), tk.spherical_kmeans(keys, 6, 10, seed=42))


# ---------------------------------------------------------------- block cache
# pkg/tests/test_block_cache.py

def build_cache(rng, sizes, cap, d=8, block=256):
    store = SlowTierStore(d=d, block_size_bytes=block)
    cache = BlockCache(store, capacity_blocks=cap)
    nxt = 0
    for cid, n in enumerate(sizes):
        cache.register_cluster(cid, store.pack_cluster(tokens(rng, n, d, start=nxt)))
        nxt += n
    return store, cache


def run_step(cache, ids, step):
    snap = cache.lookup(ids, step)
    buf = cache.assemble(ids, snap, np.empty((0, 8)), np.empty((0, 8)), [])
    return snap, buf, cache.commit_update(ids, snap, step)


def test_cache_cold_warm_and_zero_capacity(rng):
    _, c = build_cache(rng, [4] * 20, 100)  # :29-34, :37-42
    snap, _, _ = run_step(c, list(range(20)), 0)
    assert not any(snap.values()) and c.misses == 20 and c.hits == 0
    snap, _, _ = run_step(c, list(range(20)), 1)
    assert all(snap.values()) and c.hits == 20
    _, c = build_cache(rng, [4] * 5, 0)  # :45-50
    for step in range(4):
        snap, _, _ = run_step(c, [0, 1, 2], step)
        assert not any(snap.values())
    assert c.hits == 0 and c.occupied_blocks == 0
    _, c = build_cache(rng, [4], 4)  # :53-56
    with pytest.raises(IntegrityError):
        c.lookup([99], 0)


def test_cache_byte_accounting_and_payloads(rng):
    _, c = build_cache(rng, [4, 4], 10)  # :59-64
    run_step(c, [0, 1], 0)
    before = c.bytes_slow_to_fast
    run_step(c, [0, 1], 1)
    assert c.bytes_slow_to_fast == before
    store, c = build_cache(rng, [9, 5, 4], 0)  # :67-72
    run_step(c, [0, 1, 2], 0)
    assert c.bytes_slow_to_fast == 6 * 256 and store.bytes_read_total == c.bytes_slow_to_fast
    _, c = build_cache(rng, [9], 10)  # :75-82
    _, cold, _ = run_step(c, [0], 0)
    _, warm, _ = run_step(c, [0], 1)
    assert cold.spans[0][0] == "slow_miss" and warm.spans[0][0] == "cache_hit"
    assert np.array_equal(cold.keys, warm.keys) and np.array_equal(cold.values, warm.values)
    assert np.array_equal(cold.token_ids, warm.token_ids)


def test_cache_lru_script_reject_and_rank_admission(rng):
    _, c = build_cache(rng, [16, 16, 16], 10)  # :85-95
    run_step(c, [0], 0)
    run_step(c, [1], 1)
    _, _, log = run_step(c, [2], 2)
    assert [(e["type"], e["cluster"]) for e in log] == [("evict", 0), ("admit", 2)]
    assert c.mapping[0].cached is False and c.mapping[1].cached and c.mapping[2].cached
    assert c.occupied_blocks == 8
    _, c = build_cache(rng, [64], 10)  # :98-102
    _, _, log = run_step(c, [0], 0)
    assert [e["type"] for e in log] == ["reject"] and c.occupied_blocks == 0
    _, c = build_cache(rng, [8, 8, 8], 6)  # :105-109
    run_step(c, [0, 1, 2], 0)
    _, _, log = run_step(c, [0, 1, 2], 1)
    assert not [e for e in log if e["type"] == "evict"]
    _, c = build_cache(rng, [8, 8, 8], 4)  # :112-119
    _, _, log = run_step(c, [2, 0, 1], 0)
    assert [e["cluster"] for e in log if e["type"] == "admit"] == [2, 0]
    assert [e["cluster"] for e in log if e["type"] == "reject"] == [1]
    _, c = build_cache(rng, [4, 4], 10)  # :122-128
    run_step(c, [0], 0)
    run_step(c, [1], 1)
    c.lookup([0], 2)
    assert list(c.lru) == [0, 1]


def test_cache_random_workload_invariants(rng):
    _, c = build_cache(rng, [int(rng.integers(1, 20)) for _ in range(30)], 12)  # :131-140
    for step in range(50):
        run_step(c, rng.choice(30, size=int(rng.integers(1, 6)), replace=False).tolist(), step)
        assert c.occupied_blocks <= c.capacity_blocks
        for desc in c.mapping.values():
            if desc.cached:
                assert len(desc.fast_slot_ids) == len(desc.slow_block_ids)
    _, c = build_cache(rng, [8] * 6, 8)  # :143-148
    for step in range(10):
        run_step(c, [step % 6, (step + 1) % 6], step)
    slots = [s for d_ in c.mapping.values() if d_.cached for s in d_.fast_slot_ids]
    assert len(slots) == len(set(slots))


def test_cache_determinism_and_event_replay():
    def run(seed):  # :151-163
        r = np.random.default_rng(seed)
        _, c = build_cache(np.random.default_rng(0), [8] * 10, 6)
        trail = []
        for step in range(40):
            snap, _, log = run_step(c, r.choice(10, size=3, replace=False).tolist(), step)
            trail.append((tuple(sorted(snap.items())), tuple(e["type"] for e in log)))
        return trail, c.stats()

    assert run(7) == run(7)
    _, c = build_cache(np.random.default_rng(1234), [8] * 10, 6)  # :166-180
    r = np.random.default_rng(5)
    for step in range(60):
        run_step(c, r.choice(10, size=3, replace=False).tolist(), step)
    acc = [e for e in c.event_log if e["type"] == "access"]
    hits = sum(sum(e["cached"]) for e in acc)
    misses = sum(len(e["cached"]) - sum(e["cached"]) for e in acc)
    st = c.stats()
    assert st["hits"] == hits and st["misses"] == misses
    assert st["hit_ratio"] == pytest.approx(hits / (hits + misses))


def test_block_cache_matches_oracle_state_machine():
    """The device phases against the C oracle's BlockCache (pinned to tierkv)
    on a random workload: every snapshot, log, LRU order and counter."""
    from oracle import oracle as O
    r = np.random.default_rng(11)
    sizes = [int(r.integers(1, 24)) for _ in range(40)]
    store, c = build_cache(np.random.default_rng(0), sizes, 20)
    ref = O.OracleCache(20, block_size_bytes=256, d=8)
    for cid, n in enumerate(sizes):
        ref.register(cid, -(-n // 4))
    for step in range(80):
        ids = r.choice(40, size=int(r.integers(1, 7)), replace=False).tolist()
        run_step(c, ids, step)
        ref.step(ids, step)
        assert c.lru == list(ref.lru()), step
        assert all(c.mapping[i].cached == bool(ref.is_cached(i)) for i in range(40))
    k = ref.counters()
    assert (c.hits, c.misses, c.bytes_slow_to_fast) == (k["hits"], k["misses"], k["bytes_slow_to_fast"])


# --------------------------------------------------------------------- engine
# pkg/tests/test_engine.py

def test_engine_prefill_shapes_and_accounting():
    tr = Trace(68, 0)  # :34-40
    eng = HeadEngine(small()).prefill(tr.keys, tr.values)
    assert eng.index.m == 0 and eng.n_sink == 4 and len(eng.buffer) == 64 and len(eng._steady_ids()) == 68
    tr = Trace(8260, 0, d=8, seg=8260)  # :43-47
    eng = HeadEngine(small()).prefill(tr.keys, tr.values)
    assert eng.index.m == 512 and int(eng.index.sizes.sum()) == 8192
    tr = Trace(600, 0)  # :50-54
    eng = HeadEngine(small()).prefill(tr.keys, tr.values)
    assert int(eng.index.sizes.sum()) + eng.n_sink + len(eng.buffer) == 600
    with pytest.raises(ConfigError):  # :57-61
        eng.prefill(tr.keys, tr.values)
    with pytest.raises(ConfigError):  # :64-66
        HeadEngine(small()).decode_step(np.zeros(4), np.zeros(4), np.zeros(4))


def test_engine_full_retrieval_matches_oracle():
    tr = Trace(1024, 32, seed=5)  # :69-77
    cfg = EngineConfig(index=IndexConfig(kmeans_iters=3, retrieval_fraction=1.0, estimation_fraction=0.0),
                       cache_fraction=1.0)
    _, rows = tr.run(cfg, with_oracle=True)
    for _, sm in rows:
        assert sm.rel_error <= 1e-5 and sm.e == 0 and sm.r == sm.m


def test_engine_retrieval_nonempty_barrier_and_coverage():
    _, rows = Trace(1024, 8).run(small(retrieval_fraction=1e-4, estimation_fraction=0.1))  # :80-85
    assert all(sm.r >= 1 for _, sm in rows)
    tr = Trace(1024, 2, persistence=1.0, noise=0.01)  # :88-94
    _, rows = tr.run(EngineConfig(index=small(retrieval_fraction=0.1).index, cache_fraction=1.0))
    (_, a), (_, b) = rows
    assert a.hits == 0 and a.misses > 0 and b.misses == 0 and b.hits > 0
    _, rows = Trace(1024, 10).run(small())  # :132-136
    assert all(0.0 < sm.denominator_coverage <= 1.0 for _, sm in rows)


def test_engine_metrics_do_not_change_outputs_and_determinism():
    tr = Trace(512, 12, seed=3)  # :97-103
    _, a = tr.run(small(), with_oracle=True)
    _, b = tr.run(small(), with_oracle=False)
    assert all(np.array_equal(x, y) for (x, _), (y, _) in zip(a, b))
    tr = Trace(512, 12, seed=8)  # :106-113
    _, a = tr.run(small())
    _, b = tr.run(small())
    assert all(np.array_equal(x, y) and sx == sy for (x, sx), (y, sy) in zip(a, b))


def test_engine_update_schedule():
    tr = Trace(512, 1100, seed=2)  # :116-129
    eng, rows = tr.run(small())
    ms = [sm.m for _, sm in rows]
    assert len([t for t in range(1, len(ms)) if ms[t] != ms[t - 1]]) == 1
    assert ms[-1] == ms[0] + math.ceil(1024 / 16)
    assert int(eng.index.sizes.sum()) + eng.n_sink + len(eng.buffer) == eng.total_tokens


def test_engine_eq2_and_tail_modes():
    tr = Trace(1024, 10, seed=6)  # :139-149
    _, m = tr.run(EngineConfig(index=IndexConfig(kmeans_iters=3)))
    _, e = tr.run(EngineConfig(index=IndexConfig(kmeans_iters=3), denominator_mode="eq2"))
    om, oe = np.stack([o for o, _ in m]), np.stack([o for o, _ in e])
    assert np.isfinite(oe).all() and not np.array_equal(om, oe)
    tr = Trace(1024, 10, seed=7)  # :152-158
    _, rows = tr.run(EngineConfig(index=IndexConfig(kmeans_iters=3, tail_mode="denominator_only")),
                     with_oracle=True)
    assert all(np.isfinite(o).all() and sm.rel_error is not None for o, sm in rows)


def test_engine_bytes_accounting():
    eng, rows = Trace(1024, 30, seed=4).run(small())  # :161-166
    total = sum(sm.bytes_slow_to_fast for _, sm in rows)
    assert total == eng.cache.bytes_slow_to_fast and total % eng.store.block_size_bytes == 0
    assert eng.store.bytes_read_total == total


def test_engine_grows_past_its_initial_decode_capacity():
    """tierkv has no decode-length limit: the engine doubles its capacity
    (state copied) and keeps matching the oracle across the growth."""
    from oracle import oracle as O
    tr = Trace(600, 300, seed=12)
    eng = HeadEngine(small(update_segment=128), max_decode=64, blas_threads=1).prefill(tr.keys, tr.values)
    orc = O.OracleEngine(kmeans_iters=3, update_segment=128).prefill(tr.keys, tr.values)
    for t in range(300):
        out, sm = eng.decode_step(tr.q[t], tr.nk[t], tr.nv[t])
        o_ref, m_ref = orc.decode_step(tr.q[t], tr.nk[t], tr.nv[t], with_recall=True)
        assert (sm.m, sm.r, sm.e, sm.hits, sm.misses) == (m_ref.m, m_ref.r, m_ref.e, m_ref.hits, m_ref.misses), t
        assert np.linalg.norm(out - o_ref) <= 1e-5 * np.linalg.norm(o_ref), t
    assert eng.max_decode >= 300


# ----------------------------------------------------------------- acceptance
# pkg/tests/test_acceptance.py

def test_criterion_01_centroid_weight_bound():
    """:52-89, reduced from 50 builds x 1000 queries to 4 x 200."""
    worst = 0
    for seed in range(4):
        tr = Trace(32768, 0, d=64, seed=seed)
        index, _ = make_index(d=64, block=2048, kmeans_iters=2, rng_seed=seed)
        entries = index.segmented_build([TokenKV(tr.keys[i], tr.values[i], i) for i in range(len(tr.keys))])
        K = tr.keys.astype(np.float64)
        qs = np.random.default_rng(seed + 1000).standard_normal((200, 64))
        ks = qs @ K.T / 8.0
        mx = ks.max(axis=1, keepdims=True)
        w = np.exp(ks - mx)
        for e in entries:
            rhs = w[:, e.member_token_ids].mean(axis=1)
            lhs = np.exp(qs @ e.centroid / 8.0 - mx[:, 0])
            worst += int((lhs > rhs * (1 + 1e-5)).sum())
    assert worst == 0


def test_criterion_02_full_coverage_exactness():
    """:92-107: retrieval covers every cluster -> 256 steps within 1e-5."""
    tr = Trace(32768, 256, d=64, seed=2)
    cfg = EngineConfig(index=IndexConfig(retrieval_fraction=1.0, estimation_fraction=0.0), cache_fraction=1.0)
    _, rows = tr.run(cfg, with_oracle=True)
    assert max(sm.rel_error for _, sm in rows) <= 1e-5


def test_criterion_03_partition_merge_exactness():
    r = np.random.default_rng(42)  # :110-128
    worst = 0.0
    for _ in range(200):
        n, d = int(r.integers(1, 400)), int(r.integers(4, 65))
        K, V, q = r.standard_normal((n, d)), r.standard_normal((n, d)), r.standard_normal(d)
        pieces = np.array_split(r.permutation(n), int(r.integers(1, min(n, 12) + 1)))
        out = merge([exact_partial(q, K[p], V[p]) for p in pieces]).output
        worst = max(worst, tk.relative_l2(out, oracle_attention(q, K, V)))
    assert worst <= 1e-6


def test_criterion_04_denominator_bound():
    tr = Trace(32768, 256, d=64, seed=2)  # :131-149
    eng = HeadEngine(EngineConfig(index=IndexConfig())).prefill(tr.keys, tr.values)
    worst = -np.inf
    for t in range(tr.n_decode):
        q = tr.q[t].astype(np.float64)
        _, sm = eng.decode_step(q, tr.nk[t], tr.nv[t])
        s = eng._keys[: eng.total_tokens].astype(np.float64) @ q / 8.0
        worst = max(worst, sm.log_denominator - (s.max() + np.log(np.exp(s - s.max()).sum())))
    assert worst <= math.log1p(1e-5)


def test_criterion_05_estimation_benefit():
    """:152-169 through the trace runner (one batched layer)."""
    from paper_2505_02922_b200.tracefile import TraceFile
    red = []
    for seed in (3, 4):
        t = Trace(8192, 256, d=64, seed=seed, heavy_tail=0.5)
        trace = TraceFile(64, t.keys[None], t.values[None], t.q[:, None], t.nk[:, None], t.nv[:, None])
        errs = {}
        for frac in (0.0, 0.232):
            cfg = EngineConfig(index=IndexConfig(kmeans_iters=4, estimation_fraction=frac, tail_mode="drop"))
            report, _, _ = tk.run_trace(trace, cfg, with_oracle=True)
            errs[frac] = report["aggregates"]["mean_rel_error"]
        red.append(1.0 - errs[0.232] / errs[0.0])
    assert min(red) >= 0.20, red


def _hit_steps(persistence, frac, noise=0.25):
    t = Trace(8192, 192, d=64, seed=5, persistence=persistence, noise=noise)
    eng, rows = t.run(EngineConfig(index=IndexConfig(), cache_fraction=frac))
    return [sm.hits for _, sm in rows], [sm.misses for _, sm in rows]


def test_criterion_07_cache_hit_ratio_regimes():
    h, m = _hit_steps(0.9, 0.05)  # :189-223
    warm = sum(h[64:]) / (sum(h[64:]) + sum(m[64:]))
    h, m = _hit_steps(1.0, 1.0, noise=0.01)
    steady = sum(h[64:]) / (sum(h[64:]) + sum(m[64:]))
    h, m = _hit_steps(0.9, 0.0)
    empty = sum(h) / (sum(h) + sum(m))
    assert warm >= 0.5 and steady == 1.0 and empty == 0.0, (warm, steady, empty)


def test_criterion_08_transfer_accounting():
    t = Trace(4096, 80, d=32, seed=11, persistence=0.7)  # :226-249
    eng = HeadEngine(EngineConfig(index=IndexConfig(kmeans_iters=4), cache_fraction=0.05))
    eng.prefill(t.keys, t.values)
    for s in range(t.n_decode):
        eng.decode_step(t.q[s], t.nk[s], t.nv[s])
    missed = 0
    for ev in eng.cache.event_log:
        if ev["type"] == "access":
            missed += sum(len(eng.cache.mapping[c].slow_block_ids)
                          for c, hit in zip(ev["clusters"], ev["cached"]) if not hit)
    expected = missed * eng.store.block_size_bytes
    assert eng.cache.bytes_slow_to_fast == expected == eng.store.bytes_read_total


def test_criterion_09_estimation_cost_scaling():
    r = np.random.default_rng(9)  # :252-282
    ev, counts = [64, 256, 1024, 4096], []
    for e in ev:
        C, VS, sz = r.standard_normal((e, 64)), r.standard_normal((e, 64)), r.integers(1, 64, size=e)
        estimation_ops.reset()
        for _ in range(16):
            estimate_partial(r.standard_normal(64), C, VS, sz)
        counts.append(estimation_ops.count)
    fit = np.polyval(np.polyfit(ev, counts, 1), ev)
    assert float(np.max(np.abs(fit - counts) / np.asarray(counts))) < 0.05
    C, VS, sz, q = r.standard_normal((1024, 64)), r.standard_normal((1024, 64)), r.integers(1, 64, 1024), r.standard_normal(64)
    estimation_ops.reset()
    estimate_partial(q, C, VS, sz)
    base = estimation_ops.count
    estimation_ops.reset()
    estimate_partial(q, C, 2.0 * VS, 2 * sz)
    assert base == estimation_ops.count


def test_criterion_11_index_update_accounting():
    t = Trace(512, 3000, d=32, seed=23, seg=512)  # :310-334
    eng = HeadEngine(EngineConfig(index=IndexConfig(kmeans_iters=4))).prefill(t.keys, t.values)
    m_prev, updates, ok = eng.index.m, 0, True
    for s in range(t.n_decode):
        _, sm = eng.decode_step(t.q[s], t.nk[s], t.nv[s])
        if sm.m != m_prev:
            updates, m_prev = updates + 1, sm.m
        ok &= int(eng.index.sizes.sum()) + eng.n_sink + len(eng.buffer) == eng.total_tokens
    assert updates == 2 and ok
