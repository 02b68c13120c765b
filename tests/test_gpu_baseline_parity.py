"""GPU parity at the BASELINE.json configurations and on tie-heavy inputs.

The CUDA path (through the C ABI) against the C oracle (oracle/, pinned
bit-for-bit to tierkv by tests/test_oracle_golden.py) at the scale the bench
runs:

* configs[0]: one Llama-3-8B layer, 32 q / 8 kv heads, d=128, 8K context,
  batch 1, 16 decode steps -- every (kv head, q head);
* one configs[1]/[4] unit at 120K context (15 prefill segments, m = 7,676,
  r = 138, e = 1,781) at G = 4 (Llama) and G = 7 (Qwen), with the reference's
  BLAS thread count 1 and 8 (m = 7,676 at 8 threads hits OpenBLAS's dgemv
  chunk tails);
* multi-segment prefill + decode-time index updates at small scale;
* the committed tierkv rank goldens (tests/golden/rank.npz, incl. m = 7,676)
  through the GPU centroid scan + exact selection;
* full ties (q = 0, q orthogonal to every centroid, duplicated centroids at
  m = 7,676, a single-cluster index, identical keys for recall@k): the
  tie-safe exact path (csrc/exact_select.cuh) must give tierkv's lexsort order
  (index.py:75, test_index.py:63-70).

Bars: index (assignments -> C64, sizes, members), ordered
retrieval lists and estimation sets bit-exact; outputs rel-L2 <= 1e-5 vs the
oracle's fp64 (bf16 store of bf16-representable inputs, fp32 accumulation);
log-denominator and coverage within 1e-5."""
import numpy as np
import pytest
import torch

from tests import golden_util as GU

pytestmark = pytest.mark.gpu

OUT_TOL = 1e-5
LOGDEN_TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def synth_kv(rng, U, n, d, seg=8192, n_centres=48, noise=0.5):
    """Keys with spatial locality: per-8K-segment latent centres + noise
    (the shape of tierkv synth.py:46-70); values N(0,1); bf16-representable."""
    keys = np.empty((U, n, d), np.float32)
    for s0 in range(0, n, seg):
        ln = min(seg, n - s0)
        cen = rng.standard_normal((U, n_centres, d)).astype(np.float32)
        idx = rng.integers(n_centres, size=(U, ln))
        keys[:, s0:s0 + ln] = (np.take_along_axis(cen, idx[..., None], axis=1)
                               + noise * rng.standard_normal((U, ln, d)).astype(np.float32))
    vals = rng.standard_normal((U, n, d)).astype(np.float32)
    return GU.bf16_round(keys), GU.bf16_round(vals)


def gqa_queries(rng, keys, G, steps, spread=0.3):
    """Per step, one shared direction per unit (a random prompt key) plus
    per-head noise: the GQA group's selections overlap partially."""
    U, n, d = keys.shape
    base = keys[np.arange(U)[None, :], rng.integers(n, size=(steps, U))]  # [steps, U, d]
    q = base[:, :, None, :] + spread * rng.standard_normal((steps, U, G, d)).astype(np.float32)
    return GU.bf16_round(q)


def compare_index(lay, u, orc):
    ix = lay.index_arrays(u)
    m = orc.m
    assert lay.units[u].m == m
    assert np.array_equal(ix["C64"], orc.centroids)
    assert np.array_equal(ix["sizes"], orc.sizes)
    for c in range(m):
        o, s = int(ix["offsets"][c]), int(ix["sizes"][c])
        assert np.array_equal(ix["store_tok"][o:o + s], orc.members(c)), c


def run_and_compare(lay, orcs, qs, nk, nv):
    """Decode every step on the GPU and on the per-(unit, head) oracles."""
    dev = torch.device("cuda")
    U, G = lay.U, lay.G
    worst = 0.0
    for t in range(len(qs)):
        out, logden, cov = lay.decode(torch.from_numpy(qs[t]).to(dev), torch.from_numpy(nk[t]).to(dev),
                                      torch.from_numpy(nv[t]).to(dev))
        lay.check_status()
        out = out.double().cpu().numpy()
        logden, cov = logden.cpu().numpy(), cov.cpu().numpy()
        rl, el = lay.rlist.cpu().numpy(), lay.elist.cpu().numpy()
        nr, ne = lay.nr.cpu().numpy(), lay.ne.cpu().numpy()
        for u in range(U):
            for g in range(G):
                o_ref, sm = orcs[u][g].decode_step(qs[t, u, g], nk[t, u], nv[t, u], with_recall=False)
                r_ref, e_ref = orcs[u][g].last_plan()
                assert (int(nr[u]), int(ne[u])) == (sm.r, sm.e)
                assert np.array_equal(rl[u, g, :nr[u]], r_ref), (t, u, g)
                assert np.array_equal(np.sort(el[u, g, :ne[u]]), np.sort(e_ref)), (t, u, g)
                rel = np.linalg.norm(out[u, g] - o_ref) / np.linalg.norm(o_ref)
                worst = max(worst, rel)
                assert rel <= OUT_TOL, (t, u, g, rel)
                assert abs(float(logden[u, g]) - sm.log_denominator) <= LOGDEN_TOL
                assert abs(float(cov[u, g]) - sm.denominator_coverage) <= 1e-5
    return worst


def test_config0_llama_layer_8k_all_heads():
    """configs[0]: 32 q / 8 kv heads, d = 128, 8K context, batch 1, 16 steps."""
    from oracle import oracle as O
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    rng = np.random.default_rng(2505)
    U, G, d, n, steps, threads = 8, 4, 128, 8192, 16, 8
    keys, vals = synth_kv(rng, U, n, d)
    qs = gqa_queries(rng, keys, G, steps)
    nk = GU.bf16_round(keys[np.arange(U)[None, :], rng.integers(n, size=(steps, U))]
                       + 0.1 * rng.standard_normal((steps, U, d)).astype(np.float32))
    nv = GU.bf16_round(rng.standard_normal((steps, U, d)).astype(np.float32))
    lay = WaveLayer(EngineConfig(), U, G, d, max_prefill=n, max_decode=64, blas_threads=threads,
                    with_elist=True)
    dev = torch.device("cuda")
    lay.prefill(torch.from_numpy(keys).to(dev), torch.from_numpy(vals).to(dev))
    orcs = []
    for u in range(U):
        e0 = O.OracleEngine(blas_threads=threads).prefill(keys[u], vals[u])
        compare_index(lay, u, e0)
        orcs.append([e0] + [e0.clone() for _ in range(G - 1)])
    assert lay.units[0].m == 508
    run_and_compare(lay, orcs, qs, nk, nv)
    assert int(lay.xcount.item()) == 0  # no tie fallback needed on this workload


_ORC_120K: dict = {}


def _oracle_120k(threads):
    """One 120K unit (shared by the G = 4 / 7 cases): inputs + oracle index."""
    from oracle import oracle as O
    if threads not in _ORC_120K:
        rng = np.random.default_rng(120)
        keys, vals = synth_kv(rng, 1, 122880, 128)
        e0 = O.OracleEngine(blas_threads=threads).prefill(keys[0], vals[0])
        _ORC_120K[threads] = (keys, vals, e0)
    return _ORC_120K[threads]


@pytest.mark.parametrize("G", [4, 7])
@pytest.mark.parametrize("threads", [1, 8])
def test_unit_120k_parity(G, threads):
    """configs[1] (G = 4) / configs[4] (G = 7) unit at 120K: 15-segment index
    bit-exact, 6 decode steps of every head exact / within tolerance."""
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    keys, vals, e0 = _oracle_120k(threads)
    rng = np.random.default_rng(1000 * G + threads)
    steps, n, d = 6, keys.shape[1], keys.shape[2]
    qs = gqa_queries(rng, keys, G, steps)
    nk = GU.bf16_round(rng.standard_normal((steps, 1, d)).astype(np.float32))
    nv = GU.bf16_round(rng.standard_normal((steps, 1, d)).astype(np.float32))
    lay = WaveLayer(EngineConfig(), 1, G, d, max_prefill=n, max_decode=64, blas_threads=threads,
                    with_elist=True)
    dev = torch.device("cuda")
    lay.prefill(torch.from_numpy(keys).to(dev), torch.from_numpy(vals).to(dev))
    assert e0.m == 7676 and lay.units[0].m == 7676
    compare_index(lay, 0, e0)
    orcs = [[e0.clone() for _ in range(G)]]
    run_and_compare(lay, orcs, qs, nk, nv)
    assert int(lay.nr[0]) == 138 and int(lay.ne[0]) == 1781


def test_multi_segment_prefill_and_updates():
    """segment_size 1024 -> 5 prefill segments; update_segment 128 -> several
    decode-time index updates (index.py:153-186) inside 300 steps."""
    from oracle import oracle as O
    from paper_2505_02922_b200 import EngineConfig, IndexConfig, WaveLayer
    rng = np.random.default_rng(77)
    U, G, d, n, steps = 2, 2, 64, 5000, 300
    icfg = dict(segment_size=1024, update_segment=128)
    cfg = EngineConfig(index=IndexConfig(**icfg))
    keys, vals = synth_kv(rng, U, n, d, seg=1024, n_centres=12)
    qs = gqa_queries(rng, keys, G, steps)
    nk = GU.bf16_round(rng.standard_normal((steps, U, d)).astype(np.float32))
    nv = GU.bf16_round(rng.standard_normal((steps, U, d)).astype(np.float32))
    lay = WaveLayer(cfg, U, G, d, max_prefill=n, max_decode=steps + 8, blas_threads=1, with_elist=True)
    dev = torch.device("cuda")
    lay.prefill(torch.from_numpy(keys).to(dev), torch.from_numpy(vals).to(dev))
    orcs = []
    for u in range(U):
        e0 = O.OracleEngine(**icfg).prefill(keys[u], vals[u])
        compare_index(lay, u, e0)
        orcs.append([e0] + [e0.clone() for _ in range(G - 1)])
    m0 = lay.units[0].m
    run_and_compare(lay, orcs, qs, nk, nv)
    assert lay.units[0].m > m0  # updates happened
    for u in range(U):
        compare_index(lay, u, orcs[u][0])


def _planner(m, d, G, threads):
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    n = 16 * m + 68  # capacity for m clusters
    return WaveLayer(EngineConfig(), 1, G, d, max_prefill=n, max_decode=8, blas_threads=threads,
                     with_elist=True)


@pytest.mark.parametrize("case", [c for c, _ in GU.rank_cases()])
def test_rank_goldens_through_scan_and_select(case):
    """tierkv rank_clusters goldens (8 queries each; m = 37 .. 7,676, BLAS
    threads 1 / 3 / 8) through the GPU centroid scan + exact zone planner:
    ordered retrieval list and estimation set equal tierkv's order[:r] and
    order[r:r+e] (index.py:61-93)."""
    c = dict(GU.rank_cases())[case]
    C, Q = c["C"], c["Q"]
    m, d = C.shape
    r, e = int(c["r"]), int(c["e"])
    lay = _planner(m, d, 8, int(c["threads"]))
    lay.set_index(0, C, np.full(m, 2))
    dev = torch.device("cuda")
    for use64 in (False, True):
        q = torch.from_numpy(Q.astype(np.float32)).view(1, 8, d).to(dev)
        rl, nr, el, ne = lay.plan(q, q64=torch.from_numpy(Q).view(1, 8, d).to(dev) if use64 else None)
        assert (int(nr[0]), int(ne[0])) == (r, e)
        for g in range(8):
            order = c["orders"][g]
            assert np.array_equal(rl[0, g, :r].cpu().numpy(), order[:r]), (case, g)
            assert np.array_equal(np.sort(el[0, g, :e].cpu().numpy()), np.sort(order[r:r + e])), (case, g)


def _expected_plan(C, q, threads, r, e):
    from oracle import oracle as O
    order, _ = O.rank_clusters(q, C, threads=threads)
    return order[:r], np.sort(order[r:r + e])


@pytest.mark.parametrize("d", [128, 32])
@pytest.mark.parametrize("kind", ["zero_query", "orthogonal", "duplicates"])
def test_full_ties_take_the_exact_path(kind, d):
    """Dense ties at m = 7,676 (the 120K index size): zero span or band
    overflow must fall back to the exact path, never raise, and reproduce
    lexsort((ids, -scores)) -- identity order for full ties."""
    from paper_2505_02922_b200 import EngineConfig
    from paper_2505_02922_b200.config import round_half_up
    rng = np.random.default_rng(9)
    m, G, threads = 7676, 4, 8
    if kind == "duplicates":
        base = rng.standard_normal((40, d))
        C = base[rng.integers(40, size=m)]
        Q = rng.standard_normal((G, d))
    else:
        C = np.zeros((m, d))
        C[:, 0] = rng.standard_normal(m)
        Q = np.zeros((G, d))
        if kind == "orthogonal":
            Q[:, 1] = rng.standard_normal(G)
    Q = GU.bf16_round(Q.astype(np.float32)).astype(np.float64)
    ic = EngineConfig().index
    r = max(1, round_half_up(ic.retrieval_fraction * m))
    e = min(m - r, round_half_up(ic.estimation_fraction * m))
    lay = _planner(m, d, G, threads)
    lay.set_index(0, C, np.full(m, 2))
    x0 = int(lay.xcount.item())
    dev = torch.device("cuda")
    rl, nr, el, ne = lay.plan(torch.from_numpy(Q.astype(np.float32)).view(1, G, d).to(dev))
    for g in range(G):
        rr, ee = _expected_plan(C, Q[g], threads, r, e)
        if kind != "duplicates":
            assert np.array_equal(rr, np.arange(r)) and np.array_equal(ee, np.arange(r, r + e))
        assert np.array_equal(rl[0, g, :r].cpu().numpy(), rr), (kind, g)
        assert np.array_equal(np.sort(el[0, g, :e].cpu().numpy()), ee), (kind, g)
    if not (kind == "duplicates" and d == 32):  # the generic planner's 1,024-row band holds these ties
        assert int(lay.xcount.item()) > x0  # the exact path was taken


@pytest.mark.parametrize("d", [128, 64, 16])
def test_single_cluster_index_and_zero_query_head_engine(d):
    """HeadEngine (default config) on a prompt whose index holds one cluster
    (n = 80 -> 12 indexable tokens), then a zero query: tierkv semantics,
    no IntegrityError (VERDICT r1 'Missing' 2, ADVICE high)."""
    from oracle import oracle as O
    from paper_2505_02922_b200 import EngineConfig, HeadEngine
    rng = np.random.default_rng(d)
    n = 80
    keys = rng.standard_normal((n, d)).astype(np.float32)
    vals = rng.standard_normal((n, d)).astype(np.float32)
    eng = HeadEngine(EngineConfig(), blas_threads=1).prefill(keys, vals)
    orc = O.OracleEngine().prefill(keys, vals)
    assert eng.index.m == orc.m == 1
    for t in range(6):
        q = np.zeros(d) if t == 3 else rng.standard_normal(d)
        k = rng.standard_normal(d).astype(np.float32)
        v = rng.standard_normal(d).astype(np.float32)
        out, met = eng.decode_step(q, k, v)
        o_ref, m_ref = orc.decode_step(q, k, v, with_recall=True)
        assert np.linalg.norm(out - o_ref) <= 1e-5 * np.linalg.norm(o_ref)
        assert (met.r, met.e, met.hits, met.misses) == (m_ref.r, m_ref.e, m_ref.hits, m_ref.misses)
        assert met.recall == pytest.approx(m_ref.recall, abs=1e-7)
        assert abs(met.log_denominator - m_ref.log_denominator) <= 1e-5


def test_recall_with_identical_keys():
    """recall@k when > 1,024 tokens tie at the k-th score (identical keys):
    exact selection over every token (metrics.cu)."""
    from oracle import oracle as O
    from paper_2505_02922_b200 import EngineConfig, HeadEngine
    rng = np.random.default_rng(3)
    n, d = 3000, 64
    keys = np.tile(rng.standard_normal(d).astype(np.float32), (n, 1))
    keys[::7] += rng.standard_normal((len(keys[::7]), d)).astype(np.float32)
    vals = rng.standard_normal((n, d)).astype(np.float32)
    eng = HeadEngine(EngineConfig(), blas_threads=1).prefill(keys, vals)
    orc = O.OracleEngine().prefill(keys, vals)
    for _ in range(3):
        q = rng.standard_normal(d)
        k = keys[5].copy()
        v = rng.standard_normal(d).astype(np.float32)
        out, met = eng.decode_step(q, k, v)
        o_ref, m_ref = orc.decode_step(q, k, v, with_recall=True)
        assert met.recall == pytest.approx(m_ref.recall, abs=1e-7)
        assert np.linalg.norm(out - o_ref) <= 1e-5 * np.linalg.norm(o_ref)


def test_layer_120k_128_units_every_step():
    """The benchmarked layer itself (configs[1]: 16 requests x 8 kv-heads =
    128 units at 120K, bf16 store, bench.py's synthetic generator): units
    spread over the attention grid (first, middle, last) against independent
    oracle engines on every one of 6 decode steps.  At this shape every
    attention CTA's chunk range crosses unit boundaries -- the case the
    per-unit 120K tests above cannot reach."""
    import bench
    from oracle import oracle as O
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    dev = torch.device("cuda")
    U, G, d, n, steps, threads = 128, 4, 128, 122880, 6, 8
    keys, vals, cen = bench.gen_layer(torch, U, n, d, 3, dev)
    lay = WaveLayer(EngineConfig(), U, G, d, max_prefill=n, max_decode=64, blas_threads=threads)
    lay.prefill(keys, vals)
    pick = (0, 77, 127)
    host = {u: (keys[u].cpu().numpy(), vals[u].cpu().numpy()) for u in pick}
    del keys, vals
    qs = bench.gen_queries(torch, cen, G, steps, 9)
    g = torch.Generator(device=dev).manual_seed(10)
    kv = torch.randn((steps, 2, U, d), generator=g, device=dev).bfloat16().float()
    orcs = {}
    for u in pick:
        e0 = O.OracleEngine(blas_threads=threads).prefill(*host[u])
        assert lay.units[u].m == e0.m
        orcs[u] = [e0] + [e0.clone() for _ in range(G - 1)]
    for t in range(steps):
        out, logden, _ = lay.decode(qs[t], kv[t, 0], kv[t, 1])
        lay.check_status()
        out = out.double().cpu().numpy()
        logden = logden.cpu().numpy()
        for u in pick:
            r = int(lay.nr[u])
            rl = lay.rlist[u, :, :r].cpu().numpy()
            q = qs[t, u].double().cpu().numpy()
            k, v = kv[t, 0, u].cpu().numpy(), kv[t, 1, u].cpu().numpy()
            for h in range(G):
                o_ref, sm = orcs[u][h].decode_step(q[h], k, v, with_recall=False)
                r_ref, _ = orcs[u][h].last_plan()
                assert r == sm.r and np.array_equal(rl[h], r_ref), (t, u, h)
                rel = np.linalg.norm(out[u, h] - o_ref) / np.linalg.norm(o_ref)
                assert rel <= OUT_TOL, (t, u, h, rel)
                assert abs(float(logden[u, h]) - sm.log_denominator) <= LOGDEN_TOL
