"""GPU: the offload path (config 4) -- cluster store in pinned host memory, the
wave buffer as an HBM slot arena managed on the device (cache_v2.cu).

* outputs equal the all-in-HBM path (same zones; only the chunk order of the
  fp32 accumulation differs) and the CPU oracle within the stated tolerance;
* the device cache is state-equivalent to tierkv's BlockCache
  (block_cache.py:79-213) driven by the same union access stream: hits,
  misses, byte counters, occupancy, LRU order and residency, step by step --
  including capacities small enough to force rejections."""
import math

import numpy as np
import pytest
import torch

from tests import golden_util as Gu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _data(U, n, d, seed):
    rng = np.random.default_rng(seed)
    cen = rng.standard_normal((48, d)).astype(np.float32)
    keys = Gu.bf16_round(cen[rng.integers(48, size=(U, n))] + 0.3 * rng.standard_normal((U, n, d)).astype(np.float32))
    vals = Gu.bf16_round(rng.standard_normal((U, n, d)).astype(np.float32))
    return rng, keys, vals


@pytest.mark.parametrize("frac", [0.05, 0.004])
def test_offload_matches_hbm_path_and_reference_cache(frac):
    from oracle import oracle as O
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    U, G, d, n, steps = 2, 4, 128, 6000, 24
    rng, keys, vals = _data(U, n, d, 3)
    cfg = EngineConfig.from_dict({"cache_fraction": frac})
    dev = torch.device("cuda")
    lay_h = WaveLayer(cfg, U, G, d, max_prefill=n, max_decode=64)
    lay_o = WaveLayer(cfg, U, G, d, max_prefill=n, max_decode=64, offload=True)
    for lay in (lay_h, lay_o):
        lay.prefill(torch.from_numpy(keys).to(dev), torch.from_numpy(vals).to(dev))
    c = lay_o.cache
    # reference caches fed with the device's union access stream
    ref = []
    for u in range(U):
        nb = c.nblk[u, :lay_o.units[u].m].cpu().numpy()
        oc = O.OracleCache(0, cfg.block_size_bytes, d)
        sink_blocks = math.ceil(lay_o.units[u].n_sink / c.bt)
        for cid, b in enumerate(nb):
            oc.register(cid, int(b))
        total = sink_blocks + int(nb.sum())
        oc.set_capacity(math.ceil(frac * total))
        assert int(c.capacity[u]) == math.ceil(frac * total)
        ref.append(oc)
    qs = Gu.bf16_round(rng.standard_normal((steps, U, G, d)).astype(np.float32))
    nk = Gu.bf16_round(rng.standard_normal((steps, U, d)).astype(np.float32))
    nv = Gu.bf16_round(rng.standard_normal((steps, U, d)).astype(np.float32))
    for t in range(steps):
        q, k, v = (torch.from_numpy(x[t]).to(dev) for x in (qs, nk, nv))
        out_h, ld_h, _ = lay_h.decode(q, k, v)
        out_o, ld_o, _ = lay_o.decode(q, k, v)
        lay_h.check_status()
        lay_o.check_status()
        a, b = out_o.double().cpu().numpy(), out_h.double().cpu().numpy()
        assert np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(b), t
        assert torch.allclose(ld_o, ld_h, atol=1e-6)
        for u in range(U):
            ids = c.ids[u, :int(c.n_ids[u])].cpu().numpy()
            snap = ref[u].step(ids, t, int(lay_o.st_n[u]))
            assert np.array_equal(snap, c.snapshot[u, :len(ids)].cpu().numpy().astype(bool)), (t, u)
            rc = ref[u].counters()
            mine = c.stats(u)
            for key in ("hits", "misses", "bytes_slow_to_fast", "bytes_fast_internal"):
                assert mine[key] == rc[key], (t, u, key, mine[key], rc[key])
            assert mine["occupied_blocks"] == rc["occupied_blocks"], (t, u)
            assert np.array_equal(c.lru[u, :int(c.lru_n[u])].cpu().numpy(), ref[u].lru()), (t, u)
    tot = c.totals()
    assert tot["hits"] > 0 and tot["misses"] > 0
    if frac < 0.01:
        assert tot["rejections"] > 0 or tot["evictions"] > 0


def test_offload_long_rank_ordered_pieces():
    """Offload attention reads the retrieval zone as rank-ordered pieces (one
    cluster each), so one consumer folds thousands of small chunk terms into a
    running sum that the first (top-ranked) chunks made large.  256K context,
    10% retrieval, one attention CTA: the output must stay within the fp64
    bar (the tensor-core accumulate truncates: accumulating there biased the
    output by 1.7e-5 here; with per-chunk accumulators and fp32 adds 4.5e-7)."""
    from oracle import oracle as O
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    from paper_2505_02922_b200.config import IndexConfig
    rng = np.random.default_rng(256)
    n, d, Gh, steps = 262144, 128, 4, 2
    cen = rng.standard_normal((64, d)).astype(np.float32)
    keys = Gu.bf16_round(cen[rng.integers(64, size=(1, n))] + 0.5 * rng.standard_normal((1, n, d)).astype(np.float32))
    vals = Gu.bf16_round(rng.standard_normal((1, n, d)).astype(np.float32))
    qs = Gu.bf16_round(rng.standard_normal((steps, 1, Gh, d)).astype(np.float32))
    nk = Gu.bf16_round(rng.standard_normal((steps, 1, d)).astype(np.float32))
    nv = Gu.bf16_round(rng.standard_normal((steps, 1, d)).astype(np.float32))
    cfg = EngineConfig(index=IndexConfig(retrieval_fraction=0.1))
    lay = WaveLayer(cfg, 1, Gh, d, max_prefill=n, max_decode=64, offload=True, splits=1, blas_threads=8)
    dev = torch.device("cuda")
    lay.prefill(torch.from_numpy(keys).to(dev), torch.from_numpy(vals).to(dev))
    e0 = O.OracleEngine(blas_threads=8, retrieval_fraction=0.1).prefill(keys[0], vals[0])
    orcs = [e0] + [e0.clone() for _ in range(Gh - 1)]
    for t in range(steps):
        out, logden, _ = lay.decode(torch.from_numpy(qs[t]).to(dev), torch.from_numpy(nk[t]).to(dev),
                                    torch.from_numpy(nv[t]).to(dev))
        lay.check_status()
        out = out.double().cpu().numpy()
        for h in range(Gh):
            o_ref, sm = orcs[h].decode_step(qs[t, 0, h], nk[t, 0], nv[t, 0], with_recall=False)
            rel = np.linalg.norm(out[0, h] - o_ref) / np.linalg.norm(o_ref)
            assert rel <= 3e-6, (t, h, rel)
            assert abs(float(logden[0, h]) - sm.log_denominator) <= 1e-5
