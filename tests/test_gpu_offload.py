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
