"""GPU parity: the CUDA path (through the C ABI) vs the oracle / tierkv goldens.

Bars: cluster assignments, centroids (fp64), retrieval lists (ordered) and
estimation sets are bit-exact; attention outputs agree with the reference's
fp64 outputs within rel-L2 <= 1e-5 (fp32 accumulation), log-denominator and
coverage within 1e-5 absolute."""
import numpy as np
import pytest
import torch

from tests import golden_util as G

pytestmark = pytest.mark.gpu

OUT_TOL = 1e-5
LOGDEN_TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("name", G.manifest()["files"]["kmeans"])
def test_kmeans_bit_exact_vs_reference(name):
    from paper_2505_02922_b200 import spherical_kmeans
    z = G.load(name)
    a = spherical_kmeans(z["keys"], int(z["k"]), int(z["iters"]),
                         np.random.SeedSequence([int(x) for x in z["seed"]]),
                         threads=int(z["threads"]))
    assert np.array_equal(a.astype(np.int32), z["assignment"])


def _layer_from_golden(name, store_dtype=torch.float32):
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    z, cfgd = G.engine_case(name)
    cfg = EngineConfig.from_dict(cfgd)
    n = len(z["prefill_keys"])
    lay = WaveLayer(cfg, 1, 1, z["prefill_keys"].shape[1], max_prefill=n,
                    max_decode=len(z["queries"]) + 8, store_dtype=store_dtype,
                    blas_threads=int(z["threads"]), keep_vs64=True, with_elist=True)
    dev = torch.device("cuda")
    lay.prefill(torch.from_numpy(z["prefill_keys"])[None].to(dev),
                torch.from_numpy(z["prefill_values"])[None].to(dev))
    return z, lay


@pytest.mark.parametrize("name", G.manifest()["files"]["engine"])
@pytest.mark.parametrize("store", ["f32", "bf16"])
def test_engine_trace_matches_reference(name, store):
    dt = torch.float32 if store == "f32" else torch.bfloat16
    z, lay = _layer_from_golden(name, dt)
    ix = lay.index_arrays(0)
    assert np.array_equal(ix["C64"], z["centroids0"])
    assert np.array_equal(ix["VS64"], z["value_sums0"])
    assert np.array_equal(ix["sizes"], z["sizes0"])
    # members: store rows of cluster c are its member token ids in ascending order
    mem = G.split(z["members0"], np.diff(z["members0_off"]))
    for c, mref in enumerate(mem):
        o, s = int(ix["offsets"][c]), int(ix["sizes"][c])
        assert np.array_equal(ix["store_tok"][o:o + s], mref)
    rids = G.split(z["retrieval_flat"], z["retrieval_len"])
    eids = G.split(z["estimation_flat"], z["estimation_len"])
    dev = torch.device("cuda")
    worst = 0.0
    for t in range(len(z["queries"])):
        q = torch.from_numpy(z["queries"][t]).to(dev).view(1, 1, -1)
        k = torch.from_numpy(z["new_keys"][t]).to(dev).view(1, -1)
        v = torch.from_numpy(z["new_values"][t]).to(dev).view(1, -1)
        out, logden, cov = lay.decode(q, k, v)
        lay.check_status()
        ref = z["metrics"][t]
        r = int(lay.nr[0]); e = int(lay.ne[0])
        assert (r, e) == (int(ref[10]), int(ref[11]))
        assert np.array_equal(lay.rlist[0, 0, :r].cpu().numpy(), rids[t])
        assert np.array_equal(np.sort(lay.elist[0, 0, :e].cpu().numpy()), eids[t])
        o = out[0, 0].double().cpu().numpy()
        rel = np.linalg.norm(o - z["outputs"][t]) / np.linalg.norm(z["outputs"][t])
        worst = max(worst, rel)
        assert rel <= OUT_TOL, (t, rel)
        assert abs(float(logden[0, 0]) - ref[8]) <= LOGDEN_TOL
        assert abs(float(cov[0, 0]) - ref[7]) <= 1e-5
    assert lay.units[0].m == int(z["metrics"][-1][9])


@pytest.mark.parametrize("Gh,d", [(4, 128), (7, 128), (2, 64), (8, 64)])
def test_batched_gqa_matches_per_head_oracle(Gh, d):
    """U=2 units x G heads (Llama G=4, Qwen G=7, ...), bf16 store,
    bf16-representable inputs: every (unit, head) must equal an independent
    oracle HeadEngine (both head-slot widths of the attention kernel)."""
    from oracle import oracle as O
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    rng = np.random.default_rng(11 + Gh)
    U, n, steps = 2, 3000, 6
    cen = rng.standard_normal((40, d)).astype(np.float32)
    keys = G.bf16_round(cen[rng.integers(40, size=(U, n))] + 0.3 * rng.standard_normal((U, n, d)).astype(np.float32))
    vals = G.bf16_round(rng.standard_normal((U, n, d)).astype(np.float32))
    qs = G.bf16_round(rng.standard_normal((steps, U, Gh, d)).astype(np.float32))
    nk = G.bf16_round(rng.standard_normal((steps, U, d)).astype(np.float32))
    nv = G.bf16_round(rng.standard_normal((steps, U, d)).astype(np.float32))
    cfg = EngineConfig()
    lay = WaveLayer(cfg, U, Gh, d, max_prefill=n, max_decode=64, with_elist=True)
    dev = torch.device("cuda")
    lay.prefill(torch.from_numpy(keys).to(dev), torch.from_numpy(vals).to(dev))
    orc = [[O.OracleEngine().prefill(keys[u], vals[u]) for _ in range(Gh)] for u in range(U)]
    for t in range(steps):
        out, logden, cov = lay.decode(torch.from_numpy(qs[t]).to(dev), torch.from_numpy(nk[t]).to(dev),
                                      torch.from_numpy(nv[t]).to(dev))
        lay.check_status()
        for u in range(U):
            for g in range(Gh):
                o_ref, sm = orc[u][g].decode_step(qs[t, u, g], nk[t, u], nv[t, u], with_recall=False)
                r_ref, e_ref = orc[u][g].last_plan()
                r = int(lay.nr[u])
                assert np.array_equal(lay.rlist[u, g, :r].cpu().numpy(), r_ref)
                assert np.array_equal(np.sort(lay.elist[u, g, :int(lay.ne[u])].cpu().numpy()), np.sort(e_ref))
                o = out[u, g].double().cpu().numpy()
                assert np.linalg.norm(o - o_ref) <= OUT_TOL * np.linalg.norm(o_ref)
                assert abs(float(logden[u, g]) - sm.log_denominator) <= LOGDEN_TOL


@pytest.mark.parametrize("splits", [3, 7])
def test_many_units_per_attention_cta(splits):
    """Few attention CTAs over many units (each CTA's chunk range crosses
    several unit boundaries, its consumers take chunks of neighbouring units
    round-robin): every (unit, head) partial record must stay distinct -- the
    default bench layer (128 units on 148 CTAs) hits the same case.  Every
    (unit, head) against an independent oracle HeadEngine."""
    from oracle import oracle as O
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    rng = np.random.default_rng(40 + splits)
    U, Gh, d, n, steps = 12, 4, 128, 1500, 3
    cen = rng.standard_normal((30, d)).astype(np.float32)
    keys = G.bf16_round(cen[rng.integers(30, size=(U, n))] + 0.3 * rng.standard_normal((U, n, d)).astype(np.float32))
    vals = G.bf16_round(rng.standard_normal((U, n, d)).astype(np.float32))
    qs = G.bf16_round(rng.standard_normal((steps, U, Gh, d)).astype(np.float32))
    nk = G.bf16_round(rng.standard_normal((steps, U, d)).astype(np.float32))
    nv = G.bf16_round(rng.standard_normal((steps, U, d)).astype(np.float32))
    lay = WaveLayer(EngineConfig(), U, Gh, d, max_prefill=n, max_decode=64, splits=splits)
    assert lay.S == splits
    dev = torch.device("cuda")
    lay.prefill(torch.from_numpy(keys).to(dev), torch.from_numpy(vals).to(dev))
    orc = [O.OracleEngine().prefill(keys[u], vals[u]) for u in range(U)]
    orc = [[orc[u]] + [orc[u].clone() for _ in range(Gh - 1)] for u in range(U)]
    for t in range(steps):
        out, logden, _ = lay.decode(torch.from_numpy(qs[t]).to(dev), torch.from_numpy(nk[t]).to(dev),
                                    torch.from_numpy(nv[t]).to(dev))
        lay.check_status()
        out = out.double().cpu().numpy()
        for u in range(U):
            for g in range(Gh):
                o_ref, sm = orc[u][g].decode_step(qs[t, u, g], nk[t, u], nv[t, u], with_recall=False)
                rel = np.linalg.norm(out[u, g] - o_ref) / np.linalg.norm(o_ref)
                assert rel <= OUT_TOL, (t, u, g, rel)
                assert abs(float(logden[u, g]) - sm.log_denominator) <= LOGDEN_TOL


def test_full_attention_matches_fp64():
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    rng = np.random.default_rng(5)
    U, Gh, d, n = 3, 2, 64, 700
    keys = G.bf16_round(rng.standard_normal((U, n, d)).astype(np.float32))
    vals = G.bf16_round(rng.standard_normal((U, n, d)).astype(np.float32))
    q = G.bf16_round(rng.standard_normal((U, Gh, d)).astype(np.float32))
    lay = WaveLayer(EngineConfig(), U, Gh, d, max_prefill=n)
    dev = torch.device("cuda")
    lay.prefill(torch.from_numpy(keys).to(dev), torch.from_numpy(vals).to(dev))
    out = lay.full_attention(torch.from_numpy(q).to(dev)).double().cpu().numpy()
    for u in range(U):
        for g in range(Gh):
            s = keys[u].astype(np.float64) @ q[u, g].astype(np.float64) / np.sqrt(d)
            w = np.exp(s - s.max())
            ref = (w @ vals[u].astype(np.float64)) / w.sum()
            assert np.linalg.norm(out[u, g] - ref) <= 1e-5 * np.linalg.norm(ref)


@pytest.mark.parametrize("split", [2, 4])
def test_split_pipeline_matches_single_launch(split):
    """split > 1 (per-group centroid scans, the groups' zone planning and
    attention on side streams overlapping the next group's scan) gives
    bit-identical zones; outputs agree to fp32 round-off (each group's
    attention partitions its chunks over the persistent warps differently, so
    the partial sums are added in a different order)."""
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    rng = np.random.default_rng(21)
    U, Gh, d, n, steps = 8, 4, 128, 3000, 5
    cen = rng.standard_normal((40, d)).astype(np.float32)
    keys = G.bf16_round(cen[rng.integers(40, size=(U, n))] + 0.3 * rng.standard_normal((U, n, d)).astype(np.float32))
    vals = G.bf16_round(rng.standard_normal((U, n, d)).astype(np.float32))
    dev = torch.device("cuda")
    lays = [WaveLayer(EngineConfig(), U, Gh, d, max_prefill=n, max_decode=64, split=sp) for sp in (1, split)]
    assert lays[1].split == split
    for lay in lays:
        lay.prefill(torch.from_numpy(keys).to(dev), torch.from_numpy(vals).to(dev))
    for t in range(steps):
        q = torch.from_numpy(G.bf16_round(rng.standard_normal((U, Gh, d)).astype(np.float32))).to(dev)
        k = torch.from_numpy(G.bf16_round(rng.standard_normal((U, d)).astype(np.float32))).to(dev)
        v = torch.from_numpy(G.bf16_round(rng.standard_normal((U, d)).astype(np.float32))).to(dev)
        outs = [lay.decode(q, k, v)[0].clone() for lay in lays]
        torch.cuda.synchronize()
        for lay in lays:
            lay.check_status()
        assert torch.equal(lays[0].rlist, lays[1].rlist)
        assert torch.equal(lays[0].cnt, lays[1].cnt)
        rel = float((outs[0] - outs[1]).norm() / outs[0].norm())
        assert rel <= 1e-6, (t, rel)


def test_launch_step_out_argument():
    """launch_step(out=...) writes the attention output to the caller's tensor,
    bit-identical to the layer's own output buffer (the pipelined e2e path)."""
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    from paper_2505_02922_b200.errors import ConfigError
    rng = np.random.default_rng(5)
    U, Gh, d, n = 4, 4, 128, 2500
    keys = G.bf16_round(rng.standard_normal((U, n, d)).astype(np.float32))
    vals = G.bf16_round(rng.standard_normal((U, n, d)).astype(np.float32))
    dev = torch.device("cuda")
    lays = [WaveLayer(EngineConfig(), U, Gh, d, max_prefill=n, max_decode=16) for _ in range(2)]
    for lay in lays:
        lay.prefill(torch.from_numpy(keys).to(dev), torch.from_numpy(vals).to(dev))
    mine = torch.full((U, Gh, d), float("nan"), device=dev)
    for t in range(3):
        q = torch.from_numpy(G.bf16_round(rng.standard_normal((U, Gh, d)).astype(np.float32))).to(dev)
        k = torch.from_numpy(G.bf16_round(rng.standard_normal((U, d)).astype(np.float32))).to(dev)
        v = torch.from_numpy(G.bf16_round(rng.standard_normal((U, d)).astype(np.float32))).to(dev)
        lays[0].launch_step(q, k, v)
        lays[1].launch_step(q, k, v, out=mine)
        torch.cuda.synchronize()
        assert torch.equal(lays[0].out, mine), t
    with pytest.raises(ConfigError):
        lays[1].launch_step(q, k, v, out=mine[:2])
