"""The sharded path end to end with real WaveLayer shards:
two ranks (two processes on cuda:0, gloo for the gather -- the box has one
GPU) each build and decode their contiguous block of (request, kv-head)
units; the gathered outputs must equal one single-rank layer over all units
(ordered retrieval ids bit-exact, outputs to fp32 round-off).  The strong-
scaling split is shard_units; the one collective is gather_outputs."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

B, H, G, D, N, STEPS = 3, 4, 4, 128, 3000, 4


def _inputs():
    rng = np.random.default_rng(81)
    U = B * H
    cen = rng.standard_normal((U, 24, D)).astype(np.float32)
    keys = cen[np.arange(U)[:, None], rng.integers(24, size=(U, N))] + 0.4 * rng.standard_normal((U, N, D))
    vals = rng.standard_normal((U, N, D))
    q = cen[np.arange(U)[None, :], rng.integers(24, size=(STEPS, U))][:, :, None] + \
        0.3 * rng.standard_normal((STEPS, U, G, D))
    nk = rng.standard_normal((STEPS, U, D))
    nv = rng.standard_normal((STEPS, U, D))
    f = lambda x: np.ascontiguousarray(x, np.float32)
    return f(keys), f(vals), f(q), f(nk), f(nv)


def _run_units(units, keys, vals, q, nk, nv):
    from paper_2505_02922_b200 import EngineConfig, WaveLayer
    dev = torch.device("cuda", 0)
    sl = slice(units.start, units.stop)
    lay = WaveLayer(EngineConfig(), len(units), G, D, max_prefill=N, max_decode=16)
    lay.prefill(torch.from_numpy(keys[sl]).to(dev), torch.from_numpy(vals[sl]).to(dev))
    outs, rls = [], []
    for t in range(STEPS):
        out, _, _ = lay.decode(torch.from_numpy(q[t, sl]).to(dev), torch.from_numpy(nk[t, sl]).to(dev),
                               torch.from_numpy(nv[t, sl]).to(dev))
        lay.check_status()
        outs.append(out.clone())
        rls.append(lay.rlist[:, :, :int(lay.nr[0])].cpu())
    return outs, rls


def _worker(rank, world, port, q_out):
    import torch.distributed as dist
    from paper_2505_02922_b200.parallel import gather_outputs, shard_units
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys, vals, q, nk, nv = _inputs()
        sh = shard_units(B, H, world, rank)
        outs, rls = _run_units(sh.units(), keys, vals, q, nk, nv)
        full = [gather_outputs(o.cpu(), sh, B, H) for o in outs]
        q_out.put((rank, sh.start, sh.count, [f.numpy() for f in full], [r.numpy() for r in rls]))
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_equal_single_rank():
    world = 2
    port = 29700 + os.getpid() % 500
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, qo)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, start, count, full, rls = qo.get(timeout=300)
        res[rank] = (start, count, full, rls)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    keys, vals, q, nk, nv = _inputs()
    ref_out, ref_rl = _run_units(range(B * H), keys, vals, q, nk, nv)
    assert [res[r][1] for r in range(world)] == [6, 6]
    for t in range(STEPS):
        ref = ref_out[t].cpu().numpy().reshape(B, H * G, D)
        for r in range(world):
            got = res[r][2][t]  # every rank holds the gathered [B, H*G, D]
            assert np.allclose(got, ref, rtol=2e-6, atol=2e-6), (t, r, np.abs(got - ref).max())
            s, c = res[r][0], res[r][1]
            rl = res[r][3][t]
            assert np.array_equal(rl, ref_rl[t][s:s + c].numpy()), (t, r)
