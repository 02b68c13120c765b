"""Multi-rank host logic of the sharded path on CPU with the
gloo backend, world_size 2: unit partitioning and the final output gather."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_02922_b200.errors import ConfigError
from paper_2505_02922_b200.parallel import gather_outputs, shard_units


def test_shard_units_cover_and_balance():
    for B, H, W in [(16, 8, 1), (16, 8, 2), (16, 8, 8), (16, 4, 8), (3, 5, 4), (4, 8, 3)]:
        shards = [shard_units(B, H, W, r) for r in range(W)]
        got = [u for s in shards for u in s.units()]
        assert got == list(range(B * H))
        sizes = [s.count for s in shards]
        assert max(sizes) - min(sizes) <= 1


def test_shard_units_rejects_bad_args():
    with pytest.raises(ConfigError):
        shard_units(1, 2, 4, 0)
    with pytest.raises(ConfigError):
        shard_units(4, 8, 2, 2)


def _worker(rank, world, port, B, H, G, d, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = shard_units(B, H, world, rank)
        # rank-local outputs: deterministic function of the global unit id
        out = torch.stack([torch.full((G, d), float(u)) + torch.arange(G)[:, None] * 0.5
                           for u in sh.units()])
        full = gather_outputs(out, sh, B, H)
        ref = torch.stack([torch.full((G, d), float(u)) + torch.arange(G)[:, None] * 0.5
                           for u in range(B * H)]).view(B, H * G, d)
        q.put((rank, bool(torch.equal(full, ref))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B,H,G", [(4, 8, 4), (3, 4, 7)])
def test_gather_outputs_world2_gloo(B, H, G):
    world, d = 2, 16
    port = 29500 + (os.getpid() % 1000) + B
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, H, G, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
