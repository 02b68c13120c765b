"""Sharding of the wave-index decode path across GPUs.

(request, kv-head) units are independent state machines (
each owns its index, zones, block cache and host KV), so the path shards with
NO data-path collective: a rank serves a contiguous block of units and keeps
all G query heads of a kv-head together (GQA reuse of centroids and cache).
The only collective is the final gather of the attention outputs
[B, H_q, d] (NCCL all-gather over NVLink on GPUs, gloo on CPU in tests).

Two partitionings:
  * ``shard_units``  -- strong scaling: a fixed set of B x H_kv units split in
    contiguous chunks over the world (balanced to +-1 unit);
  * weak scaling (bench.py): every rank serves its own ``batch`` requests.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import ConfigError


@dataclass(frozen=True)
class UnitShard:
    rank: int
    world: int
    start: int   # first global unit (request * H_kv + kv_head)
    count: int   # units on this rank

    def units(self):
        return range(self.start, self.start + self.count)


def shard_units(batch: int, h_kv: int, world: int, rank: int) -> UnitShard:
    """Contiguous, balanced split of the B * H_kv units; rank r gets
    [floor(r N / W), floor((r + 1) N / W))."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} of world {world}")
    n = batch * h_kv
    if n < world:
        raise ConfigError(f"{n} units cannot be spread over {world} ranks")
    a, b = n * rank // world, n * (rank + 1) // world
    return UnitShard(rank, world, a, b - a)


def gather_outputs(out: torch.Tensor, shard: UnitShard, batch: int, h_kv: int, group=None) -> torch.Tensor:
    """All-gather per-rank attention outputs [count, G, d] into the full
    [batch, h_kv * G, d] tensor (the one collective of the path)."""
    import torch.distributed as dist
    if out.dim() != 3 or out.shape[0] != shard.count:
        raise ConfigError(f"expected [{shard.count}, G, d] outputs, got {tuple(out.shape)}")
    G, d = out.shape[1], out.shape[2]
    n = batch * h_kv
    counts = [n * (r + 1) // shard.world - n * r // shard.world for r in range(shard.world)]
    width = max(counts)
    pad = out.new_zeros((width, G, d))
    pad[: shard.count] = out
    bufs = [out.new_empty((width, G, d)) for _ in range(shard.world)]
    dist.all_gather(bufs, pad.contiguous(), group=group)
    full = torch.cat([bufs[r][: counts[r]] for r in range(shard.world)], dim=0)
    return full.view(batch, h_kv * G, d)
