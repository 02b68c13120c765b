"""The slow tier: cluster-private fixed-size blocks of raw K/V in host memory
(tierkv store.py:16-105).

On the B200 path the slow tier is (pinned) host memory and the engine packs it
cluster-contiguously straight from the build kernel (``WaveLayer(offload=True)``).
This module is the function-level form the reference's API exposes: a host
store with the reference's block numbering, whole-block read accounting and
error conventions.  Rows are kept in one growing host array per tensor in
pack order; a block is a contiguous row range of one cluster.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, IntegrityError

SCALAR_BYTES = 4  # the reference accounts K and V as float32 (store.py:16)


@dataclass
class TokenKV:
    """One token's key, value and context position (store.py:19-25)."""
    key: np.ndarray
    value: np.ndarray
    token_id: int


@dataclass
class Block:
    """A block's payload view (store.py:28-35)."""
    block_id: int
    payload: list
    occupied: int = field(init=False)

    def __post_init__(self):
        self.occupied = len(self.payload)


def block_capacity(block_size_bytes: int, d: int) -> int:
    """Tokens per block, K + V at 4 bytes a scalar (store.py:38-45)."""
    per_token = 2 * d * SCALAR_BYTES
    if block_size_bytes < per_token:
        raise ConfigError(f"block_size_bytes={block_size_bytes} cannot hold a single token at d={d}")
    return block_size_bytes // per_token


class _BlockTable(dict):
    """block id -> Block, materialised from the row arrays on access."""

    def __init__(self, store):
        super().__init__()
        self._s = store

    def __missing__(self, bid):
        raise KeyError(bid)

    def __getitem__(self, bid):
        return Block(bid, self._s._payload(bid))

    def get(self, bid, default=None):
        return self[bid] if bid in self else default

    def __contains__(self, bid):
        return isinstance(bid, (int, np.integer)) and 0 <= int(bid) < len(self._s._blk_row)

    def __len__(self):
        return len(self._s._blk_row)

    def __iter__(self):
        return iter(range(len(self._s._blk_row)))

    def values(self):
        return [self[b] for b in self]

    def items(self):
        return [(b, self[b]) for b in self]


class SlowTierStore:
    """Per-head slow tier (store.py:48-105): ``pack_cluster`` appends an
    ordered member list as ceil(len / capacity) fresh blocks; ``read_blocks``
    returns payloads in request order and charges whole blocks."""

    def __init__(self, d: int, block_size_bytes: int = 2048, head: int = 0):
        if d <= 0:
            raise ConfigError(f"dimension must be positive, got {d}")
        self.d = d
        self.block_size_bytes = block_size_bytes
        self.block_capacity = block_capacity(block_size_bytes, d)
        self.head = head
        self.bytes_read_total = 0
        self.bytes_written_total = 0
        self._k = np.empty((0, d), np.float32)
        self._v = np.empty((0, d), np.float32)
        self._tok = np.empty(0, np.int64)
        self._rows = 0
        self._blk_row: list[int] = []   # first row of each block
        self._blk_n: list[int] = []     # rows in each block
        self._packed: set[int] = set()
        self.blocks = _BlockTable(self)

    def _reserve(self, n):
        if self._rows + n <= len(self._tok):
            return
        cap = max(self._rows + n, 2 * len(self._tok), 256)
        for name, shape, dt in (("_k", (cap, self.d), np.float32), ("_v", (cap, self.d), np.float32),
                                ("_tok", (cap,), np.int64)):
            new = np.empty(shape, dt)
            new[: self._rows] = getattr(self, name)[: self._rows]
            setattr(self, name, new)

    def pack_cluster(self, members: list[TokenKV]) -> list[int]:
        if not members:
            raise IntegrityError("pack_cluster called with empty member list")
        for t in members:
            if len(t.key) != self.d or len(t.value) != self.d:
                raise ConfigError(f"token {t.token_id} has dimension {len(t.key)}/{len(t.value)}, "
                                  f"store expects {self.d}")
        ids = [int(t.token_id) for t in members]
        dup = next((i for i in ids if i in self._packed), None)
        if dup is not None or len(set(ids)) != len(ids):
            raise IntegrityError(f"token {dup if dup is not None else ids[0]} already packed in this store")
        n = len(members)
        self._reserve(n)
        r0 = self._rows
        self._k[r0:r0 + n] = np.stack([np.asarray(t.key, np.float32) for t in members])
        self._v[r0:r0 + n] = np.stack([np.asarray(t.value, np.float32) for t in members])
        self._tok[r0:r0 + n] = ids
        self._rows += n
        cap = self.block_capacity
        first = len(self._blk_row)
        for s in range(0, n, cap):
            self._blk_row.append(r0 + s)
            self._blk_n.append(min(cap, n - s))
        self.bytes_written_total += (len(self._blk_row) - first) * self.block_size_bytes
        self._packed.update(ids)
        return list(range(first, len(self._blk_row)))

    def _payload(self, bid):
        r0, n = self._blk_row[bid], self._blk_n[bid]
        return [TokenKV(self._k[r], self._v[r], int(self._tok[r])) for r in range(r0, r0 + n)]

    def block_rows(self, bid):
        """(keys, values, token ids) arrays of one block (views)."""
        r0, n = self._blk_row[bid], self._blk_n[bid]
        return self._k[r0:r0 + n], self._v[r0:r0 + n], self._tok[r0:r0 + n]

    def read_blocks(self, block_ids: list[int]) -> list[tuple[int, list[TokenKV]]]:
        out = []
        for bid in block_ids:
            if bid not in self.blocks:
                raise IntegrityError(f"unknown block_id {bid}")
            out.append((bid, self._payload(bid)))
        self.bytes_read_total += len(block_ids) * self.block_size_bytes
        return out

    @property
    def n_blocks(self) -> int:
        return len(self._blk_row)
