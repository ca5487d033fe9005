"""Multi-GPU batch sharding for inference.

``M:forward`` is read-only on the store (M:321-397), so a batch shards into
contiguous per-rank slices with replicated tables and **no data-path
collective**: each rank scores its slice and owns that slice of the output.
Tables are replicated by seeded on-device generation (zero communication) or,
for a trained store, by one broadcast of each block at load time.  Training is
not sharded: every example updates the bias and the whole MLP in a strict
order (M:465-481, M:525-530, T:175-185), so it runs on one GPU.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int
    stop: int

    @property
    def size(self) -> int:
        return self.stop - self.start


def shard_range(n: int, world: int, rank: int) -> Shard:
    """Contiguous, balanced (sizes differ by at most 1), ordered, disjoint."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    base, rem = divmod(int(n), int(world))
    start = rank * base + min(rank, rem)
    stop = start + base + (1 if rank < rem else 0)
    return Shard(rank, world, start, stop)


def table_digest(*arrays) -> str:
    """Digest of replicated table contents (checks replication without moving data)."""
    h = hashlib.blake2b(digest_size=16)
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def broadcast_store(store, src: int = 0, group=None):
    """Replicate a trained store's blocks from ``src`` (one broadcast per block
    over NVLink/NVSwitch with NCCL; load-time only, never on the scoring path).

    Every block travels as its raw bytes (a uint8 view: NCCL and gloo have no
    uint16, and a byte copy keeps every bit), and the per-table (min, bucket)
    headers of u16 (quantised) tables, which live on the host, are broadcast
    alongside, so every replica dequantises identically."""
    import torch
    import torch.distributed as dist
    for _, t in store.blocks(include_optimizer=store.has_optimizer):
        dist.broadcast(t.reshape(-1).view(torch.uint8), src=src, group=group)
    if store.wdtype == "u16":
        hdr = [store.q_headers]
        dist.broadcast_object_list(hdr, src=src, group=group)
        store.q_headers = dict(hdr[0])
    store.mark_mutated()  # replicas' states are invalidated like any other write
    return store


def predict_shard(idx, val, store, shard: Shard, out=None):
    """Score this rank's slice of a batch with K1 (no collective)."""
    from .model import predict_batch
    return predict_batch(idx[shard.start:shard.stop], val[shard.start:shard.stop], store,
                         out=out)
