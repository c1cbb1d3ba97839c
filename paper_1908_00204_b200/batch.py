"""Batch refactorization across GPUs (BASELINE cfg5).

A single matrix never shards (its level barriers need on-die latency); a
batch of independent same-pattern value sets does: every rank (one process
per GPU) holds a read-only replica of the pattern and plan, factors a
contiguous shard of the value sets with no communication, and the only
collective is the final gather of per-set results (status + checksum; the
LU values stay where they were computed unless the caller gathers them).
"""

from __future__ import annotations

import hashlib

import numpy as np


def shard(batch: int, rank: int, world: int) -> range:
    """Contiguous shard of [0, batch) for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def set_digest(lu_values: np.ndarray) -> int:
    """63-bit checksum of one set's LU values (bitwise identity across ranks)."""
    return int.from_bytes(hashlib.sha256(np.ascontiguousarray(lu_values).tobytes()).digest()[:8],
                          "little") >> 1


def gather_results(indices, status, digests, group=None):
    """All-gather (index, status, digest) triples of every rank's shard with
    torch.distributed (NCCL on the GPUs, gloo on the host); returns the
    per-set arrays for the whole batch, ordered by set index."""
    import torch
    import torch.distributed as dist

    local = np.stack([np.asarray(indices, np.int64), np.asarray(status, np.int64),
                      np.asarray(digests, np.int64)], axis=1) if len(indices) else np.zeros((0, 3), np.int64)
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    n = torch.tensor([len(local)], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    cap = int(max(int(x) for x in sizes))
    buf = torch.zeros((cap, 3), dtype=torch.int64, device=dev)
    if len(local):
        buf[:len(local)] = torch.from_numpy(local).to(dev)
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    rows = np.concatenate([p[:int(k)].cpu().numpy() for p, k in zip(parts, sizes)])
    rows = rows[np.argsort(rows[:, 0], kind="stable")]
    return rows[:, 0], rows[:, 1], rows[:, 2]
