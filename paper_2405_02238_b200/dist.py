"""Multi-GPU plumbing: instances are sharded across ranks with
no data-path collective; the only exchange is gathering each rank's result
ciphertexts to rank 0 (one process per GPU, torch.distributed over NCCL on the
B200 box, gloo in the CPU tests).  NCCL never reduces ciphertexts: its sums
wrap mod 2^64, not mod q, so results are moved, never added, in transit."""
from __future__ import annotations

from typing import List, Optional, Tuple


def shard(rank: int, world: int, total: int) -> Tuple[int, int]:
    """Contiguous instance range [first, first + count) of `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    lo = rank * total // world
    hi = (rank + 1) * total // world
    return lo, hi - lo


def counter_base(first_instance: int, encryptions_per_instance: int) -> int:
    """Encryption counter of an instance's first ciphertext: identical to the
    single-GPU run, so every rank's ciphertexts are bit-identical to it."""
    return first_instance * encryptions_per_instance


def gather_ciphertexts(dist, local, count: int, words: int, total: int, world: int, rank: int,
                       device=None) -> Optional[List]:
    """Gathers `count` ciphertexts of `words` uint64 words (as an int64 tensor
    `local` of count*words elements) from every rank to rank 0.  Returns, on
    rank 0, the list of per-rank tensors trimmed to their true counts (instance
    order = rank order); None elsewhere.  Shards may differ by one instance, so
    each rank sends a buffer padded to the largest shard."""
    import torch

    maxc = max(shard(r, world, total)[1] for r in range(world))
    send = torch.zeros(maxc * words, dtype=torch.int64, device=device)
    if count:
        send[: count * words] = local[: count * words]
    outs = [torch.empty_like(send) for _ in range(world)] if rank == 0 else None
    dist.gather(send, outs, dst=0)
    if rank != 0:
        return None
    return [outs[r][: shard(r, world, total)[1] * words] for r in range(world)]
