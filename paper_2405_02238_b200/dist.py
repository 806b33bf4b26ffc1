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


def row_blocks(m: int, parts: int) -> List[Tuple[int, int]]:
    """Row-block decomposition of an m-row product into `parts` contiguous
    blocks (config 5: 128 rows -> 8 blocks of 16).  Every block
    A_r (rows x l) . B is an independent product; C is their row concatenation."""
    return [shard(r, parts, m) for r in range(parts)]


def sharded_matmul(ctx, A, B, parts: int, algo: int = 1, rank: int = 0, world: int = 1, counter0: int = 0):
    """Runs this rank's share of the row blocks of A.B as one lockstep batch on
    its GPU (blocks of equal height share one compiled program).  Returns
    {block index: C block} for the blocks this rank owns."""
    import numpy as np

    blocks = row_blocks(A.shape[0], parts)
    first, count = shard(rank, world, parts)
    mine = list(range(first, first + count))
    out = {}
    by_height = {}
    for bi in mine:
        by_height.setdefault(blocks[bi][1], []).append(bi)
    for height, ids in by_height.items():
        As = np.stack([A[blocks[bi][0]: blocks[bi][0] + height] for bi in ids])
        Bs = np.stack([B for _ in ids])
        C, _ = ctx.matmul_batch(As, Bs, algo=algo, counter0=counter0 + ids[0] * 2)
        for k, bi in enumerate(ids):
            out[bi] = C[k]
    return out
