"""Multi-GPU plumbing, torch-free: one process per GPU, the
library's own NCCL communicator (``hgm_comm_*``, ``paper_2405_02238_b200.Comm``).

Work shards by independent products (config 4: instance ranges) or output row
blocks (config 5); keys are replicated per GPU, so a rank's shard needs no
data-path collective.  The only exchange is the gather of each rank's result
ciphertexts to rank 0, which decrypts (NCCL never reduces ciphertexts: its sums
wrap mod 2^64, not mod q).  Reference analogue: the std::async pool over
independent cases, /root/reference/proj/src/costmodel.cpp:273-296."""
from __future__ import annotations

import os
from typing import Dict, List, Optional, Tuple


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


def gather_layout(world: int, total: int) -> List[Tuple[int, int]]:
    """(first, count) of every rank's shard: the order and sizes in which
    Comm.gather_batch lays the gathered ciphertexts out on the root."""
    return [shard(r, world, total) for r in range(world)]


def env_rank() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun / launcher environment."""
    g = os.environ.get
    return int(g("RANK", 0)), int(g("WORLD_SIZE", 1)), int(g("LOCAL_RANK", 0))


def id_file_path() -> str:
    """Where rank 0 publishes the NCCL id for this launch: unique per launcher
    process (all ranks of one torchrun share its pid) and master port."""
    explicit = os.environ.get("HGM_COMM_ID_FILE")
    if explicit:
        return explicit
    port = os.environ.get("MASTER_PORT", "0")
    run = os.environ.get("TORCHELASTIC_RUN_ID", "none")
    return f"/tmp/hgm_comm_{port}_{run}_{os.getppid()}.id"


def comm_from_env(ctx) -> Optional["object"]:
    """The session's communicator for a multi-rank launch (None at world 1)."""
    import paper_2405_02238_b200 as hb

    rank, world, _ = env_rank()
    if world <= 1:
        return None
    # NCCL's own init lines (ranks, transports) for the launcher's logs, on stderr so
    # that rank 0's stdout stays one JSON line; NCCL is bound lazily, after this
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    return hb.Comm(ctx, rank, world, id_file=id_file_path())


def row_blocks(m: int, parts: int) -> List[Tuple[int, int]]:
    """Row-block decomposition of an m-row product into `parts` contiguous
    blocks (config 5: 128 rows -> 8 blocks of 16).  Every block
    A_r (rows x l) . B is an independent product; C is their row concatenation."""
    return [shard(r, parts, m) for r in range(parts)]


def sharded_matmul(ctx, A, B, parts: int, algo: int = 1, comm=None, counter0: int = 0,
                   timings: Optional[Dict[str, float]] = None):
    """Config-5 decomposition: the `parts` row blocks of A.B, rank r running its
    share as one lockstep batch on its GPU (block b encrypts from counter
    counter0 + 2 b, as a single GPU would), the result ciphertexts gathered to
    rank 0 over the library's NCCL communicator and decrypted there.
    Returns C (m x n, mod t) on rank 0 and None elsewhere.  Row blocks must be
    of equal height (one compiled program)."""
    import numpy as np

    import paper_2405_02238_b200 as hb

    rank, world = (comm.rank, comm.world) if comm is not None else (0, 1)
    blocks = row_blocks(A.shape[0], parts)
    heights = {h for _, h in blocks}
    if len(heights) != 1:
        raise ValueError("row blocks of unequal height: use parts dividing m")
    h = heights.pop()
    first, count = shard(rank, world, parts)
    E = hb.program_info(algo, h, A.shape[1], B.shape[1], ctx.slot_count, ctx.N)[1]["encryptions"]
    bt = None
    if count:
        As = np.stack([A[blocks[b][0]: blocks[b][0] + h] for b in range(first, first + count)])
        Bs = np.stack([B] * count)
        bt = hb.Batch(ctx, As, Bs, algo=algo, counter0=counter0 + first * E)
        ms = bt.cloud()
        if timings is not None:
            timings["cloud_ms"] = ms
    try:
        if comm is None:
            return np.concatenate(list(bt.decrypt()))
        ptr, n = comm.gather_batch(bt, root=0)
        if rank != 0:
            return None
        try:
            C = ctx.decrypt_products(ptr, n, h, A.shape[1], B.shape[1], algo=algo)
        finally:
            comm.free_buffer(ptr)
        return np.concatenate(list(C))
    finally:
        if bt is not None:
            bt.free()


def blocked_mm_sharded(ctx, A, B, rows, mids, cols, algo: int = 1, comm=None, counter0: int = 0):
    """blocked_mm (algorithms.cpp:434-498) with encrypted accumulation, output
    blocks sharded over the ranks: rank r sums its output
    blocks' products over the mid dimension as ciphertexts on its GPU
    (hgm_blocked_mm_ex, no decryption), the sums travel to rank 0 over the
    library's NCCL communicator, and rank 0 decrypts each sum once.  Counters
    are those of a single-GPU run, so every sum is bit-identical to it.
    Returns (C mod t, number of decrypts) on rank 0 and (None, 0) elsewhere."""
    import numpy as np

    rank, world = (comm.rank, comm.world) if comm is not None else (0, 1)
    n_out = len(rows) * len(cols)
    first, count = shard(rank, world, n_out)
    _, _, _, words, meta = ctx.blocked_mm_acc(A, B, rows, mids, cols, algo=algo, counter0=counter0,
                                              out_range=(first, count), export="only")
    if comm is not None:
        cap_entries = n_out * len(mids)
        all_words = comm.gather_words(words, cap_entries * ctx.ct_words)
        all_meta = comm.gather_words(meta.view(np.uint64), cap_entries * 8)
        if rank != 0:
            return None, 0
        words = all_words.reshape(-1, ctx.ct_words)
        meta = all_meta.view(np.int64).reshape(-1, 8)
    m, n = A.shape[0], B.shape[1]
    ro = np.concatenate([[0], np.cumsum(rows)])
    co = np.concatenate([[0], np.cumsum(cols)])
    C = np.zeros((m, n), dtype=np.int64)
    for k in range(meta.shape[0]):
        ob, used, bm, bl, bn, order = (int(x) for x in meta[k][:6])
        blk = ctx.decrypt_products(words[k].ctypes.data, 1, bm, bl, bn, algo=used, order=order)[0]
        bi, bj = divmod(ob, len(cols))
        C[ro[bi]:ro[bi] + bm, co[bj]:co[bj] + bn] = (C[ro[bi]:ro[bi] + bm, co[bj]:co[bj] + bn] + blk) % 65537
    return C, int(meta.shape[0])
