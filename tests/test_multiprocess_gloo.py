"""CPU, world_size 2 over gloo: the sharded HEGMM path's host logic.

Each rank encrypts and multiplies its shard of instances with the reference
algorithms over the CPU BFV oracle (the stand-in for its GPU), using the same
encryption counters a single-GPU run would use; rank 0 gathers the result
ciphertexts in the layout the library's NCCL gather uses
(paper_2405_02238_b200.dist.gather_layout: rank order, variable-size shards;
gloo stands in for hgm_comm_gather_batch here), decrypts them, and checks every
product and that the gathered words equal a single-process run of the same
instances."""
import os
import socket

import numpy as np
import pytest

from paper_2405_02238_b200.dist import counter_base, gather_layout, id_file_path, shard

TOTAL, M, L, N = 5, 3, 4, 2


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def gather_ciphertexts(dist, local, count, words, total, world, rank):
    """gloo stand-in for hgm_comm_gather_batch: pads every shard to the largest
    and trims on the root to gather_layout's counts."""
    import torch

    layout = gather_layout(world, total)
    maxc = max(c for _, c in layout)
    send = torch.zeros(maxc * words, dtype=torch.int64)
    if count:
        send[: count * words] = local[: count * words]
    outs = [torch.empty_like(send) for _ in range(world)] if rank == 0 else None
    dist.gather(send, outs, dst=0)
    if rank != 0:
        return None
    return [outs[r][: layout[r][1] * words] for r in range(world)]


def worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle.bindings import Oracle, RefLib
    from paper_2405_02238_b200.workload import batch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, B = batch(99, 0, TOTAL, M, L, N, -8, 7)
        first, count = shard(rank, world, TOTAL)
        o = Oracle(2, 1)
        local = []
        for i in range(first, first + count):
            _, _, ct, _ = RefLib.mm_oracle(A[i], B[i], param_id=2, seed=1,
                                           counter0=counter_base(i, 3), algo="basic", words=o.words)
            local.append(ct.view(np.int64))
        t = torch.from_numpy(np.concatenate(local)) if local else torch.zeros(0, dtype=torch.int64)
        got = gather_ciphertexts(dist, t, count, o.words, TOTAL, world, rank)
        if rank == 0:
            words = np.concatenate([g.numpy() for g in got]).view(np.uint64).reshape(TOTAL, o.words)
            seg = max(M * L, L * N, M * N)
            ok = []
            for i in range(TOTAL):
                slots = o.decrypt(words[i], seg)
                C = np.array([[slots[r + c * M] for c in range(N)] for r in range(M)])  # column-major
                ok.append(bool(np.array_equal(C, (A[i] @ B[i]) % 65537)))
                _, _, ct1, _ = RefLib.mm_oracle(A[i], B[i], param_id=2, seed=1, counter0=counter_base(i, 3),
                                                algo="basic", words=o.words)
                ok.append(bool(np.array_equal(ct1, words[i])))
            q.put(ok)
    finally:
        dist.destroy_process_group()


def test_sharding_is_a_partition():
    for world in (1, 2, 3, 8):
        spans = [shard(r, world, 4096) for r in range(world)]
        assert spans[0][0] == 0 and sum(c for _, c in spans) == 4096
        for (f0, c0), (f1, _) in zip(spans, spans[1:]):
            assert f0 + c0 == f1


def test_gather_layout_and_id_path(monkeypatch):
    assert gather_layout(3, 8) == [(0, 2), (2, 3), (5, 3)]
    monkeypatch.setenv("MASTER_PORT", "29511")
    monkeypatch.delenv("HGM_COMM_ID_FILE", raising=False)
    p = id_file_path()
    assert p.startswith("/tmp/hgm_comm_29511_") and p.endswith(f"_{os.getppid()}.id")
    monkeypatch.setenv("HGM_COMM_ID_FILE", "/tmp/x.id")
    assert id_file_path() == "/tmp/x.id"


def test_gloo_world2_gather_and_decrypt(ref):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ok = q.get(timeout=10)
    assert len(ok) == 2 * TOTAL and all(ok)
