"""The library's NCCL communicator (hgm_comm_*) on one B200: a world-1
communicator exercises the whole C-ABI path -- id publication through a file,
ncclCommInitRank, barrier, max over ranks, the variable-size gather of a
batch's result ciphertexts to the root and hgm_decrypt_products on the
gathered words.  Rank > 1 needs one GPU per rank (NCCL refuses two ranks on one
device); the multi-rank host logic is covered by tests/test_multiprocess_gloo.py."""
import os

import numpy as np
import pytest

from paper_2405_02238_b200.workload import batch

pytestmark = pytest.mark.gpu


def test_world1_comm_gather_decrypt(gpu_factory, tmp_path):
    import paper_2405_02238_b200 as hb

    ctx = gpu_factory(0)
    comm = hb.Comm(ctx, 0, 1, id_file=str(tmp_path / "nccl.id"))
    try:
        assert not os.path.exists(tmp_path / "nccl.id")  # rank 0 removes the id once every rank joined
        comm.barrier()
        assert comm.max(3.25) == 3.25
        A, B = batch(7, 0, 5, 8, 16, 4, -8, 7)
        bt = hb.Batch(ctx, A, B, algo=1, counter0=0)
        bt.cloud()
        ptr, n = comm.gather_batch(bt, root=0)
        assert n == 5 and ptr
        try:
            C = ctx.decrypt_products(ptr, n, 8, 16, 4, algo=1)
        finally:
            comm.free_buffer(ptr)
        assert np.array_equal(C, np.einsum("kij,kjl->kil", A, B) % 65537)
        assert np.array_equal(C, bt.decrypt())
        bt.free()
        # a rank without instances contributes nothing
        ptr, n = comm.gather_batch(None, root=0)
        assert (ptr, n) == (None, 0)
    finally:
        comm.close()


def test_world1_comm_from_unique_id(gpu_factory):
    import paper_2405_02238_b200 as hb

    ctx = gpu_factory(0)
    comm = hb.Comm(ctx, 0, 1, unique_id=hb.Comm.unique_id())
    try:
        comm.barrier()
        assert comm.max(-1.5) == -1.5
    finally:
        comm.close()


def test_comm_rejects_bad_rank(gpu_factory):
    import paper_2405_02238_b200 as hb

    with pytest.raises(hb.HEError):
        hb.Comm(gpu_factory(0), 2, 2, unique_id=hb.Comm.unique_id())


def test_sharded_matmul_world1_comm(gpu_factory, tmp_path):
    """Config-5-style row blocks through the communicator path of
    dist.sharded_matmul (the path every rank runs at N > 1)."""
    import paper_2405_02238_b200 as hb
    from paper_2405_02238_b200.dist import sharded_matmul

    ctx = gpu_factory(0)
    A, B = batch(11, 0, 1, 32, 16, 8, -8, 7)
    comm = hb.Comm(ctx, 0, 1, id_file=str(tmp_path / "id"))
    try:
        C = sharded_matmul(ctx, A[0], B[0], 4, algo=1, comm=comm)
    finally:
        comm.close()
    assert np.array_equal(C, (A[0] @ B[0]) % 65537)
