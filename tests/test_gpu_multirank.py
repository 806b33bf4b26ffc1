"""Multi-rank runs of the real entry points on one B200.

NCCL refuses two ranks on one device, so the library is pointed at a TCP
stand-in for libnccl.so.2 (tests/shim/nccl_tcp_shim.cpp, via HGM_NCCL_LIB) and
every rank uses device 0 (HGM_DEVICE).  The ranks' kernels never wait on one
another -- the only exchanges are the host-synchronised gather, barrier and max
-- so this exercises exactly the code bench.py --gpus N runs under torchrun:
the id file, the communicator, per-rank shards and counters, the gather of
result ciphertexts to rank 0 and rank 0's decryption of all of them."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "shim", "libnccl_tcp_shim.so")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(world, argv, tmp_path, timeout=600, id_file=True):
    if not os.path.exists(SHIM):
        pytest.skip("tests/shim/libnccl_tcp_shim.so not built")
    port = free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), HGM_NCCL_LIB=SHIM, HGM_DEVICE="0")
        if id_file:
            env["HGM_COMM_ID_FILE"] = str(tmp_path / f"id_{port}")
        else:  # the launcher default: /tmp/hgm_comm_<port>_<run>_<parent pid>.id (dist.id_file_path)
            env.pop("HGM_COMM_ID_FILE", None)
        procs.append(subprocess.Popen([sys.executable] + argv, cwd=ROOT, env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=timeout) for p in procs]
    bad = [r for r, p in enumerate(procs) if p.returncode != 0]
    assert not bad, "\n".join(f"rank {r} rc {procs[r].returncode}:\n{outs[r][0][-1500:]}\n{outs[r][1][-3000:]}"
                               for r in range(world))
    return outs


def test_bench_cfg4_two_ranks(tmp_path):
    outs = launch(2, ["bench.py", "--gpus", "2", "--instances", "48", "--steps", "1", "--warmup", "3"], tmp_path)
    line = json.loads(outs[0][0].strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert line["config"]["instances_per_step"] == 96 and line["config"]["instances_per_gpu"] == 48
    assert line["verified"]["gather"].startswith("96 of 96 ciphertexts gathered")
    assert line["e2e"]["value"] > 0 and line["value"] > 0
    assert outs[1][0].strip() == ""  # only rank 0 prints
    assert "hgm_comm: rank 1 of 2" in outs[1][1]


def test_bench_cfg5_two_ranks(tmp_path):
    outs = launch(2, ["bench.py", "--gpus", "2", "--config", "cfg5", "--instances", "1", "--steps", "1",
                      "--warmup", "3", "--no-e2e"], tmp_path, id_file=False)
    line = json.loads(outs[0][0].strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["row_blocks_per_gpu"] == 4
    assert line["verified"]["value"].startswith("1 of 1 128^3 products")


SHARDED = r"""
import json, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2405_02238_b200 as hb
from paper_2405_02238_b200.dist import blocked_mm_sharded, comm_from_env, env_rank, sharded_matmul
from paper_2405_02238_b200.workload import splitmix_matrices
rank, world, _ = env_rank()
ctx = hb.Context(0, 1, 0)
comm = comm_from_env(ctx)
rng = np.random.default_rng(9)
A = rng.integers(-9, 10, (100, 100)); B = rng.integers(-9, 10, (100, 100))
C, ndec = blocked_mm_sharded(ctx, A, B, [50, 50], [50, 50], [50, 50], algo=1, comm=comm)
A2, B2 = splitmix_matrices(3, 0, 32, 16, 8, -8, 7)
C2 = sharded_matmul(ctx, A2, B2, 4, algo=1, comm=comm)
# the words rank 0 decrypts equal a single-GPU run's
single = None
if rank == 0:
    _, _, _, w1, _ = ctx.blocked_mm_acc(A, B, [50, 50], [50, 50], [50, 50], algo=1, counter0=0, export="only")
    single = w1
comm.barrier()
out = {"rank": rank}
if rank == 0:
    out.update(ok=bool(np.array_equal(C, (A @ B) % 65537)), ndec=ndec,
               ok2=bool(np.array_equal(C2, (A2 @ B2) % 65537)))
print(json.dumps(out))
comm.close()
"""


def test_sharded_blocked_and_rowblocks_three_ranks(tmp_path):
    script = tmp_path / "sharded.py"
    script.write_text(SHARDED)
    outs = launch(3, [str(script)], tmp_path)
    res = json.loads(outs[0][0].strip().splitlines()[-1])
    assert res["ok"] and res["ok2"] and res["ndec"] == 4
