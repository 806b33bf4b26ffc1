"""CPU: the C-ABI library loads and exports every symbol include/hegmm_b200.h
declares (no compute calls: there is no GPU here); the Python mirror binds them."""
import os
import re

import pytest

import paper_2405_02238_b200 as hb

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "hegmm_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hgm_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = hb.lib()
    names = declared_symbols()
    assert len(names) >= 40
    for name in names:
        assert hasattr(lib, name), name


def test_python_mirror_covers_the_header():
    assert sorted(hb.EXPORTS) == declared_symbols()


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", hb.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_\d+a?", out.stdout))
    assert archs == {"sm_100a"}, archs


def test_no_gpu_context_fails_loudly():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(hb.HEError):
        hb.Context(2, 1, 0)


def test_nccl_unique_id_without_gpu():
    """The communicator bootstrap id is produced by the library (NCCL, no torch)."""
    a, b = hb.Comm.unique_id(), hb.Comm.unique_id()
    assert len(a) == 128 and a != b


def test_chacha20_known_answer():
    """The OS-seeded sampler's block function: ChaCha20 with an all-zero key,
    nonce and counter gives the published keystream 76 b8 e0 ad a0 f1 3d 90 ..."""
    import numpy as np

    out = hb.chacha_block(np.zeros(8, dtype=np.uint32), 0, 0, 20)
    stream = out.astype("<u4").tobytes()
    assert stream[:16].hex() == "76b8e0ada0f13d90405d6ae55386bd28"
    assert stream[16:32].hex() == "bdd219b8a08ded1aa836efcc8b770dc7"
    # block 1 differs, 12 rounds differ from 20
    assert not np.array_equal(hb.chacha_block(np.zeros(8, np.uint32), 0, 1, 20), out)
    assert not np.array_equal(hb.chacha_block(np.zeros(8, np.uint32), 0, 0, 12), out)
