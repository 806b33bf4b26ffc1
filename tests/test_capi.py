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
