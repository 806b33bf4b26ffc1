"""Host check of csrc/common.cuh's modular arithmetic (Shoup / Barrett products, the
column accumulator, reduce_acc and k_ks_plan's reduce_acc_wide) against unsigned
__int128, for every prime of every parameter set (tests/host/arith_check.cpp)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_common_arithmetic_against_int128(tmp_path):
    csrc = os.path.join(ROOT, "paper_2405_02238_b200", "csrc")
    exe = str(tmp_path / "arith_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", csrc, os.path.join(ROOT, "tests", "host", "arith_check.cpp"),
                    os.path.join(csrc, "params.cpp"), "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "arith ok" in out.stdout, out.stdout + out.stderr
