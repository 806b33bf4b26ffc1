"""GPU: the alternative kernel paths stay bit-exact.

The library picks its NTT layout and kernel fusions once per process from the
environment (csrc/ntt.cu: HGM_NTT3, HGM_FUSED_KS, HGM_FUSED_CONV,
HGM_FUSED_FINISH, HGM_FUSED_TENSOR, HGM_NTT_CLUSTER).  Each variant re-runs the primitive
parity tests (every op against the CPU oracle, ciphertext words bit-exact) and
the HEGMM product tests in a fresh process with that environment."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = {
    "one-cta-ntt": {"HGM_NTT3": "0"},
    "general-lincomb": {"HGM_LC_MASKED": "0"},
    # N = 32768 as two HBM passes (outer 2-stage kernel + 2^13 blocks) instead of 4-CTA clusters
    "two-pass-n32768-ntt": {"HGM_NTT_CLUSTER": "0"},
    "fused-modup-moddown": {"HGM_FUSED_KS": "1"},
    "fused-modup": {"HGM_FUSED_KS": "u"},
    "unfused-conv-finish": {"HGM_FUSED_CONV": "0", "HGM_FUSED_FINISH": "0"},
    "fused-tensor": {"HGM_FUSED_TENSOR": "1"},
    "tensor-without-intt-stage": {"HGM_TENSOR_S1": "0"},
    # device mask cache bounded to 4 MB: masks are evicted between programs all the time
    "small-mask-cache": {"HGM_MASK_CACHE_MB": "4"},
}


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_parity(name):
    env = dict(os.environ)
    env.update(VARIANTS[name])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "-k", "not acceptance", "tests/test_gpu_parity.py", "tests/test_gpu_hegmm.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, f"{name}: {VARIANTS[name]}\n{r.stdout[-3000:]}\n{r.stderr[-2000:]}"


# Masked sums of rotations (csrc/engine.cpp, Schedule::ks_terms) run as one inner
# product over masked keys; the same sums rotation by rotation (k_ks_inner +
# k_lincomb_masked) must give the same ciphertext words: with the rewrite off, and
# with a masked-key cache too small for any program (the executor's fallback).
PLAN_VARIANTS = {
    "plan-sums-off": {"HGM_KS_PLAN": "0"},
    "masked-key-cache-too-small": {"HGM_MASKED_KEY_MB": "8"},
    "plan-tile-8": {"HGM_PLAN_TILE": "8"},
    # sums read only by their ModDown keep P^-1 acc over Q (masked keys scaled by P^-1):
    # off, and on with the unfused finishing pass (k_ks_finish's own prescaled path)
    "prescale-off": {"HGM_PRESCALE": "0"},
    "prescale-unfused-finish": {"HGM_FUSED_FINISH": "0"},
}


@pytest.mark.parametrize("name", sorted(PLAN_VARIANTS))
def test_plan_sum_variants(name):
    env = dict(os.environ)
    env.update(PLAN_VARIANTS[name])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "-k", "not acceptance", "tests/test_gpu_hegmm.py", "tests/test_gpu_ct_golden.py",
                        "tests/test_gpu_widen.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, f"{name}: {PLAN_VARIANTS[name]}\n{r.stdout[-3000:]}\n{r.stderr[-2000:]}"


def test_many_lockstep_chunks_exact():
    """hgm_matmul_batch over many lockstep chunks (a small memory share forces
    several): the pipelined decrypt's pinned double buffers are reused across
    chunks, and every product must still come back exact and in order."""
    code = (
        "import numpy as np, paper_2405_02238_b200 as hb\n"
        "from paper_2405_02238_b200.workload import batch\n"
        "ctx = hb.Context(0, 1, 0)\n"
        "A, B = batch(7, 0, 300, 64, 64, 64, -8, 7)\n"
        "C, _ = ctx.matmul_batch(A, B, algo=0)\n"
        "bad = [i for i in range(300) if not np.array_equal(C[i], (A[i] @ B[i]) % 65537)]\n"
        "assert not bad, bad\n"
        "print('ok')\n")
    env = dict(os.environ)
    env["HGM_LOCKSTEP_FRAC"] = "0.06"
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
