"""The real-HE campaign (paper_2405_02238_b200/campaign.py)
against the reference's own run_campaign (costmodel.cpp:266-314, compiled in
place into oracle/_ref): the same shapes, resamples, op counts and Table-1 cost
estimates; on the GPU every product is exact and measured."""
import numpy as np
import pytest

from paper_2405_02238_b200 import campaign

ORDER = ("hegmm", "hegmm-en", "square-pad")


@pytest.fixture(scope="module")
def reflib():
    from oracle.bindings import RefLib

    if not RefLib.available():
        pytest.skip("reference build (oracle/_ref) not present")
    return RefLib


@pytest.mark.parametrize("lo,hi,seed", [(1, 16, 1), (1, 64, 7)])
def test_campaign_matches_reference(reflib, lo, hi, seed):
    cases = 40
    shapes, costs, exact, stats, resampled = reflib.campaign(cases, lo, hi, seed)
    res = campaign.run_campaign(cases, lo, hi, seed, ORDER, backend="cost-model")
    assert res["resampled"] == resampled
    for c in res["cases"]:
        i = c["case"]
        assert (c["m"], c["l"], c["n"]) == tuple(int(x) for x in shapes[i])
        for k, a in enumerate(ORDER):
            r = c["algos"][a]
            assert r["stats"] == [int(x) for x in stats[i, k]], (i, a)
            assert r["client_ms"] == pytest.approx(costs[i, k, 0], rel=1e-12)
            assert r["cloud_ms"] == pytest.approx(costs[i, k, 1], rel=1e-12)
    assert exact.all()


def test_campaign_draws_match_reference_entries(reflib):
    # the matrices themselves: the reference's product of the drawn pair is exact
    m, l, n, A, B, _ = campaign.draw_case(3, 5, 1, 16, ORDER, 4096, 8192)
    C, _ = reflib.mm(A, B, "basic")
    assert np.array_equal(C, (A @ B) % 65537)
    assert A.min() >= -9 and A.max() <= 9


@pytest.mark.gpu
def test_campaign_on_gpu_exact():
    res = campaign.run_campaign(12, 1, 16, 11, ORDER, backend="bfv-gpu")
    for c in res["cases"]:
        for a, r in c["algos"].items():
            assert r["exact"], (c["case"], a)
            assert r["measured_ms"] > 0
    assert len(res["measured_summaries"]) == 3
