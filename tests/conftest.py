import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libhegmm_b200.so)")
    config.addinivalue_line("markers", "slow: long CPU-oracle runs")


@pytest.fixture(scope="session")
def ref():
    from oracle.bindings import RefLib

    if not RefLib.available():
        pytest.skip("oracle/_ref/libhegmm_ref.so not built (needs /root/reference at build time)")
    return RefLib


_ORACLES = {}


@pytest.fixture(scope="session")
def oracle_factory():
    from oracle.bindings import Oracle

    def get(param_id=2, seed=1):
        key = (param_id, seed)
        if key not in _ORACLES:
            _ORACLES[key] = Oracle(param_id, seed)
        return _ORACLES[key]

    return get


_CTXS = {}


@pytest.fixture(scope="session")
def gpu_factory():
    import paper_2405_02238_b200 as hb

    def get(param_id=2, seed=1):
        key = (param_id, seed)
        if key not in _CTXS:
            _CTXS[key] = hb.Context(param_id, seed, 0)
        return _CTXS[key]

    return get
