"""Test configuration: `gpu` marker, repo paths, shared fixtures.

-m "not gpu": oracle vs golden fixtures, host logic, C-ABI load/exports, multi-process gloo
             logic (runs in the build container, no GPU).
-m gpu:      CUDA path through the C ABI vs the oracle and the reference's golden digests.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


@pytest.fixture(scope="session")
def golden_small():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "golden_small.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_configs():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "golden_configs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def small_inputs():
    import inputs
    return {name: (a, bd, L, rct) for name, a, bd, L, rct in inputs.small_inputs()}


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def golden_region():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "golden_region.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_tiles():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "golden_tiles.json")) as f:
        return json.load(f)
