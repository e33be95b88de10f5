import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer parity cases")


def pytest_collection_modifyitems(config, items):
    """`slow` cases (minutes, tens of GB of host RAM) run only when the
    marker expression asks for them (-m slow / -m "gpu and slow")."""
    if "slow" in (config.getoption("-m") or ""):
        return
    skip = pytest.mark.skip(reason="slow: select with -m slow")
    for item in items:
        if "slow" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def pkg():
    import paper_2404_01931_b200 as P
    return P


def random_velocities(rng_seed, *arrays):
    rng = np.random.default_rng(rng_seed)
    return [rng.normal(size=a) for a in arrays]
