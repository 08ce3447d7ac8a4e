import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libfluidrank_b200.so")
    config.addinivalue_line("markers", "slow: large-size GPU case")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("small_runs.npz")


@pytest.fixture(scope="session")
def golden_csr():
    return load_golden("csr_cases.npz")


@pytest.fixture(scope="session")
def golden_configs():
    return load_golden("config_graphs.npz")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test without a visible CUDA device (no CPU fallback exists)")
    import paper_1202_6158_b200 as fr
    return fr
